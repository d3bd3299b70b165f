"""End-to-end parity by forced replay (tests/replay.py) -- no logit escape hatch.

Every int4 decision of the B200 engine (activation sites and KV-cache codes, prefill and
decode) must equal the restatement's (oracle/quota_oracle.cpp, itself bit-exact with the
unmodified reference -- asserted here again for the R0 cases), except decisions the
restatement lists as lying within the GPU's fp32 error budget of a rounding tie; those
are replayed with the GPU's choice.  After that the retained token sets must be identical
and the logits within north_star's 1e-2 max-abs.

Shapes: BASELINE.json configs[0] (C1) in reference semantics (R0: static scales from the
reference's own fit_act_scales, SiLU d_ff = 4d, MHA) and north_star semantics (R1:
per-token scales, SwiGLU, GQA), a ragged batch, and the configs[1] C2 7B width at reduced
depth (3 layers, d 4096, 32 x 128 heads, SwiGLU 11008 / SiLU 16384, 576 + 64 tokens, the
[2]/[0.3] recipe, B = 2) in both modes.  (The unmodified reference itself cannot run the
7B width in a test: its column-strided fp64 matmul runs at ~0.1 GFLOP/s.)
"""
import os

import numpy as np
import pytest

import oracle as O
import paper_2604_17320_b200 as Q
from tests.replay import forced_replay

pytestmark = pytest.mark.gpu

LOGIT_ATOL = 1e-2  # north_star


def _engine(cfg, w, acts, max_batch, max_tokens, max_seq, max_decode):
    e = Q.Engine(Q.Config(n_layers=cfg.n_layers, d_model=cfg.d_model, n_heads=cfg.n_heads,
                          n_kv_heads=cfg.n_kv_heads, d_head=cfg.d_head, d_ff=cfg.d_ff, mlp=cfg.mlp,
                          act_mode=cfg.act_mode),
                 max_batch=max_batch, max_tokens=max_tokens, max_seq=max_seq, max_decode=max_decode)
    e.load_weights(w)
    if acts is not None:
        e.set_act_scales(acts)
    return e


def _run(cfg, w, acts, rec, seqs, n_decode, dec_seed, ref=None):
    """Engine run with capture + forced replay against the restatement; returns max |dlogit|."""
    B = len(seqs)
    O.Port.set_threads(max(1, (os.cpu_count() or 8) // B))
    port = O.Port(cfg)
    port.set_weights(w)
    port.prepare(acts)
    tot = sum(v + t for _, v, t, _ in seqs)
    smax = max(v + t for _, v, t, _ in seqs)
    e = _engine(cfg, w, acts, B, tot, smax, max(n_decode, 1))
    e.set_recipe(rec.candidate_layers, rec.keep_ratios, rec.weights, rec.v0, 4)
    e.capture(True)
    lg = e.prefill(np.concatenate([s[0] for s in seqs]).astype(np.float32), [s[1] for s in seqs],
                   [s[2] for s in seqs], v0=[s[3] for s in seqs])
    lg = lg.copy()
    traces = [e.trace(b) for b in range(B)]
    dec = [[O.synth_embeddings(1, cfg.d_model, seed=dec_seed + 100 * b + t)[0] for t in range(n_decode)]
           for b in range(B)]
    dlg = [e.decode(np.stack([dec[b][t] for b in range(B)]).astype(np.float32)).copy() for t in range(n_decode)]
    layouts = [e.layout(b) for b in range(B)]  # after the decode steps, like the restatement's
    gpu_recs = e.captured()
    e.close()

    def recipe_for(b):
        return rec

    res, forced = forced_replay(port, gpu_recs, seqs, recipe_for, dec)
    worst, off = 0.0, 0
    for b in range(B):
        rr = res[b]["run"].result()
        assert [(l, k) for l, k, _ in traces[b]] == [(l, k) for l, k, _ in rr.trace], b
        for (_, _, p1), (_, _, p2) in zip(traces[b], rr.trace):
            assert np.array_equal(p1, p2), ("retained set differs", b)
        v, t, pos = layouts[b]
        assert (v, t) == (rr.visual, rr.text) and np.array_equal(pos, rr.positions)
        n = rr.logits.shape[0]  # the prefill's final rows
        worst = max(worst, float(np.abs(lg[off:off + n].astype(np.float64) - rr.logits).max()))
        off += n
        for s in range(n_decode):
            worst = max(worst, float(np.abs(dlg[s][b].astype(np.float64) - res[b]["logits"][1 + s]).max()))
        if ref is not None and not forced[b]:  # R0: the restatement is the reference, bit for bit
            assert np.array_equal(rr.logits, ref[b].result().logits)
    assert worst <= LOGIT_ATOL, worst
    print(f"max |dlogit| {worst:.3e}; forced ties per sequence {[len(f) for f in forced]}")
    return worst


def _c1_r0():
    cfg = O.ModelCfg(n_layers=4, d_model=256, n_heads=4, n_kv_heads=4, d_head=64, d_ff=1024, weight_axis=2)
    ref = O.Ref(cfg, seed=7)
    w = O.synth_weights(cfg, seed=3)
    ref.set_weights(w)
    calib = [(O.synth_embeddings(144 + 16 + 4 * i, 256, seed=100 + i), 144, 16 + 4 * i) for i in range(4)]
    acts = ref.fit_act_scales(calib)
    ref.prepare(acts, weight_axis=2)
    return cfg, ref, w, acts


def test_replay_c1_r0_reference_semantics(torch_cuda):
    """C1 in reference semantics; the restatement is asserted bit-exact with the unmodified
    reference on the same inputs first."""
    cfg, ref, w, acts = _c1_r0()
    rec = O.Recipe([0, 1, 2, 3], [1.0, 0.5, 0.3, 0.3], v0=144)
    emb = O.synth_embeddings(184, 256, seed=11)
    rr = ref.prefill(emb, 144, 40, rec)
    port = O.Port(cfg)
    port.set_weights(w)
    port.prepare(acts)
    assert np.array_equal(port.prefill(emb, 144, 40, rec).result().logits, rr.result().logits)
    _run(cfg, w, acts, rec, [(emb, 144, 40, 144)], 16, 900, ref=[rr])


def test_replay_c1_ragged_batch_r0(torch_cuda):
    """Ragged batch with per-sequence v0 (C4-style), reference semantics."""
    cfg, _, w, acts = _c1_r0()
    rec = O.Recipe([1, 2], [0.5, 0.25], v0=144)
    seqs = [(O.synth_embeddings(v + t, 256, seed=50 + i), v, t, v) for i, (v, t) in
            enumerate([(144, 40), (100, 25), (144, 7)])]
    _run(cfg, w, acts, rec, seqs, 6, 500)


def test_replay_c1_r1_dynamic_swiglu_gqa(torch_cuda):
    cfg = O.ModelCfg(n_layers=4, d_model=256, n_heads=4, n_kv_heads=2, d_head=64, d_ff=688, mlp=1, act_mode=1,
                     weight_axis=2)
    w = O.synth_weights(cfg, seed=21)
    rec = O.Recipe([0, 1, 2, 3], [1.0, 0.5, 0.3, 0.3], v0=144)
    emb = O.synth_embeddings(184, 256, seed=13)
    _run(cfg, w, None, rec, [(emb, 144, 40, 144)], 16, 700)


def test_replay_c1_r1_decode_batch_40(torch_cuda):
    """A decode batch above the GEMV's 32 tokens: every decode GEMM runs on the int8-operand
    tcgen05 kernel (the narrow projections with k slices, tools/bench_decode_gemm.py), the
    attention merge writes the int8 activation copy; 40 ragged sequences, 3 decode steps."""
    cfg = O.ModelCfg(n_layers=4, d_model=256, n_heads=4, n_kv_heads=2, d_head=64, d_ff=688, mlp=1, act_mode=1,
                     weight_axis=2)
    w = O.synth_weights(cfg, seed=23)
    rec = O.Recipe([1, 2], [0.5, 0.3], v0=48)
    seqs = [(O.synth_embeddings(48 + 8 + i % 5, 256, seed=300 + i), 48, 8 + i % 5, 48) for i in range(40)]
    _run(cfg, w, None, rec, seqs, 3, 1700)


def _c2_weights(mlp, act_mode):
    cfg = O.ModelCfg(n_layers=3, d_model=4096, n_heads=32, n_kv_heads=32, d_head=128,
                     d_ff=11008 if mlp == 1 else 16384, mlp=mlp, act_mode=act_mode, weight_axis=2)
    return cfg, O.synth_weights(cfg, seed=31)


def _c2_seqs():
    # 576 visual + 64 text (configs[1]); the second sequence is a shorter ragged one
    return [(O.synth_embeddings(640, 4096, seed=41, outlier_frac=0.01), 576, 64, 576),
            (O.synth_embeddings(464, 4096, seed=42, outlier_frac=0.01), 400, 64, 400)]


def test_replay_c2_7b_width_r1(torch_cuda):
    """configs[1] C2 7B width (d_head 128, SwiGLU 11008, K = 4096 / 11008 GEMMs and the
    decode GEMV down projection), per-token scales, reduced to 3 layers, pruning 30 % at
    layer 2, 4 decode steps."""
    cfg, w = _c2_weights(1, 1)
    _run(cfg, w, None, O.Recipe([2], [0.3], v0=576), _c2_seqs(), 4, 1300)


def test_replay_c2_7b_width_r0(torch_cuda):
    """The same width in reference semantics (static scales, SiLU d_ff = 4d = 16384, MHA).
    The static scales come from the engine's fp64 fit_act_scales (which tests/
    test_calibration_gpu.py pins to the reference's to 1e-10); both sides use the same
    values."""
    cfg, w = _c2_weights(0, 0)
    e = Q.Engine(Q.Config(n_layers=3, d_model=4096, n_heads=32, n_kv_heads=32, d_head=128, d_ff=16384, mlp=0,
                          act_mode=0), max_batch=1, max_tokens=640, max_seq=640, max_decode=1)
    e.keep_fp_weights(True)
    e.load_weights(w)
    acts = e.fit_act_scales([(O.synth_embeddings(640, 4096, seed=60 + i, outlier_frac=0.01), 576, 64)
                             for i in range(2)])
    e.close()
    _run(cfg, w, acts, O.Recipe([2], [0.3], v0=576), _c2_seqs(), 2, 1500)


def test_replay_c4_qwen2vl_width_gqa(torch_cuda):
    """configs[3] C4 width (Qwen2-VL-7B shape: d 3584, 28 query / 4 kv heads x 128 -- GQA 7,
    SwiGLU 18944) at reduced depth (2 layers), a ragged pair of sequences with their own
    visual lengths, 30 % retention at layer 1, 3 decode steps (the 9..16-token decode GEMV
    does not apply at B = 2; the GQA-7 decode attention and the d = 3584 GEMVs do)."""
    cfg = O.ModelCfg(n_layers=2, d_model=3584, n_heads=28, n_kv_heads=4, d_head=128, d_ff=18944, mlp=1,
                     act_mode=1, weight_axis=2)
    w = O.synth_weights(cfg, seed=37)
    seqs = [(O.synth_embeddings(420 + 64, 3584, seed=43, outlier_frac=0.01), 420, 64, 420),
            (O.synth_embeddings(256 + 64, 3584, seed=44, outlier_frac=0.01), 256, 64, 256)]
    _run(cfg, w, None, O.Recipe([1], [0.3], v0=420), seqs, 3, 1900)
