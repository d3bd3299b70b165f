"""Parity across the BASELINE.json config families, at sizes the
CPU oracle finishes in seconds, plus size-independent properties at the full
7B shape.

  C3-like  long visual prefix with a multi-layer keep schedule [1, 1, 0.25, 0.2]
  C4-like  ragged packed batch, GQA, per-sequence v0 (varlen visual lengths)
  C5-like  decode sweep: batch 16 (GEMV path) and 40 (tcgen05 GEMM path), long decode
  C2 full  7B shape: budgets, ordering, determinism, identity recipe, scores

Reference semantics for the north_star switches (per-token scales, SwiGLU, GQA)
come from the restatement oracle (pinned to the reference in test_oracle_cpu).
Retained sets must match except at reference score near-ties (< 1e-4 relative,
north_star); logits within 1e-2 max-abs."""
import numpy as np
import pytest

import oracle as O
import paper_2604_17320_b200 as Q

pytestmark = pytest.mark.gpu
ATOL = 1e-2


def _pair(cfg, seed=21, max_batch=8, max_tokens=8192, max_seq=4096, max_decode=64):
    w = O.synth_weights(cfg, seed=seed)
    port = O.Port(cfg)
    port.set_weights(w)
    port.prepare(None)
    e = Q.Engine(Q.Config(n_layers=cfg.n_layers, d_model=cfg.d_model, n_heads=cfg.n_heads, n_kv_heads=cfg.n_kv_heads,
                          d_head=cfg.d_head, d_ff=cfg.d_ff, mlp=cfg.mlp, act_mode=cfg.act_mode),
                 max_batch=max_batch, max_tokens=max_tokens, max_seq=max_seq, max_decode=max_decode)
    e.load_weights(w)
    return port, e


def _gap(port, emb, v, t, rec, layer, v0):
    upto = [i for i, l in enumerate(rec.candidate_layers) if l <= layer]
    r = O.Recipe([rec.candidate_layers[i] for i in upto], [rec.keep_ratios[i] for i in upto], rec.weights, v0=v0)
    _, f = port.prefill(emb, v, t, r).last_scores()
    k = int(np.ceil(r.keep_ratios[-1] * v0))
    fs = np.sort(f)[::-1]
    return np.inf if k >= len(fs) else (fs[k - 1] - fs[k]) / max(abs(fs[k - 1]), 1e-300)


def _check_seq(port, e, i, emb, v, t, rec, v0, logits):
    res = port.prefill(emb, v, t, rec, v0=v0).result()
    tr = e.trace(i)
    assert [(a, b) for a, b, _ in tr] == [(a, b) for a, b, _ in res.trace]
    for (l, _, p1), (_, _, p2) in zip(tr, res.trace):
        if not np.array_equal(p1, p2):
            gap = _gap(port, emb, v, t, rec, l, v0)
            assert gap < 1e-4, ("retained set differs at a clear score gap", l, gap)
            return None
    assert np.array_equal(e.layout(i)[2], res.positions)
    assert np.abs(logits - res.logits).max() <= ATOL
    return res


def test_c3_long_prefix_schedule():
    cfg = O.ModelCfg(n_layers=4, d_model=128, n_heads=2, n_kv_heads=2, d_head=64, d_ff=344, mlp=1, act_mode=1,
                     weight_axis=2)
    port, e = _pair(cfg)
    V, T = 1440, 64
    rec = O.Recipe([0, 1, 2, 3], [1.0, 1.0, 0.25, 0.2], v0=V)
    e.set_recipe(rec.candidate_layers, rec.keep_ratios, rec.weights, rec.v0, 4)
    emb = O.synth_embeddings(V + T, 128, seed=31, outlier_frac=0.01)
    lg = e.prefill(emb.astype(np.float32), [V], [T])
    assert [(l, b) for l, b, _ in e.trace(0)] == [(2, 360), (3, 288)]
    if _check_seq(port, e, 0, emb, V, T, rec, V, lg) is None:
        return  # near-tie flip upstream: later scores legitimately differ
    # fused scores at the last pruning layer, end to end.  Upstream of it sit ~10^5
    # per-token int4 activation quantizations whose fp32 GPU inputs can flip a code
    # at a rounding tie (the port's tie margin reports such ties); a flip moves the
    # residual by one quantization step, so end-to-end scores are held to 1e-2.
    # Given identical metrics the scores are bit-exact (test_select_gpu).
    f_gpu, _ = e.scores(3, 0)
    r3 = port.prefill(emb, V, T, rec)
    _, f_ref = r3.last_scores()
    assert f_gpu.shape == f_ref.shape
    assert np.abs(f_gpu - f_ref).max() <= 1e-2


def test_c4_ragged_gqa_batch_with_decode():
    cfg = O.ModelCfg(n_layers=4, d_model=256, n_heads=4, n_kv_heads=2, d_head=64, d_ff=688, mlp=1, act_mode=1,
                     weight_axis=2)
    port, e = _pair(cfg)
    Vs, T = [60, 150, 97, 200], 24
    rec = O.Recipe([2], [0.3], v0=1)
    e.set_recipe(rec.candidate_layers, rec.keep_ratios, rec.weights, 1, 4)
    embs = [O.synth_embeddings(v + T, 256, seed=40 + i) for i, v in enumerate(Vs)]
    lg = e.prefill(np.concatenate(embs).astype(np.float32), Vs, [T] * 4, v0=Vs)
    off = 0
    runs = []
    for i, v in enumerate(Vs):
        vv, tt, _ = e.layout(i)
        n = vv + tt
        assert vv == int(np.ceil(0.3 * v))
        runs.append(_check_seq(port, e, i, embs[i], v, T, O.Recipe([2], [0.3], v0=v), v, lg[off:off + n]))
        off += n
    decs = [O.synth_embeddings(4, 256, seed=500 + s) for s in range(8)]
    prs = [port.prefill(embs[i], v, T, O.Recipe([2], [0.3], v0=v)) for i, v in enumerate(Vs)]
    for s in range(8):
        g = e.decode(decs[s].astype(np.float32))
        for i in range(4):
            r = prs[i].decode(decs[s][i])
            if runs[i] is not None:
                assert np.abs(g[i] - r).max() <= ATOL, (s, i)


@pytest.mark.parametrize("B,steps", [(16, 48), (40, 12)])
def test_c5_decode_sweep_batches(B, steps):
    cfg = O.ModelCfg(n_layers=4, d_model=256, n_heads=4, n_kv_heads=4, d_head=64, d_ff=688, mlp=1, act_mode=1,
                     weight_axis=2)
    port, e = _pair(cfg, max_batch=B, max_decode=steps + 1)
    V, T = 52, 20  # an already-pruned prefix (173 + 64 at the 7B shape)
    e.clear_recipe()
    embs = [O.synth_embeddings(V + T, 256, seed=900 + i) for i in range(B)]
    e.prefill(np.concatenate(embs).astype(np.float32), [V] * B, [T] * B)
    dec = [O.synth_embeddings(B, 256, seed=1200 + s) for s in range(steps)]
    got = None
    for s in range(steps):
        got = e.decode(dec[s].astype(np.float32))
    exp = port.run_batch(embs, [V] * B, [T] * B, O.Recipe([0], [1.0], v0=V), [V] * B, steps,
                         [np.stack([dec[s][i] for s in range(steps)]) for i in range(B)], n_threads=8)
    assert np.abs(got - exp).max() <= ATOL


def test_c2_full_shape_properties():
    """7B shape (32 layers x 4096, SwiGLU 11008) at batch 2: budgets 173, ascending
    retained positions inside the visual range, bit-identical repeat, identity recipe
    == no recipe, finite logits, scores in [0, 1]."""
    import torch
    c = Q.Config(n_layers=32, d_model=4096, n_heads=32, n_kv_heads=32, d_head=128, d_ff=11008, mlp=1, act_mode=1)
    B, V, T = 2, 576, 64
    e = Q.Engine(c, max_batch=B, max_tokens=B * (V + T), max_seq=V + T, max_decode=4)
    g = torch.Generator(device="cuda").manual_seed(5)
    rnd = lambda *s: torch.randn(*s, device="cuda", generator=g) * 0.02
    for l in range(32):
        e.load_layer(l, rnd(4096, 4096), rnd(4096, 4096), rnd(4096, 4096), rnd(4096, 4096), rnd(4096, 11008),
                     rnd(11008, 4096), rnd(4096, 11008))
    e.load_head(rnd(4096, 4096))
    emb = torch.randn(B * (V + T), 4096, generator=torch.Generator().manual_seed(3))
    emb[:, :41] *= 20.0
    e.set_recipe([2], [0.3], v0=576)
    a = e.prefill(emb.numpy(), [V] * B, [T] * B).copy()
    tr = [e.trace(i) for i in range(B)]
    b = e.prefill(emb.numpy(), [V] * B, [T] * B).copy()
    assert np.array_equal(a, b)
    assert np.isfinite(a).all() and a.shape == (B * (173 + T), 4096)
    for i in range(B):
        (l, bud, pos), = tr[i]
        assert (l, bud) == (2, 173) and len(pos) == 173
        assert np.all(np.diff(pos) > 0) and pos[0] >= 0 and pos[-1] < V
        f, m = e.scores(2, i)
        assert f.shape == (576,) and np.all((m >= 0) & (m <= 1))
    e.set_recipe([2], [1.0], v0=576)
    c1 = e.prefill(emb.numpy(), [V] * B, [T] * B).copy()
    e.clear_recipe()
    c2 = e.prefill(emb.numpy(), [V] * B, [T] * B).copy()
    assert np.array_equal(c1, c2)
    out = e.decode(np.random.default_rng(0).standard_normal((B, 4096)).astype(np.float32))
    assert np.isfinite(out).all()
    e.close()
