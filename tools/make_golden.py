#!/usr/bin/env python3
"""Generate the committed golden fixtures under tests/golden/ from the UNMODIFIED
reference library (oracle/_ref/libquota_ref.so, built by `make -C oracle ref`
from /root/reference/proj/src where it lies).  Run here, in the container that
has /root/reference; the fixtures then travel with the repo (the GPU box has no
/root/reference).

  c1_r0.npz   BASELINE.json configs[0] through the reference forward_prefill +
              decode_step (quantized mode, recipe hook), reference semantics:
              SiLU MLP d_ff = 4d, MHA, static per-tensor activation scales from
              the reference's own fit_act_scales; weights per output channel
              (GroupAxis::PerColumn).
  kats.json   kernel-level known answers from the reference primitives:
              quantizer codes/scales, kv_quantize, percentile, robust_normalize,
              select_top_k, compute_budget, parse_recipe errors.

Inputs are regenerated from the seeds stored in the fixture (numpy
default_rng, oracle.synth_*), so the fixtures hold only outputs.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")

C1 = dict(L=4, d=256, H=4, V=144, T=40, wseed=3, eseed=11, calib_seeds=[100, 101, 102, 103],
          layers=[0, 1, 2, 3], keeps=[1.0, 0.5, 0.3, 0.3], v0=144, dec_seeds=[900, 901, 902, 903])


def c1_setup():
    c = C1
    cfg = O.ModelCfg(n_layers=c["L"], d_model=c["d"], n_heads=c["H"], n_kv_heads=c["H"], d_head=c["d"] // c["H"],
                     d_ff=4 * c["d"], weight_axis=2)
    ref = O.Ref(cfg, seed=7)
    w = O.synth_weights(cfg, seed=c["wseed"])
    ref.set_weights(w)
    calib = [(O.synth_embeddings(c["V"] + 16 + 4 * i, c["d"], seed=s), c["V"], 16 + 4 * i)
             for i, s in enumerate(c["calib_seeds"])]
    acts = ref.fit_act_scales(calib)
    ref.prepare(acts, weight_axis=2)
    emb = O.synth_embeddings(c["V"] + c["T"], c["d"], seed=c["eseed"])
    rec = O.Recipe(c["layers"], c["keeps"], v0=c["v0"])
    return cfg, ref, w, acts, emb, rec


def make_c1():
    cfg, ref, w, acts, emb, rec = c1_setup()
    rr = ref.prefill(emb, C1["V"], C1["T"], rec)
    res = rr.result()
    out = dict(act_scales=acts, logits=res.logits, visual=res.visual, text=res.text, positions=res.positions,
               logits_fnv=np.uint64(O.ref_lib().qref_fnv1a64(O._d(O.f64(res.logits)), res.logits.size)))
    for i, (lay, bud, pos) in enumerate(res.trace):
        out[f"trace{i}_layer"] = lay
        out[f"trace{i}_budget"] = bud
        out[f"trace{i}_positions"] = pos
    out["n_prunes"] = len(res.trace)
    for l in range(cfg.n_layers):
        for which, nm in ((0, "k"), (1, "v")):
            codes = []
            scales = []
            for h in range(cfg.n_heads):
                c, s, p = rr.kv(l, h, which)
                codes.append(c)
                scales.append(s)
            out[f"kv{l}_{nm}_codes"] = np.stack(codes)
            out[f"kv{l}_{nm}_scales"] = np.stack(scales)
            out[f"kv{l}_pos"] = p
    dec = []
    for s in C1["dec_seeds"]:
        dec.append(rr.decode(O.synth_embeddings(1, cfg.d_model, seed=s)[0]))
    out["decode_logits"] = np.stack(dec)
    out["config"] = json.dumps(C1)
    np.savez_compressed(os.path.join(OUT, "c1_r0.npz"), **out)
    print("c1_r0.npz", res.logits.shape, [(l, b) for l, b, _ in res.trace])


def make_kats():
    rng = np.random.default_rng(2024)
    k = {}
    # quantizer (quant.cpp:47-106): per-row, per-column, per-tensor fits, incl. an all-zero row
    x = rng.normal(0, 1, size=(6, 40))
    x[2] = 0.0
    x[4, 5] = 25.0
    for ax in (0, 1, 2):
        c, s = O.ref_quantize_fit(x, ax)
        k[f"quant_axis{ax}"] = dict(codes=c.tolist(), scales=s.tolist())
    k["quant_x"] = x.tolist()
    kv = rng.normal(0, 1, size=(5, 64))
    kv[1] = 0.0
    c, s = O.ref_kv_quantize(kv)
    k["kv_x"] = kv.tolist()
    k["kv"] = dict(codes=c.tolist(), scales=s.tolist())
    # percentile / robust_normalize (numeric.cpp:84-96, selector.cpp:70-84)
    v = rng.normal(0, 1, size=37)
    k["pct_v"] = v.tolist()
    k["pct"] = {str(p): O.ref_percentile(v, p) for p in (0, 5, 50, 95, 100)}
    k["robust"] = O.ref_robust_normalize(v).tolist()
    k["robust_const"] = O.ref_robust_normalize(np.full(9, 3.5)).tolist()
    # select_top_k (selector.cpp:117-136), including ties and -0.0 vs +0.0
    cases = [([0.1, 0.9, 0.5], 2), ([0.5, 0.5, 0.5], 2), ([0.0, -0.0, 0.0, 1.0], 2), ([3.0, 1.0], 5),
             (rng.integers(0, 4, size=50).astype(float).tolist(), 17), (rng.normal(0, 1, 300).tolist(), 90)]
    k["topk"] = [dict(scores=list(map(float, s)), k=kk, slots=O.ref_select_top_k(s, kk).tolist()) for s, kk in cases]
    # compute_budget (selector.cpp:11-17)
    k["budget"] = [dict(r=r, v0=v0, k=O.ref_compute_budget(r, v0))
                   for r, v0 in ((0.3, 576), (0.5, 144), (0.3, 144), (1.0, 144), (0.25, 2880), (0.2, 2880),
                                 (0.3, 1), (1e-9, 100))]
    # parse_recipe errors (recipe.cpp:21-46,65-116): message per malformed recipe
    good = O.Recipe([2], [0.3], v0=576).to_json()
    bad = {
        "unknown_key": good[:-1] + ', "extra": 1}',
        "schema": good.replace('"schema_version": 1', '"schema_version": 2'),
        "not_increasing": O.Recipe([2, 2], [0.5, 0.3], v0=576).to_json(),
        "keep_increasing": O.Recipe([1, 2], [0.3, 0.5], v0=576).to_json(),
        "keep_zero": O.Recipe([1], [0.0], v0=576).to_json(),
        "weights_sum": O.Recipe([1], [0.5], weights=(0.5, 0.5, 0.5, 0.5), v0=576).to_json(),
        "v0_zero": O.Recipe([1], [0.5], v0=0).to_json(),
        "missing": '{"schema_version": 1}',
        "syntax": '{"schema_version": 1,',
    }
    k["recipe_good"] = dict(text=good, parsed=O.ref_parse_recipe(good))
    errs = {}
    for name, txt in bad.items():
        try:
            O.ref_parse_recipe(txt)
            errs[name] = dict(text=txt, error=None)
        except O.OracleError as e:
            errs[name] = dict(text=txt, error=str(e))
    k["recipe_bad"] = errs
    with open(os.path.join(OUT, "kats.json"), "w") as f:
        json.dump(k, f, indent=0)
    print("kats.json", len(k))


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    make_kats()
    make_c1()
