import sys, numpy as np
import os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O, paper_2604_17320_b200 as Q
cfg = O.ModelCfg(n_layers=4, d_model=256, n_heads=4, n_kv_heads=2, d_head=64, d_ff=688, mlp=1, act_mode=1, weight_axis=2)
w = O.synth_weights(cfg, seed=21)
port = O.Port(cfg); port.set_weights(w); port.prepare(None)
rec = O.Recipe([0, 1, 2, 3], [1.0, 0.5, 0.3, 0.3], v0=144)
emb = O.synth_embeddings(184, 256, seed=13)
pr = port.prefill(emb, 144, 40, rec); res = pr.result()
m, f = pr.last_scores()
fs = np.sort(f)[::-1]
pass
e = Q.Engine(Q.Config(n_layers=4, d_model=256, n_heads=4, n_kv_heads=2, d_head=64, d_ff=688, mlp=1, act_mode=1),
             max_batch=4, max_tokens=4096, max_seq=1024, max_decode=16)
e.load_weights(w)
e.set_recipe(rec.candidate_layers, rec.keep_ratios, rec.weights, rec.v0, 4)
ref_l = None; ref_pos = None
for it in range(30):
    lg = e.prefill(emb.astype(np.float32), [144], [40]).copy()
    v, t, pos = e.layout(0)
    tr = e.trace(0)
    if ref_l is None:
        ref_l, ref_pos, ref_tr = lg, pos, tr
        print("port==gpu layout", np.array_equal(pos, res.positions), [(a[0], a[1]) for a in tr], flush=True)
    else:
        same = np.array_equal(pos, ref_pos) and np.array_equal(lg, ref_l)
        if not same:
            print("run", it, "DIFFERS: pos equal", np.array_equal(pos, ref_pos), "max dlogit", float(np.abs(lg - ref_l).max()) if lg.shape == ref_l.shape else "shape",
                  [ (x[0], np.setdiff1d(x[2], y[2]).tolist(), np.setdiff1d(y[2], x[2]).tolist()) for x, y in zip(tr, ref_tr)], flush=True)
print("done")
