"""Cross-process check of the R1 tiny prefill: retained sets and fused scores vs the port."""
import os, sys, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

def one():
    import oracle as O, paper_2604_17320_b200 as Q
    cfg = O.ModelCfg(n_layers=4, d_model=256, n_heads=4, n_kv_heads=2, d_head=64, d_ff=688, mlp=1, act_mode=1,
                     weight_axis=2)
    w = O.synth_weights(cfg, seed=21)
    port = O.Port(cfg); port.set_weights(w); port.prepare(None)
    rec = O.Recipe([0, 1, 2], [1.0, 0.5, 0.3], v0=144)
    emb = O.synth_embeddings(184, 256, seed=13)
    pr = port.prefill(emb, 144, 40, rec); res = pr.result()
    m, f = pr.last_scores()
    e = Q.Engine(Q.Config(n_layers=4, d_model=256, n_heads=4, n_kv_heads=2, d_head=64, d_ff=688, mlp=1, act_mode=1),
                 max_batch=4, max_tokens=4096, max_seq=1024, max_decode=16)
    e.load_weights(w)
    e.set_recipe(rec.candidate_layers, rec.keep_ratios, rec.weights, rec.v0, 4)
    lg = e.prefill(emb.astype(np.float32), [144], [40])
    tr = e.trace(0)
    last = res.trace[-1][0]
    gf, gm = e.scores(last, 0)
    K = res.trace[-1][1]
    fs = np.sort(f)[::-1]
    gap = (fs[K - 1] - fs[K]) / max(abs(fs[K - 1]), 1e-30)
    same = [np.array_equal(a[2], b[2]) for a, b in zip(tr, res.trace)]
    print("same per layer", same, "max|dfused| %.3g" % np.abs(gf - f).max(), "boundary gap rel %.3g" % gap,
          "max|dlogit| %.3g" % (np.abs(lg - res.logits).max() if lg.shape == res.logits.shape else -1))
    for a, b in zip(tr, res.trace):
        if not np.array_equal(a[2], b[2]):
            print("  layer", a[0], "gpu-only", np.setdiff1d(a[2], b[2]), "port-only", np.setdiff1d(b[2], a[2]))

if __name__ == "__main__":
    if len(sys.argv) > 1:
        one()
    else:
        for i in range(int(os.environ.get("N", "6"))):
            r = subprocess.run([sys.executable, __file__, "one"], capture_output=True, text=True, timeout=300)
            print(r.stdout.strip(), r.stderr[-500:] if r.returncode else "")
