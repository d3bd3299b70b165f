import sys, os, numpy as np
sys.path.insert(0, "/root/repo")
import oracle as O, paper_2604_17320_b200 as Q
cfg = O.ModelCfg(n_layers=4, d_model=256, n_heads=4, n_kv_heads=4, d_head=64, d_ff=1024, weight_axis=2, act_mode=1)
w = O.synth_weights(cfg, seed=3)
port = O.Port(cfg); port.set_weights(w); port.prepare(None)
rec = O.Recipe([0, 1, 2, 3], [1.0, 0.5, 0.3, 0.3], v0=144)
emb = O.synth_embeddings(184, 256, seed=12)
e = Q.Engine(Q.Config(n_layers=4, d_model=256, n_heads=4, n_kv_heads=4, d_head=64, d_ff=1024, act_mode=1), max_batch=2, max_tokens=2048, max_seq=512, max_decode=24)
e.load_weights(w)
for variant in ["recipe", "norecipe"]:
    if variant == "recipe":
        e.set_recipe(rec.candidate_layers, rec.keep_ratios, rec.weights, rec.v0, 4); r = rec
    else:
        e.clear_recipe(); r = None
    outs = []
    for rep in range(2):
        pr = port.prefill(emb, 144, 40, r)
        lg = e.prefill(emb.astype(np.float32), [144], [40])
        o = []
        for step in range(8):
            de = O.synth_embeddings(1, 256, seed=1200 + step)
            g = e.decode(de.astype(np.float32))[0].copy()
            ref = pr.decode(de[0])
            o.append(g)
            print(variant, rep, step, "err vs ref %.3g" % np.abs(g - ref).max(), flush=True)
        outs.append(np.array(o))
    print(variant, "run-to-run max diff", np.abs(outs[0] - outs[1]).max())
