import sys, numpy as np
sys.path.insert(0, "/root/repo")
import oracle as O, paper_2604_17320_b200 as Q
def run(cfg, w, acts, mlp, act_mode, seedbase, nsteps=24):
    port = O.Port(cfg); port.set_weights(w); port.prepare(acts)
    rec = O.Recipe([0, 1, 2, 3], [1.0, 0.5, 0.3, 0.3], v0=144)
    emb = O.synth_embeddings(184, cfg.d_model, seed=seedbase)
    pr = port.prefill(emb, 144, 40, rec); res = pr.result()
    e = Q.Engine(Q.Config(n_layers=cfg.n_layers, d_model=cfg.d_model, n_heads=cfg.n_heads, n_kv_heads=cfg.n_kv_heads,
                          d_head=cfg.d_head, d_ff=cfg.d_ff, mlp=mlp, act_mode=act_mode), max_batch=2, max_tokens=2048,
                 max_seq=512, max_decode=nsteps)
    e.load_weights(w)
    if acts is not None: e.set_act_scales(acts)
    e.set_recipe(rec.candidate_layers, rec.keep_ratios, rec.weights, rec.v0, 4)
    lg = e.prefill(emb.astype(np.float32), [144], [40])
    print("prefill err", np.abs(lg - res.logits).max(), "margin", pr.tie_margin(0), flush=True)
    for step in range(nsteps):
        de = O.synth_embeddings(1, cfg.d_model, seed=seedbase * 100 + step)
        r = pr.decode(de[0]); g = e.decode(de.astype(np.float32))[0]
        print("step", step, "err %.3g" % np.abs(g - r).max(), "margin %.3g" % pr.tie_margin(1), flush=True)
cfg = O.ModelCfg(n_layers=4, d_model=256, n_heads=4, n_kv_heads=4, d_head=64, d_ff=1024, weight_axis=2)
w = O.synth_weights(cfg, seed=3)
ref = O.Ref(cfg, seed=7); ref.set_weights(w)
calib = [(O.synth_embeddings(144 + 16 + 4 * i, 256, seed=100 + i), 144, 16 + 4 * i) for i in range(4)]
acts = ref.fit_act_scales(calib)
print("== R0"); run(cfg, w, acts, 0, 0, 11)
print("== R0 dynamic"); cfg.act_mode = 1; run(cfg, w, None, 0, 1, 12)
cfg2 = O.ModelCfg(n_layers=4, d_model=256, n_heads=4, n_kv_heads=2, d_head=64, d_ff=688, mlp=1, act_mode=1, weight_axis=2)
w2 = O.synth_weights(cfg2, seed=21)
print("== R1 gqa swiglu"); run(cfg2, w2, None, 1, 1, 13)
cfg3 = O.ModelCfg(n_layers=4, d_model=256, n_heads=4, n_kv_heads=4, d_head=64, d_ff=688, mlp=1, act_mode=1, weight_axis=2)
w3 = O.synth_weights(cfg3, seed=21)
print("== R1 mha swiglu"); run(cfg3, w3, None, 1, 1, 13)
