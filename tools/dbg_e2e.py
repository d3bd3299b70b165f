import sys, time, numpy as np
sys.path.insert(0, "/root/repo")
import oracle as O, paper_2604_17320_b200 as Q
def log(*a):
    print(*a, flush=True)
cfg = O.ModelCfg(n_layers=4, d_model=256, n_heads=4, n_kv_heads=4, d_head=64, d_ff=1024, weight_axis=2)
w = O.synth_weights(cfg, seed=3)
acts = np.full(4*4+1, 0.5)
log("create")
e = Q.Engine(Q.Config(n_layers=4, d_model=256, n_heads=4, n_kv_heads=4, d_head=64, d_ff=1024), max_batch=4, max_tokens=4096, max_seq=1024, max_decode=16)
log("load")
e.load_weights(w); e.set_act_scales(acts)
e.set_recipe([0,1,2,3],[1.0,0.5,0.3,0.3], v0=144)
emb = O.synth_embeddings(184, 256, seed=11).astype(np.float32)
log("prefill")
lg = e.prefill(emb, [144], [40]); log("prefill done", lg.shape, e.trace(0)[0][:2] if e.trace(0) else None)
for s in range(3):
    g = e.decode(O.synth_embeddings(1,256,seed=9+s).astype(np.float32)); log("decode", s, g[0,:3])
