"""In-process determinism stress: ragged R0 batch prefill + B=40 decode, repeated; prints
how many distinct output hashes each case produced."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import oracle as O
import paper_2604_17320_b200 as Q

N = int(sys.argv[1]) if len(sys.argv) > 1 else 20
h = lambda a: hashlib.md5(np.ascontiguousarray(a).tobytes()).hexdigest()[:10]

# case 1: ragged R0-mode batch (test_r0_batch_of_sequences...)
cfg = O.ModelCfg(n_layers=4, d_model=256, n_heads=4, n_kv_heads=4, d_head=64, d_ff=1024, weight_axis=2)
w = O.synth_weights(cfg, seed=3)
e = Q.Engine(Q.Config(n_layers=4, d_model=256, n_heads=4, n_kv_heads=4, d_head=64, d_ff=1024),
             max_batch=4, max_tokens=4096, max_seq=1024, max_decode=16)
e.load_weights(w)
e.set_act_scales(np.full(17, 0.07))
e.set_recipe([1, 2], [0.5, 0.25], v0=144)
vis, txt = [144, 100, 144], [40, 25, 7]
emb = np.concatenate([O.synth_embeddings(v + t, 256, seed=50 + i) for i, (v, t) in enumerate(zip(vis, txt))])
seen = {}
for it in range(N):
    lg = e.prefill(emb.astype(np.float32), vis, txt, v0=[144, 100, 144])
    key = h(lg) + "/" + "/".join(h(p) for i in range(3) for _, _, p in e.trace(i))
    seen[key] = seen.get(key, 0) + 1
print("ragged R0 prefill:", len(seen), "distinct of", N, list(seen.values()), flush=True)
e.close()

# case 2: B=40 decode (test_c5[40-12])
cfg = O.ModelCfg(n_layers=4, d_model=256, n_heads=4, n_kv_heads=4, d_head=64, d_ff=688, mlp=1, act_mode=1,
                 weight_axis=2)
w = O.synth_weights(cfg, seed=21)
B, steps = 40, 12
e = Q.Engine(Q.Config(n_layers=4, d_model=256, n_heads=4, n_kv_heads=4, d_head=64, d_ff=688, mlp=1, act_mode=1),
             max_batch=B, max_tokens=8192, max_seq=4096, max_decode=steps + 1)
e.load_weights(w)
e.clear_recipe()
embs = np.concatenate([O.synth_embeddings(72, 256, seed=900 + i) for i in range(B)]).astype(np.float32)
dec = [O.synth_embeddings(B, 256, seed=1200 + s).astype(np.float32) for s in range(steps)]
seen = {}
for it in range(N):
    pre = e.prefill(embs, [52] * B, [20] * B)
    outs = [e.decode(dec[s]).copy() for s in range(steps)]
    key = h(pre) + "/" + "/".join(h(o) for o in outs)
    seen[key] = seen.get(key, 0) + 1
print("B=40 decode:", len(seen), "distinct of", N, list(seen.values()), flush=True)
if len(seen) > 1:
    ks = list(seen)
    print("keys", ks[:3])
