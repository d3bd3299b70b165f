"""Megakernel decode vs the unfused graph path: parity on the tiny configs, then 7B-shape speed."""
import os, subprocess, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

def tiny(mk, mlp=1, act_mode=1, hkv=2, B=3):
    import oracle as O
    import paper_2604_17320_b200 as Q
    cfg = O.ModelCfg(n_layers=4, d_model=256, n_heads=4, n_kv_heads=hkv, d_head=64, d_ff=688 if mlp else 1024,
                     mlp=mlp, act_mode=act_mode, weight_axis=2)
    w = O.synth_weights(cfg, seed=21)
    e = Q.Engine(Q.Config(n_layers=4, d_model=256, n_heads=4, n_kv_heads=hkv, d_head=64, d_ff=cfg.d_ff, mlp=mlp,
                          act_mode=act_mode), max_batch=8, max_tokens=4096, max_seq=1024, max_decode=16)
    e.load_weights(w)
    if act_mode == 0:
        e.set_act_scales(np.full(17, 0.05))
    e.set_recipe([0, 1, 2, 3], [1.0, 0.5, 0.3, 0.3], v0=144)
    vis, txt = [144] * B, [40 - 5 * i for i in range(B)]
    emb = np.concatenate([O.synth_embeddings(v + t, 256, seed=13 + i) for i, (v, t) in enumerate(zip(vis, txt))])
    lg = e.prefill(emb.astype(np.float32), vis, txt)
    outs = []
    for s in range(6):
        de = O.synth_embeddings(B, 256, seed=700 + s).astype(np.float32)
        outs.append(e.decode(de).copy())
    kv = [e.kv(l, b, h, w_)[0] for l in range(4) for b in range(B) for h in range(hkv) for w_ in (0, 1)]
    return lg, outs, kv

if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "tiny":
        for kw in [dict(), dict(mlp=0, act_mode=0, hkv=4, B=1), dict(B=8, hkv=4)]:
            r = {}
            for mk in (0, 1):
                out = subprocess.run([sys.executable, __file__, "one", str(mk), json.dumps(kw)], capture_output=True,
                                     text=True, env=dict(os.environ, QT_DECODE_MK=str(mk)), timeout=300)
                print(out.stderr[-2000:])
                r[mk] = np.load(f"/tmp/mk{mk}.npz")
            print(kw, "prefill same:", np.array_equal(r[0]["lg"], r[1]["lg"]),
                  "decode max|d|:", float(np.abs(r[0]["dec"] - r[1]["dec"]).max()),
                  "kv codes equal:", np.array_equal(r[0]["kv"], r[1]["kv"]))
    elif mode == "one":
        mk, kw = int(sys.argv[2]), json.loads(sys.argv[3])
        lg, outs, kv = tiny(mk, **kw)
        np.savez(f"/tmp/mk{mk}.npz", lg=lg, dec=np.stack(outs), kv=np.concatenate([k.ravel() for k in kv]))
