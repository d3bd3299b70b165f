"""Per-class decode chain times (qt_engine_profile_chain) on the 7B shape, B = 8."""
import sys, torch
sys.path.insert(0, "/root/repo")
import paper_2604_17320_b200 as Q
L, B, V, T, D = 32, 8, 576, 64, 16
cfg = Q.Config(n_layers=L, d_model=4096, n_heads=32, n_kv_heads=32, d_head=128, d_ff=11008, mlp=1, act_mode=1)
e = Q.Engine(cfg, max_batch=B, max_tokens=B * (V + T), max_seq=V + T, max_decode=D + 4)
torch.manual_seed(0)
for l in range(L):
    g = lambda *s: torch.randn(*s, device="cuda") * 0.02
    e.load_layer(l, g(4096, 4096), g(4096, 4096), g(4096, 4096), g(4096, 4096), g(4096, 11008), g(11008, 4096),
                 g(4096, 11008))
e.load_head(torch.randn(4096, 4096, device="cuda") * 0.02)
e.set_recipe([2], [0.3], v0=576)
s = torch.cuda.Stream(); e.set_stream(s)
with torch.cuda.stream(s):
    e.prefill(torch.randn(B * (V + T), 4096, device="cuda"), [V] * B, [T] * B)
    for _ in range(4):
        e.decode(torch.randn(B, 4096, device="cuda"))
s.synchronize()
for rep in range(2):
    r = {k: e.profile_chain(m, 30) for k, m in [("full", 0), ("gemm", 14), ("attention", 13), ("quant", 11),
                                                 ("kv", 7), ("none", 15)]}
    print(" ".join(f"{k} {v * 1e3:7.1f}us" for k, v in r.items()), flush=True)
