import sys, time, numpy as np, torch
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_2604_17320_b200 as Q
L = int(sys.argv[1]) if len(sys.argv) > 1 else 32
cfg = Q.Config(n_layers=L, d_model=4096, n_heads=32, n_kv_heads=32, d_head=128, d_ff=11008, mlp=1, act_mode=1)
B, V, T, D = 8, 576, 64, int(sys.argv[2]) if len(sys.argv) > 2 else 32
e = Q.Engine(cfg, max_batch=B, max_tokens=B * (V + T), max_seq=V + T, max_decode=D + 4)
torch.manual_seed(0)
t0 = time.time()
for l in range(L):
    g = lambda *s: torch.randn(*s, device="cuda") * 0.02
    e.load_layer(l, g(4096, 4096), g(4096, 4096), g(4096, 4096), g(4096, 4096), g(4096, 11008), g(11008, 4096), g(4096, 11008))
e.load_head(torch.randn(4096, 4096, device="cuda") * 0.02)
torch.cuda.synchronize(); print("load", time.time() - t0, flush=True)
e.set_recipe([2], [0.3], v0=576)
emb = torch.randn(B * (V + T), 4096, device="cuda")
s = torch.cuda.Stream(); e.set_stream(s)
logits = torch.empty(B * (V + T), 4096, device="cuda")
demb = torch.randn(B, 4096, device="cuda"); dlog = torch.empty(B, 4096, device="cuda")
for it in range(int(sys.argv[3]) if len(sys.argv) > 3 else 3):
    ev0, ev1, ev2 = torch.cuda.Event(True), torch.cuda.Event(True), torch.cuda.Event(True)
    with torch.cuda.stream(s):
        ev0.record(s)
        e.prefill(emb, [V] * B, [T] * B, logits_out=logits)
        ev1.record(s)
        for k in range(D):
            e.decode(demb, logits_out=dlog)
        ev2.record(s)
    s.synchronize()
    print("prefill ms %.2f  decode ms/step %.3f" % (ev0.elapsed_time(ev1), ev1.elapsed_time(ev2) / D), flush=True)
print(e.info())
