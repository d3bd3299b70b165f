"""Experiment: decode of B sequences as ONE engine vs TWO engines of B/2 on two streams
(concurrent latency chains).  7B shape, random weights (2 copies in the 2-engine case)."""
import sys, time, torch
sys.path.insert(0, "/root/repo")
import paper_2604_17320_b200 as Q
L, B, V, T, D = 32, 8, 576, 64, 32
cfg = Q.Config(n_layers=L, d_model=4096, n_heads=32, n_kv_heads=32, d_head=128, d_ff=11008, mlp=1, act_mode=1)


def mk(bs):
    e = Q.Engine(cfg, max_batch=bs, max_tokens=bs * (V + T), max_seq=V + T, max_decode=D + 4)
    torch.manual_seed(0)
    for l in range(L):
        g = lambda *s: torch.randn(*s, device="cuda") * 0.02
        e.load_layer(l, g(4096, 4096), g(4096, 4096), g(4096, 4096), g(4096, 4096), g(4096, 11008), g(11008, 4096),
                     g(4096, 11008))
    e.load_head(torch.randn(4096, 4096, device="cuda") * 0.02)
    e.set_recipe([2], [0.3], v0=576)
    return e


def run(engines, bs):
    ss = [torch.cuda.Stream() for _ in engines]
    for e, s in zip(engines, ss):
        e.set_stream(s)
        emb = torch.randn(bs * (V + T), 4096, device="cuda")
        with torch.cuda.stream(s):
            e.prefill(emb, [V] * bs, [T] * bs)
    torch.cuda.synchronize()
    demb = torch.randn(bs, 4096, device="cuda")
    dl = [torch.empty(bs, 4096, device="cuda") for _ in engines]
    for _ in range(2):  # warm (graph capture)
        for e, s, o in zip(engines, ss, dl):
            with torch.cuda.stream(s):
                e.decode(demb, logits_out=o)
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(True); t1 = torch.cuda.Event(True)
    main = torch.cuda.current_stream()
    t0.record(main)
    for s in ss:
        s.wait_stream(main)
    for k in range(D - 4):
        for e, s, o in zip(engines, ss, dl):
            with torch.cuda.stream(s):
                e.decode(demb, logits_out=o)
    for s in ss:
        main.wait_stream(s)
    t1.record(main)
    torch.cuda.synchronize()
    return t0.elapsed_time(t1) / (D - 4)


one = mk(B)
print("1 engine  B=%d: %.3f ms/step" % (B, run([one], B)), flush=True)
del one
torch.cuda.empty_cache()
two = [mk(B // 2), mk(B // 2)]
print("2 engines B=%d each, 2 streams: %.3f ms/step" % (B // 2, run(two, B // 2)), flush=True)
print("1 of them alone B=%d: %.3f ms/step" % (B // 2, run([two[0]], B // 2)), flush=True)
