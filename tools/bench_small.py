"""Decode-sized quantizer timing: 64 chained K1 launches (RMSNorm + int4 quantizer) captured
in a CUDA graph, us per launch."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_17320_b200 as Q


def run(M, D, dtype, gain, mode, iters=64):
    x = torch.randn(M, D, dtype=dtype, device="cuda")
    g = torch.rand(D, dtype=torch.float32, device="cuda") if gain else None
    codes = torch.zeros(((M + 15) // 16 * 16, D // 2), dtype=torch.uint8, device="cuda")
    sc = torch.zeros(M, dtype=torch.float64, device="cuda")
    Q.rmsnorm_quant(x, g, D, mode, 0.5, codes, sc)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(gr, stream=s):
            for _ in range(iters):
                Q.rmsnorm_quant(x, g, D, mode, 0.5, codes, sc, stream=s.cuda_stream)
    gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    gr.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3


for M, D, dt, gain, name in [(8, 4096, torch.float64, True, "x norm"), (8, 11008, torch.float32, False, "mid"),
                             (8, 4096, torch.float32, False, "attn"), (1, 4096, torch.float64, True, "x norm M1")]:
    print(f"{name:10s} M={M} D={D}: dynamic {run(M, D, dt, gain, 1):6.2f} us  static {run(M, D, dt, gain, 0):6.2f} us",
          flush=True)
