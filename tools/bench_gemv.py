"""Decode GEMV (M = 8 tokens) timing through the C ABI: back-to-back launches on one weight
matrix (L2-warm) and rotating over copies larger than L2 (HBM-cold); CUDA events."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_17320_b200 as Q

M = int(sys.argv[1]) if len(sys.argv) > 1 else 8


def run(N, K, epi, copies, iters=64, impl=0):
    rows = 16
    a = (torch.randint(0, 256, (rows, K // 2), dtype=torch.uint8, device="cuda") & 0x77)
    ws = [(torch.randint(0, 256, ((N + 127) // 128 * 128, K // 2), dtype=torch.uint8, device="cuda") & 0x77)
          for _ in range(copies)]
    sa = torch.rand(M, dtype=torch.float64, device="cuda")
    sw = torch.rand(ws[0].shape[0], dtype=torch.float64, device="cuda")
    if epi == Q.EPI_RESADD:
        out = torch.zeros((M, N), dtype=torch.float64, device="cuda")
    elif epi == Q.EPI_SWIGLU:
        out = torch.zeros((M, N // 2), dtype=torch.float32, device="cuda")
    else:
        out = torch.zeros((M, N), dtype=torch.float32, device="cuda")
    for i in range(4):
        Q.w4a4_gemm(epi, a, sa, ws[i % copies], sw, M, N, K, out, impl=impl)
    torch.cuda.synchronize()
    # captured in a CUDA graph: the launches replay without host overhead (as the decode graph)
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for i in range(iters):
                Q.w4a4_gemm(epi, a, sa, ws[i % copies], sw, M, N, K, out, impl=impl, stream=s.cuda_stream)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / iters * 1e3
    return us, ws[0].numel() / (us * 1e-6) / 1e9


for N, K, epi, name in [(12288, 4096, Q.EPI_STORE, "qkv"), (4096, 4096, Q.EPI_RESADD, "o"),
                        (22016, 4096, Q.EPI_SWIGLU, "gu"), (4096, 11008, Q.EPI_RESADD, "down")]:
    wb = (N + 127) // 128 * 128 * K // 2
    cold = max(2, int(400e6 // wb) + 1)
    for impl in (0,):
        uw, gw = run(N, K, epi, 1, impl=impl)
        uc, gc = run(N, K, epi, cold, impl=impl)
        print(f"{name:5s} M={M} N={N} K={K} {wb/1e6:6.1f} MB  warm {uw:7.2f} us "
              f"{gw:7.0f} GB/s   cold {uc:7.2f} us {gc:7.0f} GB/s", flush=True)
