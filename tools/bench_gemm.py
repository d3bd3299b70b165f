"""Isolated W4A4 GEMM timing through the C ABI (qt_w4a4_gemm), CUDA events, TOPS per shape."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2604_17320_b200 as Q

def run(M, N, K, epi, impl=1, iters=20):
    rows = (M + 15) // 16 * 16
    a = torch.randint(0, 256, (rows, K // 2), dtype=torch.uint8, device="cuda")
    w = torch.randint(0, 256, ((N + 127) // 128 * 128, K // 2), dtype=torch.uint8, device="cuda")
    a &= 0x77; w &= 0x77  # codes in [0, 7]
    sa = torch.rand(M, dtype=torch.float64, device="cuda")
    sw = torch.rand(w.shape[0], dtype=torch.float64, device="cuda")
    if epi == Q.EPI_RESADD:
        out = torch.zeros((M, N), dtype=torch.float64, device="cuda")
    elif epi == Q.EPI_SWIGLU:
        out = torch.zeros((M, N // 2), dtype=torch.float32, device="cuda")
    else:
        out = torch.zeros((M, N), dtype=torch.float32, device="cuda")
    for _ in range(3):
        Q.w4a4_gemm(epi, a, sa, w, sw, M, N, K, out, impl=impl)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(iters):
        Q.w4a4_gemm(epi, a, sa, w, sw, M, N, K, out, impl=impl)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    return ms, 2.0 * M * N * K / (ms / 1e3) / 1e12

for (M, N, K, epi, name) in [(1896, 4096, 4096, Q.EPI_STORE, "o_store"), (1896, 4096, 11008, Q.EPI_STORE, "dn_store"),
                             (1896, 12288, 4096, Q.EPI_STORE, "qkv"), (1896, 4096, 4096, Q.EPI_RESADD, "o"),
                             (1896, 22016, 4096, Q.EPI_SWIGLU, "gu"), (1896, 4096, 11008, Q.EPI_RESADD, "down"),
                             (5120, 12288, 4096, Q.EPI_STORE, "qkv5120"), (8192, 8192, 8192, Q.EPI_STORE, "8k")]:
    ms, tops = run(M, N, K, epi)
    print(f"{name:8s} M={M} N={N} K={K}: {ms*1e3:8.1f} us  {tops:7.1f} TOPS", flush=True)
