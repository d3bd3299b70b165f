"""Isolated int8-operand W4A4 GEMM timing (qt_w4a4_gemm_i8): the 2-SM pair kernel vs the
single-CTA one at the 7B prefill shapes; CUDA events, TOPS per shape."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2604_17320_b200 as Q


def run(M, N, K, epi, single, iters=20):
    a = (torch.randint(-7, 8, (M, K), dtype=torch.int8, device="cuda") * 16).contiguous()
    w = (torch.randint(-7, 8, ((N + 127) // 128 * 128, K), dtype=torch.int8, device="cuda") * 16).contiguous()
    sa = torch.rand(M, dtype=torch.float64, device="cuda")
    sw = torch.rand(w.shape[0], dtype=torch.float64, device="cuda")
    if epi == Q.EPI_RESADD:
        out = torch.zeros((M, N), dtype=torch.float64, device="cuda")
    elif epi == Q.EPI_SWIGLU:
        out = torch.zeros((M, N // 2), dtype=torch.float32, device="cuda")
    else:
        out = torch.zeros((M, N), dtype=torch.float32, device="cuda")
    for _ in range(3):
        Q.w4a4_gemm_i8(epi, a, sa, w, sw, M, N, K, out, single=single)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(iters):
        Q.w4a4_gemm_i8(epi, a, sa, w, sw, M, N, K, out, single=single)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    return ms, 2.0 * M * N * K / (ms / 1e3) / 1e12


for (M, N, K, epi, name) in [(1896, 12288, 4096, Q.EPI_STORE, "qkv"), (1896, 4096, 4096, Q.EPI_RESADD, "o"),
                             (1896, 22016, 4096, Q.EPI_SWIGLU, "gu"), (1896, 4096, 11008, Q.EPI_RESADD, "down"),
                             (5120, 12288, 4096, Q.EPI_STORE, "qkv5120"), (5120, 22016, 4096, Q.EPI_SWIGLU, "gu5120"),
                             (8192, 8192, 8192, Q.EPI_STORE, "8k")]:
    r = [run(M, N, K, epi, s) for s in (True, False)]
    print(f"{name:8s} M={M:5d} N={N:5d} K={K:5d}: single {r[0][0]*1e3:8.1f} us {r[0][1]:7.1f} TOPS | "
          f"pair {r[1][0]*1e3:8.1f} us {r[1][1]:7.1f} TOPS", flush=True)
