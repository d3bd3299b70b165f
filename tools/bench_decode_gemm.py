"""Decode-batch GEMM timing (M = 16..256 tokens) per implementation, HBM-cold (rotating weight
copies larger than L2), launches replayed from a CUDA graph; CUDA events.
  gemv  impl 0: mma.sync weight-streaming GEMV / GEMM (int4 tiles)
  pk    impl 1: packed-int4 tcgen05 GEMM (converter warps), no split-K
  pks   impl 2: the same with split-K (fixed-order int32 reduction)
  i8    qt_w4a4_gemm_i8 single-CTA int8-operand TMA kernel (int8 weight copy: 2x the bytes)
  i8a   the same with the automatic split-K choice (workspace given)
  i8kN  the same with N k slices forced
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2604_17320_b200 as Q

MS = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [64, 128, 256]
IMPLS = sys.argv[2].split(",") if len(sys.argv) > 2 else ["gemv", "pk", "pks", "i8"]


def out_for(epi, M, N):
    if epi == Q.EPI_RESADD:
        return torch.zeros((M, N), dtype=torch.float64, device="cuda")
    if epi == Q.EPI_SWIGLU:
        return torch.zeros((M, N // 2), dtype=torch.float32, device="cuda")
    return torch.zeros((M, N), dtype=torch.float32, device="cuda")


def run(M, N, K, epi, impl, iters=24):
    npad = (N + 127) // 128 * 128
    i8 = impl.startswith("i8")
    wbytes = npad * K // (1 if i8 else 2)
    copies = max(2, int(300e6 // wbytes) + 1)
    rows = max(16, (M + 127) // 128 * 128)
    ks, wsp = 0, None
    if impl == "i8a":
        nb = Q.lib().qt_w4a4_gemm_i8_workspace(M, N, K)
        wsp = torch.empty(max(nb // 4, 1), dtype=torch.int32, device="cuda") if nb > 0 else None
    elif impl.startswith("i8k"):
        ks = int(impl[3:])
        wsp = torch.empty(ks * M * N, dtype=torch.int32, device="cuda")
    if i8:
        a = (torch.randint(-7, 8, (M, K), dtype=torch.int8, device="cuda") * 16).contiguous()
        ws = [(torch.randint(-7, 8, (npad, K), dtype=torch.int8, device="cuda") * 16).contiguous()
              for _ in range(copies)]
    else:
        a = torch.randint(0, 256, (rows, K // 2), dtype=torch.uint8, device="cuda") & 0x77
        ws = [torch.randint(0, 256, (npad, K // 2), dtype=torch.uint8, device="cuda") & 0x77 for _ in range(copies)]
    sa = torch.rand(M, dtype=torch.float64, device="cuda")
    sw = torch.rand(npad, dtype=torch.float64, device="cuda")
    out = out_for(epi, M, N)

    def call(i, st=0):
        if i8:
            Q.w4a4_gemm_i8(epi, a, sa, ws[i % copies], sw, M, N, K, out, workspace=wsp, single=True, stream=st,
                           ksplit=ks)
        else:
            Q.w4a4_gemm(epi, a, sa, ws[i % copies], sw, M, N, K, out,
                        impl={"gemv": 0, "pk": 1, "pks": 2}[impl], stream=st)

    for i in range(3):
        call(i)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for i in range(iters):
                call(i, s.cuda_stream)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / iters * 1e3
    return us, wbytes / (us * 1e-6) / 1e9, 2.0 * M * N * K / (us * 1e-6) / 1e12


for M in MS:
    for N, K, epi, name in [(12288, 4096, Q.EPI_STORE, "qkv"), (4096, 4096, Q.EPI_RESADD, "o"),
                            (22016, 4096, Q.EPI_SWIGLU, "gu"), (4096, 11008, Q.EPI_RESADD, "down")]:
        row = []
        for impl in IMPLS:
            if impl == "gemv" and M > 64:
                continue
            try:
                us, gbs, tops = run(M, N, K, epi, impl)
                row.append(f"{impl} {us:7.1f}us {gbs:5.0f}GB/s {tops:5.0f}T")
            except Exception as e:  # noqa: BLE001 -- report and continue the sweep
                row.append(f"{impl} ERR {str(e)[:60]}")
        print(f"M={M:3d} {name:5s} | " + " | ".join(row), flush=True)
