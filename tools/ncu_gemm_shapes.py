"""One launch per 7B prefill GEMM shape of the single-CTA int8 kernel (for ncu --set full)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2604_17320_b200 as Q

for (M, N, K, epi) in [(1896, 12288, 4096, Q.EPI_STORE), (1896, 4096, 4096, Q.EPI_RESADD),
                       (1896, 22016, 4096, Q.EPI_SWIGLU), (1896, 4096, 11008, Q.EPI_RESADD)]:
    a = (torch.randint(-7, 8, (M, K), dtype=torch.int8, device="cuda") * 16).contiguous()
    w = (torch.randint(-7, 8, ((N + 127) // 128 * 128, K), dtype=torch.int8, device="cuda") * 16).contiguous()
    sa = torch.rand(M, dtype=torch.float64, device="cuda")
    sw = torch.rand(w.shape[0], dtype=torch.float64, device="cuda")
    out = (torch.zeros((M, N), dtype=torch.float64, device="cuda") if epi == Q.EPI_RESADD else
           torch.zeros((M, N // 2 if epi == Q.EPI_SWIGLU else N), dtype=torch.float32, device="cuda"))
    Q.w4a4_gemm_i8(epi, a, sa, w, sw, M, N, K, out, single=True)
    torch.cuda.synchronize()
print("ok")
