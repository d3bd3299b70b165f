import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2604_17320_b200 as Q
from tests.test_kernels_gpu import _tiled
for (M, N, K) in [(128, 256, 128), (128, 256, 512), (40, 640, 1024), (1000, 640, 1024)]:
    rng = np.random.default_rng(M + N)
    a = rng.integers(-7, 8, size=(M, K)); w = rng.integers(-7, 8, size=(N, K))
    sa = np.ones(M); sw = np.ones(N)
    out = torch.zeros((M, N), dtype=torch.float32, device="cuda")
    acc = torch.zeros((M, N), dtype=torch.int32, device="cuda")
    Q.w4a4_gemm(0, torch.from_numpy(_tiled(a)).cuda(), torch.from_numpy(sa).cuda(), torch.from_numpy(_tiled(w)).cuda(),
                torch.from_numpy(sw).cuda(), M, N, K, out, acc, impl=1)
    torch.cuda.synchronize()
    exp = a.astype(np.int64) @ w.T.astype(np.int64)
    got = acc.cpu().numpy()
    bad = np.argwhere(got != exp)
    print(M, N, K, "mismatches", len(bad), "of", exp.size, bad[:5].tolist(), got[0, :4].tolist(), exp[0, :4].tolist(), flush=True)
