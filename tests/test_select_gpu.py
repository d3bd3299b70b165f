"""K3c (robust normalisation + fusion) and K4 (deterministic budgeted top-k) on
the B200 against the unmodified reference (score_tokens / select_top_k,
selector.cpp:70-136) GIVEN IDENTICAL METRICS: normalised metrics and fused
scores bit-exact (fp64, no contraction), retained slots bit-exact, including
the ties the P5/P95 clipping creates and the -0.0 / +0.0 case."""
import json
import os

import numpy as np
import pytest

import oracle as O
import paper_2604_17320_b200 as Q

pytestmark = pytest.mark.gpu
KATS = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "kats.json")))


def _pad_metrics(torch, rows, vstride):
    m = np.zeros((len(rows), 4, vstride))
    for b, r in enumerate(rows):
        m[b, :, :r.shape[1]] = r
    return torch.from_numpy(m).cuda()


def test_topk_known_answers(torch_cuda):
    torch = torch_cuda
    cases = KATS["topk"]
    vs = max(len(c["scores"]) for c in cases)
    rows = [np.vstack([np.array(c["scores"])] + [np.zeros(len(c["scores"]))] * 3) for c in cases]
    slots, _, _ = Q.quota_topk(_pad_metrics(torch, rows, vs), [len(c["scores"]) for c in cases],
                               [c["k"] for c in cases], None)
    for s, c in zip(slots, cases):
        assert s.tolist() == c["slots"], c


def _record(rng, n, d, H, T, tie_levels=None):
    vis = rng.normal(0, 1, size=(n, d))
    vis[:, rng.integers(0, d)] *= 20.0
    inter = rng.dirichlet(np.ones(n), size=(H, T))
    intra = rng.dirichlet(np.ones(n), size=(H, n))
    if tie_levels:
        inter = np.round(inter * tie_levels) / tie_levels
    return vis, inter, intra


@pytest.mark.parametrize("n,H,T,k", [(50, 2, 5, 17), (144, 4, 40, 44), (576, 32, 64, 173), (2880, 8, 16, 720),
                                     (7, 1, 1, 7), (1, 2, 3, 1), (300, 4, 10, 299)])
def test_scores_and_topk_bit_exact_vs_reference(torch_cuda, n, H, T, k):
    torch = torch_cuda
    rng = np.random.default_rng(n * 31 + k)
    rows, refs = [], []
    B = 3
    for b in range(B):
        vis, inter, intra = _record(rng, n, 16, H, T, tie_levels=50 if b == 1 else None)
        m, nn, f = O.ref_score_tokens(vis, inter, intra)
        rows.append(m)
        refs.append((nn, f, O.ref_select_top_k(f, k)))
    w = (0.25, 0.45, 0.10, 0.20)
    slots, fused, norm = Q.quota_topk(_pad_metrics(torch, rows, n), [n] * B, [k] * B, w)
    fused, norm = fused.cpu().numpy(), norm.cpu().numpy()
    for b, (nn, f, sl) in enumerate(refs):
        assert np.array_equal(norm[b, :, :n], nn)
        assert np.array_equal(fused[b, :n], f)
        assert np.array_equal(slots[b], sl)


def test_ragged_batch_topk(torch_cuda):
    """Per-sequence V and budget (ragged C4 batches): each row equals its own reference call."""
    torch = torch_cuda
    rng = np.random.default_rng(7)
    Vs = [256, 1280, 700, 33]
    Ks = [O.ref_compute_budget(0.3, v) for v in Vs]
    rows, exp = [], []
    for v, kk in zip(Vs, Ks):
        s = rng.normal(0, 1, size=v)
        s[rng.integers(0, v, size=v // 4)] = 0.5  # heavy ties
        rows.append(np.vstack([s, np.zeros((3, v))]))
        exp.append(O.ref_select_top_k(s, kk))
    slots, _, _ = Q.quota_topk(_pad_metrics(torch, rows, max(Vs)), Vs, Ks, None)
    for s, e in zip(slots, exp):
        assert np.array_equal(s, e)
