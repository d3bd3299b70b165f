"""Kernel-level parity at the headline 7B shapes (BASELINE.json configs[1] C2: d_head 128,
32 x 128 MHA, K = 4096 / 11008; configs[3] C4: 28 / 4 GQA) and at the tiny d_head 64 shape,
through the per-kernel C ABI (include/quota_b200.h), each kernel on inputs identical to the
checker's:

* K5 qt_kv_quant_append_i4 vs the unmodified reference rope_in_place + kv_quantize
  (model.cpp:156-168, quant.cpp:117-119): KV codes bit-exact, scales = fp32(reference).
* K7 qt_attn_prefill_i4kv vs the restatement's masked attention (model.cpp:272-292,366-391)
  on the GPU's own int4 rows.
* K3a/K3b qt_quota_score vs the unmodified reference compute_metrics (selector.cpp:19-68)
  on probabilities from the restatement -- north_star's 1e-3 relative.
* K6 qt_attn_decode_i4kv vs the restatement's decode attention (model.cpp:515-535).
* K4 qt_topk_compact vs the reference score_tokens + select_top_k (selector.cpp:70-136)
  and apply_pruning's row filter (selector.cpp:138-209).
* K2 decode GEMV at M <= 8 with K = 4096 and 11008 (the 7B down projection): int32 exact.
"""
import numpy as np
import pytest

import oracle as O
import paper_2604_17320_b200 as Q

pytestmark = pytest.mark.gpu

PAGE = 64


class Cache:
    """A paged int4 KV pool with a shuffled page table (exercises the indirection)."""

    def __init__(self, torch, B, Hkv, dh, max_len, seed=0):
        self.B, self.Hkv, self.dh = B, Hkv, dh
        self.page_bytes = 2 * Hkv * PAGE * (dh // 2 + 4)
        self.max_pages = (max_len + PAGE - 1) // PAGE
        n = B * self.max_pages
        perm = np.random.default_rng(seed).permutation(n).astype(np.int32)
        self.pt_host = perm.reshape(B, self.max_pages)
        self.pt = torch.from_numpy(self.pt_host.copy()).cuda()
        self.pool = torch.zeros(n * self.page_bytes, dtype=torch.uint8, device="cuda")

    def rows(self, b, n):
        """(K codes [n x Hkv*dh], K scales [n x Hkv] fp32, V codes, V scales) of seq b."""
        dh, Hkv = self.dh, self.Hkv
        pages = self.pool.cpu().numpy().reshape(-1, self.page_bytes)[self.pt_host[b, np.arange(n) // PAGE]]
        slot, idx = np.arange(n) % PAGE, np.arange(n)
        cb = Hkv * PAGE * (dh // 2)
        sc = np.ascontiguousarray(pages[:, 2 * cb:]).view(np.float32).reshape(n, 2, Hkv, PAGE)
        out = []
        for w in range(2):
            c = pages[:, w * cb:(w + 1) * cb].reshape(n, Hkv, PAGE, dh // 2)[idx, :, slot]
            out += [Q.unpack_i4(c, dh).reshape(n, Hkv * dh), sc[idx, w, :, slot]]
        return out


def _kv_append(torch, cache, qkv, ld, H, positions, tok_seq, tok_row):
    """qt_kv_quant_append_i4 on a torch fp32 qkv buffer (q heads RoPE'd in place)."""
    M = qkv.shape[0]
    rope = Q.rope_table(int(np.max(positions)) + 2, cache.dh)
    rope_d = torch.from_numpy(rope.reshape(-1).copy()).cuda()
    pos_d, ts_d, tr_d = (torch.from_numpy(np.asarray(a, np.int32)).cuda() for a in (positions, tok_seq, tok_row))
    Q.check(Q.lib().qt_kv_quant_append_i4(Q._ptr(qkv), ld, M, H, cache.Hkv, cache.dh, Q._ptr(pos_d), Q._ptr(ts_d),
                                          Q._ptr(tr_d), Q._ptr(rope_d), Q._ptr(cache.pt), cache.max_pages,
                                          Q._ptr(cache.pool), cache.page_bytes, None, None))
    torch.cuda.synchronize()


def _layout(lens, seed):
    """Packed tokens of sequences with lengths `lens`: strictly increasing original positions
    with gaps (pruned tokens keep their original position ids, model.cpp:156-168)."""
    rng = np.random.default_rng(seed)
    pos, ts, tr, off = [], [], [], [0]
    for b, n in enumerate(lens):
        p = np.sort(rng.choice(np.arange(n * 3), size=n, replace=False)).astype(np.int32)
        pos.append(p)
        ts += [b] * n
        tr += list(range(n))
        off.append(off[-1] + n)
    return pos, np.array(ts, np.int32), np.array(tr, np.int32), np.array(off, np.int32)


SHAPES = [  # (H, Hkv, dh, lens): C2 MHA 7B, C4 GQA 7B, the tiny GQA config; d_head 128 runs the
    # tcgen05 prefill attention (k_attn_prefill_ws), d_head 64 the mma.sync one
    (32, 32, 128, [640, 237]),
    (28, 4, 128, [300, 77]),
    (28, 4, 128, [700, 515, 77]),
    (4, 2, 64, [184, 45]),
]


@pytest.mark.parametrize("H,Hkv,dh,lens", SHAPES)
def test_kv_quant_append_bit_exact(torch_cuda, H, Hkv, dh, lens):
    torch = torch_cuda
    cache = Cache(torch, len(lens), Hkv, dh, max(lens), seed=1)
    pos, ts, tr, _ = _layout(lens, seed=2)
    M = sum(lens)
    n_qkv = (H + 2 * Hkv) * dh
    rng = np.random.default_rng(3)
    qkv_h = (rng.standard_normal((M, n_qkv)) * rng.uniform(0.1, 4.0, size=(1, n_qkv))).astype(np.float32)
    qkv = torch.from_numpy(qkv_h.copy()).cuda()
    _kv_append(torch, cache, qkv, n_qkv, H, np.concatenate(pos), ts, tr)
    q_gpu = qkv.cpu().numpy()
    o = 0
    for b, n in enumerate(lens):
        kc, ks, vc, vs = cache.rows(b, n)
        for r in range(n):
            m, p = o + r, int(pos[b][r])
            for h in range(Hkv):
                k = O.ref_rope(qkv_h[m, (H + h) * dh:(H + h + 1) * dh].astype(np.float64), p)
                v = qkv_h[m, (H + Hkv + h) * dh:(H + Hkv + h + 1) * dh].astype(np.float64)
                ck, sk = O.ref_kv_quantize(k[None])
                cv, sv = O.ref_kv_quantize(v[None])
                assert np.array_equal(kc[r, h * dh:(h + 1) * dh], ck[0]), (b, r, h)
                assert np.array_equal(vc[r, h * dh:(h + 1) * dh], cv[0]), (b, r, h)
                assert ks[r, h] == np.float32(sk[0]) and vs[r, h] == np.float32(sv[0])
            if r % 17 == 0:  # q heads RoPE'd in place: fp32 of the reference's fp64 rotation
                for h in range(0, H, 5):
                    qr = O.ref_rope(qkv_h[m, h * dh:(h + 1) * dh].astype(np.float64), p)
                    assert np.array_equal(q_gpu[m, h * dh:(h + 1) * dh], qr.astype(np.float32))
        o += n


def _prefill_setup(torch, H, Hkv, dh, lens, vis):
    cache = Cache(torch, len(lens), Hkv, dh, max(lens), seed=4)
    pos, ts, tr, off = _layout(lens, seed=5)
    M = sum(lens)
    n_qkv = (H + 2 * Hkv) * dh
    rng = np.random.default_rng(6)
    qkv = torch.from_numpy((rng.standard_normal((M, n_qkv)) * 0.8).astype(np.float32)).cuda()
    _kv_append(torch, cache, qkv, n_qkv, H, np.concatenate(pos), ts, tr)
    return cache, pos, off, qkv, n_qkv


def _port_attention(cache, qkv_h, pos, off, b, n, V, H, dh, want_probs=False):
    kc, ks, vc, vs = cache.rows(b, n)
    q = qkv_h[off[b]:off[b] + n, :H * dh].astype(np.float64)
    return O.port_masked_attention(q, kc, ks.astype(np.float64), vc, vs.astype(np.float64), pos[b], V, H,
                                   cache.Hkv, dh, want_probs)


@pytest.mark.parametrize("H,Hkv,dh,lens", SHAPES)
def test_prefill_attention_matches_restatement(torch_cuda, H, Hkv, dh, lens):
    """K7 (k_attn_prefill<d_head>) on the GPU's own int4 rows vs model.cpp:272-292 in fp64."""
    torch = torch_cuda
    O.Port.set_threads(8)
    vis = [int(0.9 * n) for n in lens]  # visual prefix, then text (mask model.cpp:35-44)
    cache, pos, off, qkv, n_qkv = _prefill_setup(torch, H, Hkv, dh, lens, vis)
    M = sum(lens)
    out = torch.zeros((M, H * dh), dtype=torch.float32, device="cuda")
    stats = torch.zeros((M, H, 2), dtype=torch.float32, device="cuda")
    Q.attn_prefill(qkv, n_qkv, H, Hkv, dh, off, vis, lens, cache.pool, cache.page_bytes, cache.pt, cache.max_pages,
                   out, stats)
    torch.cuda.synchronize()
    got, qkv_h = out.cpu().numpy(), qkv.cpu().numpy()
    for b, n in enumerate(lens):
        exp = _port_attention(cache, qkv_h, pos, off, b, n, vis[b], H, dh)
        err = np.abs(got[off[b]:off[b] + n] - exp).max() / np.abs(exp).max()
        assert err < 2e-6, (b, err)


@pytest.mark.parametrize("H,Hkv,dh,lens", SHAPES)
def test_quota_metrics_match_reference_compute_metrics(torch_cuda, H, Hkv, dh, lens):
    """K3a (k_attn_colsum<d_head>) + K3b (k_token_metrics) vs the unmodified reference
    compute_metrics on the same residual rows and the restatement's fp64 probabilities:
    north_star's 1e-3 relative, measured ~1e-6."""
    torch = torch_cuda
    O.Port.set_threads(8)
    vis = [int(0.9 * n) for n in lens]
    cache, pos, off, qkv, n_qkv = _prefill_setup(torch, H, Hkv, dh, lens, vis)
    M, d = sum(lens), H * dh
    out = torch.zeros((M, d), dtype=torch.float32, device="cuda")
    stats = torch.zeros((M, H, 2), dtype=torch.float32, device="cuda")
    Q.attn_prefill(qkv, n_qkv, H, Hkv, dh, off, vis, lens, cache.pool, cache.page_bytes, cache.pt, cache.max_pages,
                   out, stats)
    x_h = O.synth_embeddings(M, d, seed=7, outlier_frac=0.01)
    x = torch.from_numpy(x_h).cuda()
    met = Q.quota_score(x, qkv, n_qkv, H, Hkv, dh, off, vis, lens, cache.pool, cache.page_bytes, cache.pt,
                        cache.max_pages, stats, res_bits=4)
    torch.cuda.synchronize()
    met, qkv_h = met.cpu().numpy(), qkv.cpu().numpy()
    for b, n in enumerate(lens):
        V = vis[b]
        _, probs = _port_attention(cache, qkv_h, pos, off, b, n, V, H, dh, want_probs=True)
        xb = x_h[off[b]:off[b] + n]
        exp = O.ref_compute_metrics(xb[:V], xb[V:], probs[:, V:, :V], probs[:, :V, :V], res_bits=4)
        got = met[b, :, :V]
        np.testing.assert_allclose(got[0], exp[0], rtol=1e-12)   # mag: fp64 from the fp64 residual
        np.testing.assert_allclose(got[3], exp[3], rtol=1e-9)    # res: fp64 per-row fake quant
        for k in (1, 2):  # attention received: fp32 probabilities summed per head, fp64 over heads
            rel = np.abs(got[k] - exp[k]) / np.maximum(np.abs(exp[k]), 1e-30)
            assert rel.max() < 1e-3, (b, k, rel.max())
            assert np.median(rel) < 1e-5, (b, k, np.median(rel))


DECODE_SHAPES = [  # (H, Hkv, dh, lens): C2 (237 + t), C5 long context, C4 GQA, tiny
    (32, 32, 128, [237, 238, 300, 365, 1, 64, 129, 191]),
    (32, 32, 128, [2285, 1000]),
    (28, 4, 128, [300, 1344, 77, 64]),
    (4, 2, 64, [84, 150, 1, 63]),
    # enough work units for the persistent, double-buffered grid (units > 2 waves of CTAs)
    (32, 32, 128, [300, 64, 1, 129, 511, 257] * 8),
    (28, 4, 128, [700, 65, 1290, 3] * 16),
]


@pytest.mark.parametrize("H,Hkv,dh,lens", DECODE_SHAPES)
def test_decode_attention_matches_restatement(torch_cuda, H, Hkv, dh, lens):
    """K6 decode attention (every kv_len, including 1 row and exact page multiples) vs the
    reference decode loop model.cpp:515-535 on the same int4 rows."""
    torch = torch_cuda
    B = len(lens)
    cache = Cache(torch, B, Hkv, dh, max(lens), seed=8)
    pos, ts, tr, off = _layout(lens, seed=9)
    n_qkv = (H + 2 * Hkv) * dh
    rng = np.random.default_rng(10)
    qkv = torch.from_numpy((rng.standard_normal((sum(lens), n_qkv)) * 0.8).astype(np.float32)).cuda()
    _kv_append(torch, cache, qkv, n_qkv, H, np.concatenate(pos), ts, tr)
    q_h = (rng.standard_normal((B, H * dh)) * 1.5).astype(np.float32)
    q = torch.from_numpy(q_h).cuda()
    out = torch.zeros((B, H * dh), dtype=torch.float32, device="cuda")
    Q.attn_decode(q, H * dh, H, Hkv, dh, lens, cache.pool, cache.page_bytes, cache.pt, cache.max_pages, out)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    for b, n in enumerate(lens):
        kc, ks, vc, vs = cache.rows(b, n)
        exp = O.port_decode_attention(q_h[b].astype(np.float64), kc, ks.astype(np.float64), vc,
                                      vs.astype(np.float64), H, Hkv, dh)
        err = np.abs(got[b] - exp).max() / np.abs(exp).max()
        assert err < 2e-6, (b, n, err)


@pytest.mark.parametrize("B,V,T", [(3, 576, 64), (2, 2880, 128)])
def test_topk_compact_matches_reference(torch_cuda, B, V, T):
    """K3c + K4 + compaction: the reference score_tokens / select_top_k on the same metrics,
    then x, positions and the layer's K/V rows filtered like apply_pruning."""
    torch = torch_cuda
    rng = np.random.default_rng(11)
    d, Hkv, dh = 256, 2, 64
    vis = [V - 7 * b for b in range(B)]
    txt = [T] * B
    lens = [v + t for v, t in zip(vis, txt)]
    budget = [int(np.ceil(0.3 * v)) for v in vis]
    vs = (V + 63) // 64 * 64
    met_h = np.zeros((B, 4, vs))
    for b in range(B):
        met_h[b, :, :vis[b]] = rng.gamma(2.0, 1.0, size=(4, vis[b]))
        met_h[b, 1, :8] = met_h[b, 1, 8]  # ties inside a metric
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    x_h = rng.standard_normal((off[-1], d))
    pos_h = np.concatenate([np.arange(n, dtype=np.int32) * 2 for n in lens])
    cache = Cache(torch, B, Hkv, dh, max(lens), seed=12)
    n_qkv = (4 + 2 * Hkv) * dh
    qkv = torch.from_numpy((rng.standard_normal((off[-1], n_qkv))).astype(np.float32)).cuda()
    ts = np.concatenate([[b] * n for b, n in enumerate(lens)]).astype(np.int32)
    tr = np.concatenate([np.arange(n) for n in lens]).astype(np.int32)
    _kv_append(torch, cache, qkv, n_qkv, 4, pos_h, ts, tr)
    before = [cache.rows(b, lens[b]) for b in range(B)]
    w = (0.25, 0.45, 0.10, 0.20)
    x_out, pos_out, kept, noff = Q.topk_compact(torch.from_numpy(met_h).cuda(), vis, txt, budget, w, off,
                                                torch.from_numpy(x_h).cuda(), torch.from_numpy(pos_h).cuda(),
                                                cache.pool, cache.page_bytes, cache.pt, cache.max_pages, Hkv, dh)
    x_out, pos_out = x_out.cpu().numpy(), pos_out.cpu().numpy()
    for b in range(B):
        fused = _ref_fused(met_h[b, :, :vis[b]], w)
        exp_slots = O.ref_select_top_k(fused, budget[b])
        assert np.array_equal(kept[b], exp_slots)
        keep = np.concatenate([exp_slots, np.arange(vis[b], lens[b])])
        assert np.array_equal(x_out[noff[b]:noff[b + 1]], x_h[off[b] + keep])
        assert np.array_equal(pos_out[noff[b]:noff[b + 1]], pos_h[off[b] + keep])
        after = cache.rows(b, len(keep))
        for k in range(4):
            assert np.array_equal(after[k], before[b][k][keep]), (b, k)


def _ref_fused(m4, w):
    """robust_normalize + fuse_scores (selector.cpp:70-104): the reference normalisation, and
    the fusion's left-to-right fp64 sum (numpy evaluates it in the same order, no FMA)."""
    norm = [O.ref_robust_normalize(m4[k]) for k in range(4)]
    return w[0] * norm[0] + w[1] * norm[1] + w[2] * norm[2] + w[3] * norm[3]


@pytest.mark.parametrize("M", [1, 5, 8, 12, 16])
@pytest.mark.parametrize("K,N,epi", [(4096, 4096, Q.EPI_RESADD), (11008, 4096, Q.EPI_RESADD),
                                     (4096, 12288, Q.EPI_STORE), (4096, 22016, Q.EPI_SWIGLU)])
def test_decode_gemv_7b_shapes_int32_exact(torch_cuda, M, K, N, epi):
    """The decode GEMV (k_gemv_reg) at the C2 shapes: register-resident activations for
    K = 4096, smem-staged for the K = 11008 down projection; int32 accumulators exact,
    epilogue within fp64 rounding."""
    torch = torch_cuda
    from tests.test_kernels_gpu import _tiled
    rng = np.random.default_rng(M * 7 + K + N)
    a = rng.integers(-7, 8, size=(M, K))
    w = rng.integers(-7, 8, size=(N, K))
    sa = rng.uniform(0.01, 0.5, M)
    sw = rng.uniform(0.001, 0.01, N)
    acc_exp = a.astype(np.int64) @ w.T.astype(np.int64)
    y = acc_exp * sa[:, None] * sw[None, :]
    if epi == Q.EPI_RESADD:
        base = rng.standard_normal((M, N))
        out = torch.from_numpy(base.copy()).cuda()
        exp, tol = base + y, dict(rtol=1e-14, atol=1e-14)
    elif epi == Q.EPI_SWIGLU:
        out = torch.zeros((M, N // 2), dtype=torch.float32, device="cuda")
        g, u = y[:, 0::2], y[:, 1::2]
        exp, tol = g / (1.0 + np.exp(-g)) * u, dict(rtol=2e-7, atol=1e-7)
    else:
        out = torch.zeros((M, N), dtype=torch.float32, device="cuda")
        exp, tol = y, dict(rtol=2e-7, atol=1e-7)
    acc = torch.zeros((M, N), dtype=torch.int32, device="cuda")
    Q.w4a4_gemm(epi, torch.from_numpy(_tiled(a)).cuda(), torch.from_numpy(sa).cuda(),
                torch.from_numpy(_tiled(w, 128)).cuda(), torch.from_numpy(sw).cuda(), M, N, K, out, acc, impl=0)
    torch.cuda.synchronize()
    assert np.array_equal(acc.cpu().numpy(), acc_exp)
    np.testing.assert_allclose(out.cpu().numpy(), exp, **tol)


def test_unpack_codes_roundtrip(torch_cuda):
    torch = torch_cuda
    from tests.test_kernels_gpu import _tiled
    rng = np.random.default_rng(13)
    c = rng.integers(-7, 8, size=(37, 640))
    t = torch.from_numpy(_tiled(c)).cuda()
    got = Q.unpack_codes(t, 37, 640)
    torch.cuda.synchronize()
    assert np.array_equal(got.cpu().numpy(), c)
