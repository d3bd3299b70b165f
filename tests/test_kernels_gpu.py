"""Kernel-level parity on the B200: each CUDA kernel against the reference
functions (oracle/_ref, the unmodified reference library) on identical inputs.
Integer outputs (int4 codes, int32 accumulators, KV codes) must be bit-exact."""
import numpy as np
import pytest

import oracle as O
import paper_2604_17320_b200 as Q

pytestmark = pytest.mark.gpu


def _ref():
    return O.ref_lib()


def ref_rms(x, g):
    lib = _ref()
    out = np.empty_like(x)
    O._check(lib.qref_rms_norm_rows(O._d(x), x.shape[0], x.shape[1], O._d(g), O._d(out)), lib, "qref")
    return out


def ref_quant_fit(x, axis, bits=4):
    lib = _ref()
    rows, cols = x.shape
    n = {0: 1, 1: rows, 2: cols}[axis]
    sc = np.empty(n)
    codes = np.empty(x.size, dtype=np.int8)
    O._check(lib.qref_quantize_fit(O._d(x), rows, cols, bits, axis, O._d(sc), O._b(codes)), lib, "qref")
    return codes.reshape(x.shape), sc


def ref_quant_with(x, scale):
    lib = _ref()
    rows, cols = x.shape
    s = np.array([scale], dtype=np.float64)
    codes = np.empty(x.size, dtype=np.int8)
    O._check(lib.qref_quantize_with(O._d(x), rows, cols, 4, 0, O._d(s), 1, O._b(codes), None), lib, "qref")
    return codes.reshape(x.shape)


def _x(M, D, seed, outlier=0.02):
    return O.synth_embeddings(M, D, seed, outlier_frac=outlier).astype(np.float32)


@pytest.mark.parametrize("M,D", [(1, 256), (37, 256), (64, 4096), (5, 688)])
@pytest.mark.parametrize("mode", [0, 1])
def test_rmsnorm_quant_codes_bit_exact(torch_cuda, M, D, mode):
    torch = torch_cuda
    x = _x(M, D, seed=M * 7 + D)
    g = (1.0 + 0.1 * np.random.default_rng(3).standard_normal(D)).astype(np.float32)
    d_pad = (D + 127) // 128 * 128
    xd = torch.from_numpy(x).cuda()
    gd = torch.from_numpy(g).cuda()
    normed_ref = ref_rms(x.astype(np.float64), g.astype(np.float64))
    if mode == 0:
        s_static = float(np.abs(normed_ref).max() / 7.0 * 0.8)  # some clipping
        exp_codes = ref_quant_with(normed_ref, s_static)
        exp_scales = np.full(M, s_static)
    else:
        exp_codes, exp_scales = ref_quant_fit(normed_ref, 1)
        s_static = 0.0
    codes, scales = Q.rmsnorm_quant(xd.double() if M % 2 else xd, gd, d_pad, mode, s_static)
    torch.cuda.synchronize()
    got = Q.unpack_i4(Q.untile_w4(codes.cpu().numpy(), codes.shape[0], d_pad // 2), d_pad)[:M]
    assert np.array_equal(got[:, :D], exp_codes)
    assert np.all(got[:, D:] == 0)
    # the RMS sum is a parallel fp64 reduction: scales agree to a few ulp
    np.testing.assert_allclose(scales.cpu().numpy(), exp_scales, rtol=1e-14)


def test_norm_free_site_quant(torch_cuda):
    """attn_out / mlp_mid sites: no RMSNorm, per-token fake_quant_per_row (quant.cpp:108-110)."""
    torch = torch_cuda
    x = _x(9, 1024, seed=5)
    codes, scales = Q.rmsnorm_quant(torch.from_numpy(x).cuda(), None, 1024, 1)
    exp_codes, exp_scales = ref_quant_fit(x.astype(np.float64), 1)
    assert np.array_equal(Q.unpack_i4(Q.untile_w4(codes.cpu().numpy(), codes.shape[0], 512), 1024)[:9], exp_codes)
    assert np.array_equal(scales.cpu().numpy(), exp_scales)


def test_weight_quant_per_output_channel(torch_cuda):
    torch = torch_cuda
    K, N = 300, 200
    w = (np.random.default_rng(1).standard_normal((K, N)) * 0.02).astype(np.float32)
    w[:, 7] = 0.0  # all-zero group -> scale 1, codes 0 (quant.cpp:66)
    k_pad, n_pad = 384, 256
    codes, scales = Q.quant_weight(torch.from_numpy(w).cuda(), k_pad, n_pad)
    exp_codes, exp_scales = ref_quant_fit(w.astype(np.float64), 2)
    got = Q.unpack_i4(Q.untile_w4(codes.cpu().numpy(), n_pad, k_pad // 2), k_pad)
    assert np.array_equal(got[:N, :K], exp_codes.T)
    assert np.all(got[:N, K:] == 0)
    assert np.array_equal(scales.cpu().numpy()[:N], exp_scales)
    assert scales.cpu().numpy()[7] == 1.0


def _pack(c):
    c = np.asarray(c, dtype=np.int16) & 0xF
    return (c[..., 0::2] | (c[..., 1::2] << 4)).astype(np.uint8)


def _tiled(c, pad=16):
    """int4 codes [rows x K] -> packed + tiled (rows zero-padded to `pad`), the engine's code layout."""
    p = _pack(c)
    rows = (p.shape[0] + pad - 1) // pad * pad
    out = np.zeros((rows, p.shape[1]), dtype=np.uint8)
    out[:p.shape[0]] = p
    return Q.tile_w4(out)


@pytest.mark.parametrize("M,impl", [(1, 0), (3, 0), (8, 0), (13, 0), (16, 0), (40, 0), (128, 0), (300, 0),
                                    (40, 1), (128, 1), (300, 1), (1000, 1), (40, 2), (64, 2), (200, 2)])
def test_w4a4_gemm_int32_exact(torch_cuda, M, impl):
    """impl 0: mma.sync GEMM/GEMV; impl 1: tcgen05 kind::i8 GEMM (TMEM accumulators);
    impl 2: tcgen05 with split-K (int32 partials reduced in fixed order)."""
    torch = torch_cuda
    rng = np.random.default_rng(M)
    K, N = (512, 384) if impl == 0 else ((1024, 640) if impl == 1 else (2048, 520))
    a = rng.integers(-7, 8, size=(M, K))
    w = rng.integers(-7, 8, size=(N, K))
    sa = rng.uniform(0.01, 0.5, M)
    sw = rng.uniform(0.001, 0.01, N)
    ad = torch.from_numpy(_tiled(a)).cuda()
    wd = torch.from_numpy(_tiled(w)).cuda()
    sad, swd = torch.from_numpy(sa).cuda(), torch.from_numpy(sw).cuda()
    out = torch.zeros((M, N), dtype=torch.float32, device="cuda")
    acc = torch.zeros((M, N), dtype=torch.int32, device="cuda")
    Q.w4a4_gemm(Q.EPI_STORE, ad, sad, wd, swd, M, N, K, out, acc, impl=impl)
    torch.cuda.synchronize()
    exp = a.astype(np.int64) @ w.T.astype(np.int64)
    assert np.array_equal(acc.cpu().numpy(), exp)
    y = exp * sa[:, None].astype(np.float64) * sw[None, :].astype(np.float64)
    np.testing.assert_allclose(out.cpu().numpy(), y, rtol=2e-7, atol=1e-7)


@pytest.mark.parametrize("M", [4, 96])
@pytest.mark.parametrize("epi", [Q.EPI_RESADD, Q.EPI_SILU, Q.EPI_SWIGLU])
def test_w4a4_gemm_epilogues(torch_cuda, M, epi):
    torch = torch_cuda
    rng = np.random.default_rng(10 + M + epi)
    K, N = 256, 256
    a = rng.integers(-7, 8, size=(M, K))
    w = rng.integers(-7, 8, size=(N, K))
    sa = rng.uniform(0.01, 0.5, M)
    sw = rng.uniform(0.001, 0.01, N)
    y = (a.astype(np.int64) @ w.T.astype(np.int64)) * (sa[:, None] * sw[None, :])
    if epi == Q.EPI_SWIGLU:
        out = torch.zeros((M, N // 2), dtype=torch.float32, device="cuda")
        g, u = y[:, 0::2], y[:, 1::2]
        exp = g / (1 + np.exp(-g)) * u
        tol = dict(rtol=1e-6, atol=1e-7)
    elif epi == Q.EPI_RESADD:  # fp64 residual stream
        base = rng.standard_normal((M, N))
        out = torch.from_numpy(base.copy()).cuda()
        exp = base + y
        tol = dict(rtol=1e-14, atol=1e-14)
    else:
        out = torch.zeros((M, N), dtype=torch.float32, device="cuda")
        exp = y / (1 + np.exp(-y))
        tol = dict(rtol=1e-6, atol=1e-7)
    Q.w4a4_gemm(epi, torch.from_numpy(_tiled(a)).cuda(), torch.from_numpy(sa).cuda(), torch.from_numpy(_tiled(w)).cuda(),
                torch.from_numpy(sw).cuda(), M, N, K, out)
    torch.cuda.synchronize()
    np.testing.assert_allclose(out.cpu().numpy(), exp, **tol)


def test_gemm_matches_reference_quantized_linear(torch_cuda):
    """End to end through the device quantizers vs quantized_linear (quant.cpp:112-115),
    with per-output-channel weight scales."""
    torch = torch_cuda
    M, K, N = 24, 256, 128
    x = _x(M, K, seed=9).astype(np.float64)
    w = (np.random.default_rng(2).standard_normal((K, N)) * 0.05).astype(np.float32).astype(np.float64)
    wc, ws = ref_quant_fit(w, 2)
    lib = _ref()
    exp = np.empty((M, N))
    O._check(lib.qref_quantized_linear(O._d(np.ascontiguousarray(x)), M, K, O._b(np.ascontiguousarray(wc)),
                                       O._d(ws), 2, N, 4, O._d(exp)), lib, "qref")
    codes, scales = Q.rmsnorm_quant(torch.from_numpy(x.astype(np.float32)).cuda(), None, 256, 1)
    wcd, wsd = Q.quant_weight(torch.from_numpy(w.astype(np.float32)).cuda(), 256, 128)
    out = torch.zeros((M, N), dtype=torch.float32, device="cuda")
    Q.w4a4_gemm(Q.EPI_STORE, codes, scales, wcd, wsd, M, N, K, out)
    torch.cuda.synchronize()
    np.testing.assert_allclose(out.cpu().numpy(), exp, rtol=1e-6, atol=1e-7)


@pytest.mark.parametrize("epi", [Q.EPI_STORE, Q.EPI_RESADD, Q.EPI_SWIGLU])
def test_w4a4_gemm_splitk_epilogues(torch_cuda, epi):
    """tcgen05 split-K (decode batches): fixed-order int32 reduction then the row-wise epilogue."""
    torch = torch_cuda
    rng = np.random.default_rng(77 + epi)
    M, K, N = 48, 1024, 512
    a = rng.integers(-7, 8, size=(M, K))
    w = rng.integers(-7, 8, size=(N, K))
    sa = rng.uniform(0.01, 0.5, M)
    sw = rng.uniform(0.001, 0.01, N)
    acc_exp = a.astype(np.int64) @ w.T.astype(np.int64)
    y = acc_exp * (sa[:, None] * sw[None, :])
    if epi == Q.EPI_SWIGLU:
        out = torch.zeros((M, N // 2), dtype=torch.float32, device="cuda")
        g, u = y[:, 0::2], y[:, 1::2]
        exp, tol = g / (1 + np.exp(-g)) * u, dict(rtol=1e-6, atol=1e-7)
    elif epi == Q.EPI_RESADD:
        base = rng.standard_normal((M, N))
        out = torch.from_numpy(base.copy()).cuda()
        exp, tol = base + y, dict(rtol=1e-14, atol=1e-14)
    else:
        out = torch.zeros((M, N), dtype=torch.float32, device="cuda")
        exp, tol = y, dict(rtol=2e-7, atol=1e-7)
    acc = torch.zeros((M, N), dtype=torch.int32, device="cuda")
    Q.w4a4_gemm(epi, torch.from_numpy(_tiled(a)).cuda(), torch.from_numpy(sa).cuda(),
                torch.from_numpy(_tiled(w)).cuda(), torch.from_numpy(sw).cuda(), M, N, K, out, acc, impl=2)
    torch.cuda.synchronize()
    assert np.array_equal(acc.cpu().numpy(), acc_exp)
    np.testing.assert_allclose(out.cpu().numpy(), exp, **tol)


@pytest.mark.parametrize("epi", [Q.EPI_STORE, Q.EPI_RESADD, Q.EPI_SILU, Q.EPI_SWIGLU])
@pytest.mark.parametrize("M,N,K", [(300, 640, 1024), (129, 256, 512), (1000, 1536, 384), (64, 4096, 256),
                                   (2048, 2560, 512), (520, 512, 4096), (1896, 4352, 256), (256, 4096, 4096),
                                   (200, 3072, 2048)])
@pytest.mark.parametrize("impl", [3, 4])
def test_w4a4_gemm_int8_operands(torch_cuda, epi, M, N, K, impl):
    """impl 3: the int8-operand tcgen05 GEMM (TMA SWIZZLE_128B tensor loads, no converter warps):
    int32 accumulators bit-exact, epilogues as the other paths; ragged M and N tiles.  M > 128
    runs the 2-SM kernel (cta_group::2, 256 x 256 tiles; more tiles than CTA pairs for the
    larger shapes, so the pair's persistent loop and double-buffered accumulators cycle).
    impl 4: the same with the split-K workspace (decode batches of 129..256 tokens: k slices
    across CTA pairs, int32 partials reduced in fixed order)."""
    torch = torch_cuda
    rng = np.random.default_rng(1000 * epi + M)
    a = rng.integers(-7, 8, size=(M, K))
    w = rng.integers(-7, 8, size=(N, K))
    sa = rng.uniform(0.01, 0.5, M)
    sw = rng.uniform(0.001, 0.01, N)
    acc_exp = a.astype(np.int64) @ w.T.astype(np.int64)
    y = acc_exp * (sa[:, None] * sw[None, :])
    if epi == Q.EPI_SWIGLU:
        out = torch.zeros((M, N // 2), dtype=torch.float32, device="cuda")
        g, u = y[:, 0::2], y[:, 1::2]
        exp, tol = g / (1 + np.exp(-g)) * u, dict(rtol=1e-5, atol=1e-6)
    elif epi == Q.EPI_SILU:
        out = torch.zeros((M, N), dtype=torch.float32, device="cuda")
        exp, tol = y / (1 + np.exp(-y)), dict(rtol=1e-5, atol=1e-6)
    elif epi == Q.EPI_RESADD:
        base = rng.standard_normal((M, N))
        out = torch.from_numpy(base.copy()).cuda()
        exp, tol = base + y, dict(rtol=1e-14, atol=1e-14)
    else:
        out = torch.zeros((M, N), dtype=torch.float32, device="cuda")
        exp, tol = y, dict(rtol=2e-7, atol=1e-7)
    acc = torch.zeros((M, N), dtype=torch.int32, device="cuda")
    Q.w4a4_gemm(epi, torch.from_numpy(_tiled(a)).cuda(), torch.from_numpy(sa).cuda(),
                torch.from_numpy(_tiled(w, 128)).cuda(), torch.from_numpy(sw).cuda(), M, N, K, out, acc, impl=impl)
    torch.cuda.synchronize()
    assert np.array_equal(acc.cpu().numpy(), acc_exp)
    np.testing.assert_allclose(out.cpu().numpy(), exp, **tol)


@pytest.mark.parametrize("M", [17, 24, 32, 40, 64])
def test_w4a4_gemv_wide_batches_int32_exact(torch_cuda, M):
    """Decode batches of 17..64 tokens: the weight-streaming GEMV with B fragments read from the
    tiled codes in global memory (rows padded to 32 / 64)."""
    torch = torch_cuda
    rng = np.random.default_rng(300 + M)
    K, N = 1024, 272
    a = rng.integers(-7, 8, size=(M, K))
    w = rng.integers(-7, 8, size=(N, K))
    sa = rng.uniform(0.01, 0.5, M)
    sw = rng.uniform(0.001, 0.01, N)
    ad = torch.from_numpy(_tiled(a, pad=64)).cuda()
    out = torch.zeros((M, N), dtype=torch.float32, device="cuda")
    acc = torch.zeros((M, N), dtype=torch.int32, device="cuda")
    Q.w4a4_gemm(Q.EPI_STORE, ad, torch.from_numpy(sa).cuda(), torch.from_numpy(_tiled(w)).cuda(),
                torch.from_numpy(sw).cuda(), M, N, K, out, acc, impl=0)
    torch.cuda.synchronize()
    exp = a.astype(np.int64) @ w.T.astype(np.int64)
    assert np.array_equal(acc.cpu().numpy(), exp)
    np.testing.assert_allclose(out.cpu().numpy(), exp * sa[:, None] * sw[None, :], rtol=2e-7, atol=1e-7)


@pytest.mark.parametrize("epi", [Q.EPI_STORE, Q.EPI_RESADD, Q.EPI_SWIGLU])
@pytest.mark.parametrize("M,N,K,ks", [(64, 4096, 4096, 4), (256, 12288, 1024, 3), (200, 1536, 11008, 5),
                                      (8, 512, 512, 2), (256, 4096, 4096, 0)])
def test_w4a4_gemm_i8_single_splitk(torch_cuda, epi, M, N, K, ks):
    """The single-CTA int8 tcgen05 kernel with k slices (decode batches): int32 partials per slice
    in the workspace, reduced in fixed order -- bit-exact accumulators, the same epilogues.
    ks = 0: the automatic slice choice (qt_w4a4_gemm_i8_workspace)."""
    torch = torch_cuda
    rng = np.random.default_rng(31 * M + ks + epi)
    a = rng.integers(-7, 8, size=(M, K))
    w = rng.integers(-7, 8, size=(N, K))
    sa = rng.uniform(0.01, 0.5, M)
    sw = rng.uniform(0.001, 0.01, N)
    acc_exp = a.astype(np.int64) @ w.T.astype(np.int64)
    y = acc_exp * (sa[:, None] * sw[None, :])
    if epi == Q.EPI_SWIGLU:
        out = torch.zeros((M, N // 2), dtype=torch.float32, device="cuda")
        g, u = y[:, 0::2], y[:, 1::2]
        exp, tol = g / (1 + np.exp(-g)) * u, dict(rtol=1e-5, atol=1e-6)
    elif epi == Q.EPI_RESADD:
        base = rng.standard_normal((M, N))
        out = torch.from_numpy(base.copy()).cuda()
        exp, tol = base + y, dict(rtol=1e-14, atol=1e-14)
    else:
        out = torch.zeros((M, N), dtype=torch.float32, device="cuda")
        exp, tol = y, dict(rtol=2e-7, atol=1e-7)
    a8 = torch.from_numpy((a * 16).astype(np.int8)).cuda()
    w8 = torch.from_numpy((w * 16).astype(np.int8)).cuda()
    if ks:
        wsp = torch.empty(ks * M * N, dtype=torch.int32, device="cuda")
    else:
        nb = Q.lib().qt_w4a4_gemm_i8_workspace(M, N, K)
        assert nb > 0  # the automatic choice splits this decode shape
        wsp = torch.empty(nb // 4, dtype=torch.int32, device="cuda")
    acc = torch.zeros((M, N), dtype=torch.int32, device="cuda")
    Q.w4a4_gemm_i8(epi, a8, torch.from_numpy(sa).cuda(), w8, torch.from_numpy(sw).cuda(), M, N, K, out, acc,
                   workspace=wsp, ksplit=ks)
    torch.cuda.synchronize()
    assert np.array_equal(acc.cpu().numpy(), acc_exp)
    np.testing.assert_allclose(out.cpu().numpy(), exp, **tol)
