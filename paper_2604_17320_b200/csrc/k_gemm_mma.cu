// k_gemm_mma.cu -- W4A4 GEMM / GEMV on int8 tensor cores through mma.sync
// (m16n8k32 s8.s8.s32), with packed int4 operands unpacked in registers.
//
// Replaces the reference's simulated W4A4 linear: matmul(fake_quant(x), W.deq)
// (numeric.cpp:33-46 at model.cpp:351-353,395,432,436,445,481-483,540,545,548,560;
// kernel-level oracle quantized_linear, quant.cpp:112-115).
//
//   y[m][n] = s_a[m] * s_w[n] * sum_k a[m][k] * w[n][k]      (int32 exact)
//
// Operands: A codes [M x K/2] bytes (token rows), W codes [N x K/2] bytes
// (output-channel rows = reference columns), both int4 two's complement, low
// nibble = even k, K padded to a multiple of 128 with zero codes.
//
// Register unpack: unpack_x16 turns 8 nibbles into two int8x4 words holding
// 16*code (even k, odd k).  A and W are unpacked identically and placed in the
// same fragment slots, so slot<->k assignment agrees for both operands and the
// dot product is exact; the accumulator carries a factor 256 removed by an
// exact arithmetic shift.  |16*7|^2 * K < 2^31 for K <= 170k.
//
//   k_gemm_tc  : token-tiled GEMM for prefill (M >= 32), 3-stage cp.async.
//   k_gemv_tc  : swap-AB GEMV for decode (M <= 16): weights stream from HBM
//                straight into A fragments (128-bit loads), tokens are the
//                n8 dimension; split-K across warps, reduced in smem.
#include "qt_common.cuh"
#include "qt_kernels.h"

namespace qt {

// y = (acc / 256) * s_a[m] * s_w[n] in fp64 (scales are the reference's fp64
// scales; the integer sum is exact), then the epilogue: store fp32, add into
// the fp64 residual, SiLU, or SwiGLU over interleaved (gate, up) columns.
template <int EPI>
QT_DEV void epi_store(void* __restrict__ outv, int ldo, int m, int n, double y0, double y1, int N) {
    if (EPI == QT_EPI_RESADD) {
        double* p = static_cast<double*>(outv) + (size_t)m * ldo + n;
        if (n + 1 < N) {
            double2 v = *reinterpret_cast<double2*>(p);
            v.x += y0;
            v.y += y1;
            *reinterpret_cast<double2*>(p) = v;
        } else if (n < N) {
            p[0] += y0;
        }
        return;
    }
    float* out = static_cast<float*>(outv);
    if (EPI == QT_EPI_SWIGLU) {
        // silu(g) * u (model.cpp:170-172 silu; SwiGLU is the R1 extension)
        if (n < N) out[(size_t)m * ldo + n / 2] = (float)(y0 / (1.0 + exp(-y0)) * y1);
        return;
    }
    float* p = out + (size_t)m * ldo + n;
    float v0, v1;
    if (EPI == QT_EPI_SILU) {
        v0 = (float)(y0 / (1.0 + exp(-y0)));
        v1 = (float)(y1 / (1.0 + exp(-y1)));
    } else {
        v0 = (float)y0;
        v1 = (float)y1;
    }
    if (n + 1 < N) *reinterpret_cast<float2*>(p) = make_float2(v0, v1);
    else if (n < N) p[0] = v0;
}

// ---------------------------------------------------------------- prefill GEMM
constexpr int GB_N = 128, GB_K = 128, G_STAGES = 3, G_ROWB = GB_K / 2;  // 64 bytes per row per stage

template <int BM, int EPI>
__global__ void __launch_bounds__(256) k_gemm_tc(const uint8_t* __restrict__ A, int lda, const double* __restrict__ sa,
                                                 const uint8_t* __restrict__ W, int ldw, const double* __restrict__ sw,
                                                 int M, int N, int K, void* __restrict__ out, int ldo,
                                                 int* __restrict__ acc_dbg) {
    constexpr int WM = BM / 2;       // warp tile rows (2 warps along M)
    constexpr int MI = WM / 16;      // m16 tiles per warp
    constexpr int NI = 4;            // n8 tiles per warp (warp tile 32 cols, 4 warps along N)
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t* As = smem;                                  // [STAGES][BM][64]
    uint8_t* Ws = smem + G_STAGES * BM * G_ROWB;         // [STAGES][128][64]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, tig = lane & 3;
    const int wm = warp >> 2, wn = warp & 3;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * GB_N;
    const int KT = K / GB_K;

    auto load_stage = [&](int stage, int kt) {
        const int kb = kt * G_ROWB;
        uint8_t* as = As + stage * BM * G_ROWB;
        uint8_t* ws = Ws + stage * GB_N * G_ROWB;
#pragma unroll
        for (int c = tid; c < BM * 4; c += 256) {
            int r = c >> 2, q = c & 3;
            bool ok = m0 + r < M;
            const uint8_t* src = A + (size_t)(ok ? m0 + r : 0) * lda + kb + q * 16;
            cp_async16(as + c * 16, src, ok);
        }
#pragma unroll
        for (int c = tid; c < GB_N * 4; c += 256) {
            int r = c >> 2, q = c & 3;
            const uint8_t* src = W + (size_t)(n0 + r) * ldw + kb + q * 16;  // W rows padded to the N tile
            cp_async16(ws + c * 16, src, true);
        }
    };

    int acc[MI][NI][4];
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j)
#pragma unroll
            for (int t = 0; t < 4; ++t) acc[i][j][t] = 0;

#pragma unroll
    for (int s = 0; s < G_STAGES - 1; ++s) {
        if (s < KT) load_stage(s, s);
        cp_async_commit();
    }
    for (int kt = 0; kt < KT; ++kt) {
        cp_async_wait<G_STAGES - 2>();
        __syncthreads();
        {
            int nk = kt + G_STAGES - 1;
            if (nk < KT) load_stage(nk % G_STAGES, nk);
            cp_async_commit();
        }
        const int stage = kt % G_STAGES;
        const uint8_t* as = As + stage * BM * G_ROWB;
        const uint8_t* ws = Ws + stage * GB_N * G_ROWB;
        uint4 av[MI][2], wv[NI];
#pragma unroll
        for (int i = 0; i < MI; ++i) {
            int r = wm * WM + i * 16 + g;
            av[i][0] = *reinterpret_cast<const uint4*>(as + r * G_ROWB + tig * 16);
            av[i][1] = *reinterpret_cast<const uint4*>(as + (r + 8) * G_ROWB + tig * 16);
        }
#pragma unroll
        for (int j = 0; j < NI; ++j) {
            int r = wn * 32 + j * 8 + g;
            wv[j] = *reinterpret_cast<const uint4*>(ws + r * G_ROWB + tig * 16);
        }
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            uint32_t bf[NI][2];
#pragma unroll
            for (int j = 0; j < NI; ++j) {
                uint32_t w = (&wv[j].x)[s];
                unpack_x16(w, bf[j][0], bf[j][1]);
            }
#pragma unroll
            for (int i = 0; i < MI; ++i) {
                uint32_t a[4];
                uint32_t w0 = (&av[i][0].x)[s], w1 = (&av[i][1].x)[s];
                unpack_x16(w0, a[0], a[2]);
                unpack_x16(w1, a[1], a[3]);
#pragma unroll
                for (int j = 0; j < NI; ++j) mma_s8_16832(acc[i][j], a, bf[j]);
            }
        }
    }
    cp_async_wait<0>();

    // epilogue: y = (acc / 256) * s_a[m] * s_w[n]
#pragma unroll
    for (int i = 0; i < MI; ++i) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int m = m0 + wm * WM + i * 16 + g + h * 8;
            if (m >= M) continue;
            const double a_s = sa[m];
#pragma unroll
            for (int j = 0; j < NI; ++j) {
                const int n = n0 + wn * 32 + j * 8 + tig * 2;
                const int c0 = acc[i][j][2 * h] >> 8, c1 = acc[i][j][2 * h + 1] >> 8;
                if (acc_dbg) {
                    if (n < N) acc_dbg[(size_t)m * N + n] = c0;
                    if (n + 1 < N) acc_dbg[(size_t)m * N + n + 1] = c1;
                }
                const double y0 = (double)c0 * (a_s * sw[n]);
                const double y1 = (double)c1 * (a_s * sw[n + 1]);
                epi_store<EPI>(out, ldo, m, n, y0, y1, N);
            }
        }
    }
}

// ---------------------------------------------------------------- decode GEMV
// Block = 8 warps = RB row-blocks (16 channels each) x KS = 8/RB K-slices.
// Tokens (M <= 8*NT) are staged once per block in smem (row stride padded so
// the 16-byte fragment loads are bank-conflict free).
template <int NT, int RB, int EPI>
__global__ void __launch_bounds__(256) k_gemv_tc(const uint8_t* __restrict__ A, int lda, const double* __restrict__ sa,
                                                 const uint8_t* __restrict__ W, int ldw, const double* __restrict__ sw,
                                                 int M, int N, int K, void* __restrict__ out, int ldo,
                                                 int* __restrict__ acc_dbg) {
    constexpr int KS = 8 / RB;
    constexpr int TOK = 8 * NT;
    extern __shared__ __align__(128) uint8_t smem[];
    const int kb = K / 2;
    const int ldsA = kb + 64;                  // bytes; ((kb + 64) mod 128) == 64 when kb mod 128 == 0
    uint8_t* As = smem;                        // [TOK][ldsA]
    int* red = reinterpret_cast<int*>(smem + TOK * ldsA);  // [KS][RB*16][TOK]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, tig = lane & 3;
    const int rb = warp % RB, ks = warp / RB;
    const int c0 = blockIdx.x * (16 * RB);

    // stage activations (zero rows beyond M)
    for (int c = tid; c < TOK * (kb / 16); c += 256) {
        int r = c / (kb / 16), q = c % (kb / 16);
        bool ok = r < M;
        cp_async16(As + r * ldsA + q * 16, A + (size_t)(ok ? r : 0) * lda + q * 16, ok);
    }
    cp_async_commit();

    // K slice for this warp, in 128-k chunks (64 bytes per row)
    const int chunks = K / 128;
    const int per = (chunks + KS - 1) / KS;
    const int ch0 = ks * per, ch1 = min(chunks, ch0 + per);
    const uint8_t* w0p = W + (size_t)(c0 + rb * 16 + g) * ldw + tig * 16;
    const uint8_t* w1p = w0p + (size_t)8 * ldw;

    int acc[NT][4];
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int t = 0; t < 4; ++t) acc[j][t] = 0;

    cp_async_wait<0>();
    __syncthreads();

    constexpr int U = 4;
    int ch = ch0;
    for (; ch + U <= ch1; ch += U) {
        uint4 wa[U], wb[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            wa[u] = ldg_nc_v4(w0p + (size_t)(ch + u) * 64);
            wb[u] = ldg_nc_v4(w1p + (size_t)(ch + u) * 64);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            uint4 bv[NT];
#pragma unroll
            for (int j = 0; j < NT; ++j)
                bv[j] = *reinterpret_cast<const uint4*>(As + (j * 8 + g) * ldsA + (ch + u) * 64 + tig * 16);
#pragma unroll
            for (int s = 0; s < 4; ++s) {
                uint32_t a[4];
                unpack_x16((&wa[u].x)[s], a[0], a[2]);
                unpack_x16((&wb[u].x)[s], a[1], a[3]);
#pragma unroll
                for (int j = 0; j < NT; ++j) {
                    uint32_t b[2];
                    unpack_x16((&bv[j].x)[s], b[0], b[1]);
                    mma_s8_16832(acc[j], a, b);
                }
            }
        }
    }
    for (; ch < ch1; ++ch) {
        uint4 wa = ldg_nc_v4(w0p + (size_t)ch * 64);
        uint4 wb = ldg_nc_v4(w1p + (size_t)ch * 64);
        uint4 bv[NT];
#pragma unroll
        for (int j = 0; j < NT; ++j)
            bv[j] = *reinterpret_cast<const uint4*>(As + (j * 8 + g) * ldsA + ch * 64 + tig * 16);
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            uint32_t a[4];
            unpack_x16((&wa.x)[s], a[0], a[2]);
            unpack_x16((&wb.x)[s], a[1], a[3]);
#pragma unroll
            for (int j = 0; j < NT; ++j) {
                uint32_t b[2];
                unpack_x16((&bv[j].x)[s], b[0], b[1]);
                mma_s8_16832(acc[j], a, b);
            }
        }
    }

    // split-K reduction: red[ks][row][tok]
#pragma unroll
    for (int j = 0; j < NT; ++j) {
        const int r = rb * 16 + g;
        const int t = j * 8 + tig * 2;
        int* base = red + (size_t)ks * (RB * 16 * TOK);
        base[r * TOK + t] = acc[j][0];
        base[r * TOK + t + 1] = acc[j][1];
        base[(r + 8) * TOK + t] = acc[j][2];
        base[(r + 8) * TOK + t + 1] = acc[j][3];
    }
    __syncthreads();
    // epilogue over (channel pair, token): channels cp*2, cp*2+1
    for (int e = tid; e < RB * 8 * TOK; e += 256) {
        const int t = e % TOK, cpair = e / TOK;
        if (t >= M) continue;
        int s0 = 0, s1 = 0;
#pragma unroll
        for (int k = 0; k < KS; ++k) {
            s0 += red[(size_t)k * (RB * 16 * TOK) + (2 * cpair) * TOK + t];
            s1 += red[(size_t)k * (RB * 16 * TOK) + (2 * cpair + 1) * TOK + t];
        }
        s0 >>= 8;
        s1 >>= 8;
        const int n = c0 + 2 * cpair;
        if (acc_dbg) {
            if (n < N) acc_dbg[(size_t)t * N + n] = s0;
            if (n + 1 < N) acc_dbg[(size_t)t * N + n + 1] = s1;
        }
        const double a_s = sa[t];
        epi_store<EPI>(out, ldo, t, n, (double)s0 * (a_s * sw[n]), (double)s1 * (a_s * sw[n + 1]), N);
    }
}

template <int EPI>
int launch_gemm(const uint8_t* A, int lda, const double* sa, const uint8_t* W, int ldw, const double* sw, int M,
                int N, int K, void* out, int ldo, int* acc_dbg, cudaStream_t st) {
    if (M <= 0) return 0;
    if (K % 128 || lda % 16 || ldw % 16) return -1;
    const int nb = (N + GB_N - 1) / GB_N;
    if (M <= 16) {
        const int kb = K / 2;
        const int n16 = (N + 15) / 16;
        int RB = (n16 / 4 >= 296) ? 4 : ((n16 / 2 >= 148) ? 2 : 1);
        if ((N % (16 * RB)) != 0) RB = 1;
        const int TOK = M <= 8 ? 8 : 16;
        const size_t smem = (size_t)TOK * (kb + 64) + (size_t)(8 / RB) * RB * 16 * TOK * 4;
        const dim3 grid((N + 16 * RB - 1) / (16 * RB));
#define QT_GEMV(NT_, RB_)                                                                               \
    do {                                                                                                \
        auto kfn = k_gemv_tc<NT_, RB_, EPI>;                                                            \
        cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);              \
        kfn<<<grid, 256, smem, st>>>(A, lda, sa, W, ldw, sw, M, N, K, out, ldo, acc_dbg);               \
    } while (0)
        if (TOK == 8) {
            if (RB == 4) QT_GEMV(1, 4);
            else if (RB == 2) QT_GEMV(1, 2);
            else QT_GEMV(1, 1);
        } else {
            if (RB == 4) QT_GEMV(2, 4);
            else if (RB == 2) QT_GEMV(2, 2);
            else QT_GEMV(2, 1);
        }
#undef QT_GEMV
        return (int)cudaGetLastError();
    }
    if (M <= 512 || (long long)((M + 127) / 128) * nb < 148) {
        constexpr int BM = 64;
        const size_t smem = (size_t)G_STAGES * (BM + GB_N) * G_ROWB;
        auto kfn = k_gemm_tc<BM, EPI>;
        cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kfn<<<dim3(nb, (M + BM - 1) / BM), 256, smem, st>>>(A, lda, sa, W, ldw, sw, M, N, K, out, ldo, acc_dbg);
    } else {
        constexpr int BM = 128;
        const size_t smem = (size_t)G_STAGES * (BM + GB_N) * G_ROWB;
        auto kfn = k_gemm_tc<BM, EPI>;
        cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kfn<<<dim3(nb, (M + BM - 1) / BM), 256, smem, st>>>(A, lda, sa, W, ldw, sw, M, N, K, out, ldo, acc_dbg);
    }
    return (int)cudaGetLastError();
}

}  // namespace qt

extern "C" int qt_launch_w4a4_mma(int epi, const uint8_t* A, int lda, const double* sa, const uint8_t* W, int ldw,
                                  const double* sw, int M, int N, int K, void* out, int ldo, int* acc_dbg,
                                  cudaStream_t st) {
    using namespace qt;
    switch (epi) {
        case QT_EPI_STORE: return launch_gemm<QT_EPI_STORE>(A, lda, sa, W, ldw, sw, M, N, K, out, ldo, acc_dbg, st);
        case QT_EPI_RESADD: return launch_gemm<QT_EPI_RESADD>(A, lda, sa, W, ldw, sw, M, N, K, out, ldo, acc_dbg, st);
        case QT_EPI_SILU: return launch_gemm<QT_EPI_SILU>(A, lda, sa, W, ldw, sw, M, N, K, out, ldo, acc_dbg, st);
        case QT_EPI_SWIGLU: return launch_gemm<QT_EPI_SWIGLU>(A, lda, sa, W, ldw, sw, M, N, K, out, ldo, acc_dbg, st);
    }
    return -1;
}
