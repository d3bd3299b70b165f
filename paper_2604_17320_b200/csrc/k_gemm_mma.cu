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
#include <algorithm>
#include <cstdlib>

#include "qt_common.cuh"
#include "qt_epilogue.cuh"
#include "qt_kernels.h"

namespace qt {

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
            const uint8_t* src = A + w4t_offset(ok ? m0 + r : 0, kb + q * 16, lda);  // tiled rows
            cp_async16(as + c * 16, src, ok);
        }
#pragma unroll
        for (int c = tid; c < GB_N * 4; c += 256) {
            int r = c >> 2, q = c & 3;
            const uint8_t* src = W + w4t_offset(n0 + r, kb + q * 16, ldw);  // tiled rows, padded to the N tile
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
// row blocks per CTA beyond the first whose weights are L2-prefetched before the
// dependency wait
constexpr int kGemvL2Rows = 1;
// Persistent, HBM-streaming GEMV for decode (M <= 16 tokens).  Each CTA owns a
// strided set of 16-channel row blocks; its 8 warps split K.  The token codes
// are staged once per CTA in smem.  Weight loads run one batch (U tiles of
// 16 rows x 128 k per warp, each warp load instruction = 512 contiguous bytes
// of a tile) ahead of the MMAs across row-block boundaries; the first batch is
// issued before the programmatic-dependency wait and overlaps the upstream
// kernel.  Swap-AB mma.sync m16n8k32: weights are the 16-row operand, tokens
// the n8 operand; split-K partials are reduced in smem for the fused epilogue.
//
// NT <= 2 (<= 16 tokens): the token codes are staged in smem.  NT 4 / 8 (17..64
// tokens, decode batches): they do not fit for K = d_ff, so the B fragments are
// read straight from the (L1/L2-resident) tiled activation codes; each warp
// keeps re-reading the same k slice across its row blocks.
#ifndef QT_GEMV_MINB
#define QT_GEMV_MINB 2  // 3 spills (80 regs) and measured slower
#endif
// AREG (NT = 1, K <= 4096: one batch per row block): each lane's activation fragments for its
// k slice are loaded once into registers after the dependency wait -- no smem staging, no
// block barrier before the first MMA.
template <int NT, int EPI, bool AREG = false>
__global__ void __launch_bounds__(256, (NT <= 2 && !(AREG && NT == 2)) ? QT_GEMV_MINB : 1) k_gemv_reg(const uint8_t* __restrict__ A, int lda, const double* __restrict__ sa,
                                                  const uint8_t* __restrict__ W, int ldw, const double* __restrict__ sw,
                                                  int M, int N, int K, void* __restrict__ out, int ldo,
                                                  int* __restrict__ acc_dbg, int l2rows,
                                                  float* __restrict__ pmax, int pmax_ld) {
    constexpr int TOK = 8 * NT;
    constexpr bool ASM = NT <= 2 && !AREG;  // activation codes staged in smem
    constexpr int U = NT <= 2 ? 4 : 2;
    extern __shared__ __align__(128) uint8_t smem[];
    const int kb = K / 2;
    const int ldsA = ASM ? kb + 64 : 0;
    uint8_t* As = smem;
    int* red = reinterpret_cast<int*>(smem + TOK * ldsA);
    __shared__ int smx[TOK];  // per-token max |v| of this CTA's fp32 outputs (float bits, >= 0)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid < TOK) smx[tid] = 0;
    const int g = lane >> 2, tig = lane & 3;
    const int n_rb = (N + 15) / 16;
    const int KT = K / 128;
    const int per = (KT + 7) / 8;
    const int ch0 = warp * per, ch1 = min(KT, ch0 + per);
    const int nbat = (per + U - 1) / U;
    uint4 wa[U], wb[U];
    auto fetch = [&](int rb, int bat, uint4* xa, uint4* xb) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int c = ch0 + bat * U + u;
            const bool ok = rb < n_rb && c < ch1;
            const uint8_t* tile = W + ((size_t)c * (ldw >> 4) + rb) * 1024 + g * 64 + tig * 16;
            xa[u] = ok ? ldg_nc_v4(tile) : make_uint4(0, 0, 0, 0);
            xb[u] = ok ? ldg_nc_v4(tile + 512) : make_uint4(0, 0, 0, 0);
        }
    };
    int rb = blockIdx.x, bat = 0;
    fetch(rb, 0, wa, wb);
    {   // weights do not depend on the upstream kernel: while it still runs, pull this warp's
        // k slice of the CTA's next row blocks toward L2 (fire-and-forget, no registers)
        const int pre_rb = l2rows;
        for (int j = 1; j <= pre_rb; ++j) {
            const int r2 = blockIdx.x + j * gridDim.x;
            if (r2 >= n_rb) break;
            for (int c = ch0 + (lane >> 3); c < ch1; c += 4)  // 8 lanes x 128 B per 1 KB tile
                asm volatile("prefetch.global.L2 [%0];\n" ::"l"(W + ((size_t)c * (ldw >> 4) + r2) * 1024 +
                                                               (lane & 7) * 128));
        }
        if (nbat > 1)  // and the rest of the first row block beyond the register batch
            for (int c = ch0 + U + (lane >> 3); c < ch1; c += 4)
                asm volatile("prefetch.global.L2 [%0];\n" ::"l"(W + ((size_t)c * (ldw >> 4) + rb) * 1024 +
                                                               (lane & 7) * 128));
    }
    pdl_wait();
    uint4 bA[AREG ? U : 1][AREG ? NT : 1];
    if constexpr (AREG) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int c = ch0 + u;
#pragma unroll
            for (int j = 0; j < NT; ++j)
                bA[u][j] = c < ch1 ? ldg_nc_v4(A + w4t_offset(j * 8 + g, c * 64 + tig * 16, lda))
                                   : make_uint4(0, 0, 0, 0);
        }
    }
    if (ASM) {  // each warp stages only its own k slice of the token codes: no block barrier
        const int q0 = ch0 * 4, nq = (ch1 - ch0) * 4;  // 16-byte chunks of the slice
        for (int c = lane; c < TOK * nq; c += 32) {
            const int r = c / nq, q = q0 + c % nq;
            const bool ok = r < M;
            cp_async16(As + r * ldsA + q * 16, A + w4t_offset(ok ? r : 0, q * 16, lda), ok);
        }
        cp_async_commit();
        cp_async_wait<0>();
        __syncwarp();
    }
    pdl_launch_dependents();
    int acc[NT][4];
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0;
    // epilogue operands of the current row block (8 * TOK <= 256: one (token, column pair) per
    // thread), loaded when the row block starts so their latency hides behind its MMAs
    constexpr bool EPRE = 8 * TOK <= 256;
    const int et = tid % TOK, ecp = tid / TOK;
    const bool eon = EPRE && tid < 8 * TOK && et < M;
    const double e_sa = eon ? sa[et] : 0.0;
    double2 e_sw = make_double2(0.0, 0.0), e_x = make_double2(0.0, 0.0);
    int rbi = 0;  // row blocks finished (reduction buffer parity)
    while (rb < n_rb) {
        int nrb = rb, nbt = bat + 1;
        if (nbt == nbat) {
            nbt = 0;
            nrb = rb + gridDim.x;
        }
        if (eon && bat == 0) {
            const int n = rb * 16 + 2 * ecp;
            e_sw = make_double2(n < N ? sw[n] : 0.0, n + 1 < N ? sw[n + 1] : 0.0);
            if constexpr (EPI == QT_EPI_RESADD) {
                const double* p = static_cast<const double*>(out) + (size_t)et * ldo + n;
                if (n + 1 < N) e_x = *reinterpret_cast<const double2*>(p);
                else if (n < N) e_x.x = p[0];
            }
        }
        uint4 na[U], nb[U];
        fetch(nrb, nbt, na, nb);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int c = ch0 + bat * U + u;
            if (c >= ch1) break;
            uint4 bv[NT];
#pragma unroll
            for (int j = 0; j < NT; ++j) {
                if constexpr (AREG) bv[j] = bA[u][j];  // nbat == 1: batch u is k tile ch0 + u
                else if (ASM) bv[j] = *reinterpret_cast<const uint4*>(As + (j * 8 + g) * ldsA + c * 64 + tig * 16);
                else bv[j] = ldg_nc_v4(A + w4t_offset(j * 8 + g, c * 64 + tig * 16, lda));  // rows >= M: discarded
            }
#pragma unroll
            for (int s2 = 0; s2 < 4; ++s2) {
                uint32_t a[4];
                unpack_x16((&wa[u].x)[s2], a[0], a[2]);
                unpack_x16((&wb[u].x)[s2], a[1], a[3]);
#pragma unroll
                for (int j = 0; j < NT; ++j) {
                    uint32_t b[2];
                    unpack_x16((&bv[j].x)[s2], b[0], b[1]);
                    mma_s8_16832(acc[j], a, b);
                }
            }
        }
        if (bat == nbat - 1) {
            // double-buffered reduction buffer: the 2 epilogue warps finish row block i while the
            // others run the MMAs of row block i + 1 (no barrier after the epilogue)
            int* redb = red + (size_t)(rbi & 1) * (8 * 16 * TOK);
            ++rbi;
            int* base = redb + (size_t)warp * (16 * TOK);
#pragma unroll
            for (int j = 0; j < NT; ++j) {
                const int t = j * 8 + tig * 2;
                base[g * TOK + t] = acc[j][0];
                base[g * TOK + t + 1] = acc[j][1];
                base[(g + 8) * TOK + t] = acc[j][2];
                base[(g + 8) * TOK + t + 1] = acc[j][3];
                acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0;
            }
            __syncthreads();
            for (int e = tid; e < 8 * TOK; e += 256) {
                const int t = e % TOK, cpair = e / TOK;
                if (t < M) {
                    int s0 = 0, s1 = 0;
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        s0 += redb[(size_t)k * (16 * TOK) + (2 * cpair) * TOK + t];
                        s1 += redb[(size_t)k * (16 * TOK) + (2 * cpair + 1) * TOK + t];
                    }
                    s0 >>= 8;
                    s1 >>= 8;
                    const int n = rb * 16 + 2 * cpair;
                    if (acc_dbg) {
                        if (n < N) acc_dbg[(size_t)t * N + n] = s0;
                        if (n + 1 < N) acc_dbg[(size_t)t * N + n + 1] = s1;
                    }
                    if constexpr (EPRE) {  // e == tid: the prefetched scales / residual
                        const double y0 = (double)s0 * (e_sa * e_sw.x), y1 = (double)s1 * (e_sa * e_sw.y);
                        if constexpr (EPI == QT_EPI_RESADD) {
                            double* p = static_cast<double*>(out) + (size_t)t * ldo + n;
                            if (n + 1 < N) *reinterpret_cast<double2*>(p) = make_double2(e_x.x + y0, e_x.y + y1);
                            else if (n < N) p[0] = e_x.x + y0;
                        } else {
                            const float v = epi_store<EPI>(out, ldo, t, n, y0, y1, N);
                            if (pmax) atomicMax(&smx[t], __float_as_int(v));
                        }
                    } else {
                        const double a_s = sa[t];
                        const float v = epi_store<EPI>(out, ldo, t, n, (double)s0 * (a_s * sw[n]),
                                                       (double)s1 * (a_s * sw[n + 1]), N);
                        if (pmax) atomicMax(&smx[t], __float_as_int(v));
                    }
                }
            }
        }
        rb = nrb;
        bat = nbt;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            wa[u] = na[u];
            wb[u] = nb[u];
        }
    }
    if (pmax) {  // this CTA's slot of the per-row partial max (every CTA writes its own), or with
        // pmax_ld == 0 one max per row by integer atomicMax (non-negative float bits: exact,
        // order-independent); the caller zeroes those slots between uses
        __syncthreads();
        if (tid < M && tid < TOK) {
            if (pmax_ld == 0) atomicMax(reinterpret_cast<int*>(pmax) + tid, smx[tid]);
            else pmax[(size_t)tid * pmax_ld + blockIdx.x] = __int_as_float(smx[tid]);
        }
    }
}

template <int EPI>
int launch_gemm(const uint8_t* A, int lda, const double* sa, const uint8_t* W, int ldw, const double* sw, int M,
                int N, int K, void* out, int ldo, int* acc_dbg, cudaStream_t st, float* pmax = nullptr,
                int pmax_ld = 0, int* n_part = nullptr) {
    if (n_part) *n_part = 0;
    if (M <= 0) return 0;
    if (K % 128 || lda % 16 || ldw % 16 || M > lda || N > ldw) return -1;  // lda/ldw = padded rows
    const int nb = (N + GB_N - 1) / GB_N;
    float* pm = nullptr;  // GEMV paths: one partial-max slot per CTA
    auto want_pmax = [&](int ctas) {
        if (pmax && (pmax_ld == 0 || ctas <= pmax_ld)) {
            pm = pmax;
            if (n_part) *n_part = pmax_ld == 0 ? 1 : ctas;
        }
    };
    if (M > 16 && M <= 64 && lda >= ((M + 31) / 32) * 32) {
        // 17..64 tokens: B fragments from global (padded tile rows up to 32 / 64 must exist)
        const int n_rb = (N + 15) / 16;
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
        const dim3 grid(std::min(n_rb, 2 * sms));
        if (M <= 32) {
            want_pmax((int)grid.x);
            const size_t smem = (size_t)2 * 8 * 16 * 32 * 4;
            auto kfn = k_gemv_reg<4, EPI>;
            cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            return launch_pdl(kfn, grid, dim3(256), smem, st, A, lda, sa, W, ldw, sw, M, N, K, out, ldo, acc_dbg,
                              kGemvL2Rows, pm, pmax_ld);
        }
        if (lda >= 64) {
            want_pmax((int)grid.x);
            const size_t smem = (size_t)2 * 8 * 16 * 64 * 4;
            auto kfn = k_gemv_reg<8, EPI>;
            cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            return launch_pdl(kfn, grid, dim3(256), smem, st, A, lda, sa, W, ldw, sw, M, N, K, out, ldo, acc_dbg,
                              kGemvL2Rows, pm, pmax_ld);
        }
    }
    if (M <= 16) {
        const int kb = K / 2;
        const int TOK = M <= 8 ? 8 : 16;
        const size_t smem = (size_t)TOK * (kb + 64) + (size_t)2 * 8 * 16 * TOK * 4;
        const int n_rb = (N + 15) / 16;
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
        const dim3 grid(std::min(n_rb, QT_GEMV_MINB * sms));
        want_pmax((int)grid.x);
#ifndef QT_GEMV_AREG2
#define QT_GEMV_AREG2 1  // CTAs per SM of the 9..16-token AREG GEMV (0: the smem-staged one).
                         // A/B (tools/gpu_attn_ab.sh): C4 decode 2.10 -> 2.04 ms/step, C5 B = 16
                         // 2.19 -> 2.05 ms/step at 1; 2 (two waves) 2.17 / 2.17
#endif
        // AREG: K <= 4096 is one register batch per warp (the 9..16-token variant spills at 2
        // CTAs per SM -- 183 registers -- so it runs one CTA per SM)
        if (QT_GEMV_AREG2 && TOK == 16 && (K / 128 + 7) / 8 <= 4) {
            const size_t smem2 = (size_t)2 * 8 * 16 * TOK * 4;
            auto kfn = k_gemv_reg<2, EPI, true>;
            cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2);
            return launch_pdl(kfn, dim3(std::min(n_rb, QT_GEMV_AREG2 * sms)), dim3(256), smem2, st, A, lda, sa, W,
                              ldw, sw, M, N, K, out, ldo, acc_dbg, kGemvL2Rows, pm, pmax_ld);
        }
        if (TOK == 8 && (K / 128 + 7) / 8 <= 4) {
            const size_t smem2 = (size_t)2 * 8 * 16 * TOK * 4;  // split-K reduction buffers only
            auto kfn = k_gemv_reg<1, EPI, true>;
            cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2);
            return launch_pdl(kfn, grid, dim3(256), smem2, st, A, lda, sa, W, ldw, sw, M, N, K, out, ldo, acc_dbg,
                              kGemvL2Rows, pm, pmax_ld);
        }
        if (TOK == 8) {
            auto kfn = k_gemv_reg<1, EPI>;
            cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            return launch_pdl(kfn, grid, dim3(256), smem, st, A, lda, sa, W, ldw, sw, M, N, K, out, ldo, acc_dbg,
                              kGemvL2Rows, pm, pmax_ld);
        }
        auto kfn = k_gemv_reg<2, EPI>;
        cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        return launch_pdl(kfn, grid, dim3(256), smem, st, A, lda, sa, W, ldw, sw, M, N, K, out, ldo, acc_dbg,
                              kGemvL2Rows, pm, pmax_ld);
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

// pmax (may be null): per-row partial max |v| of the fp32 outputs, pmax[m * pmax_ld + p],
// p < *n_part (one slot per GEMV CTA); *n_part = 0 when this launch produced none.
extern "C" int qt_launch_w4a4_mma_ex(int epi, const uint8_t* A, int lda, const double* sa, const uint8_t* W,
                                     int ldw, const double* sw, int M, int N, int K, void* out, int ldo,
                                     int* acc_dbg, float* pmax, int pmax_ld, int* n_part, cudaStream_t st) {
    using namespace qt;
    switch (epi) {
        case QT_EPI_STORE:
            return launch_gemm<QT_EPI_STORE>(A, lda, sa, W, ldw, sw, M, N, K, out, ldo, acc_dbg, st, pmax, pmax_ld,
                                             n_part);
        case QT_EPI_RESADD:
            return launch_gemm<QT_EPI_RESADD>(A, lda, sa, W, ldw, sw, M, N, K, out, ldo, acc_dbg, st, nullptr, 0,
                                              n_part);
        case QT_EPI_SILU:
            return launch_gemm<QT_EPI_SILU>(A, lda, sa, W, ldw, sw, M, N, K, out, ldo, acc_dbg, st, pmax, pmax_ld,
                                            n_part);
        case QT_EPI_SWIGLU:
            return launch_gemm<QT_EPI_SWIGLU>(A, lda, sa, W, ldw, sw, M, N, K, out, ldo, acc_dbg, st, pmax, pmax_ld,
                                              n_part);
    }
    return -1;
}

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
