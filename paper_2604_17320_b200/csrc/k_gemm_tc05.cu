// k_gemm_tc05.cu -- W4A4 prefill GEMM on the 5th-generation tensor cores
// (tcgen05.mma kind::i8, int32 accumulators in TMEM), sm_100a.
//
//   y[m][n] = s_a[m] * s_w[n] * sum_k a[m][k] * w[n][k]
//
// replaces matmul(fake_quant(x), W.deq) (numeric.cpp:33-46 at
// model.cpp:351-353,395,432,436,445) for the prefill token batch.
//
// Persistent CTAs (one per SM) walk 128 x 256 output tiles (m-tile fastest,
// so concurrent CTAs share weight tiles in L2), K in 128-wide blocks:
//   warp 0      TMA producer: 1D bulk copies of the packed int4 tiles (both
//               operands use the 16-row x 128-k 1 KB tile layout) into a
//               5-stage packed ring (mbarrier complete_tx).
//   warps 2..5  converters: packed int4 -> int8 (x16, two's complement in the
//               high nibble, exact) written in the UMMA canonical K-major
//               SWIZZLE_128B layout of a 2-stage int8 ring; fence.proxy.async
//               then arrive.
//   warp 1      TMEM allocator + single-thread MMA issuer: 4 x
//               tcgen05.mma.cta_group::1.kind::i8 (M128 N256 K32) per k-block
//               into one of two 256-column TMEM accumulators; tcgen05.commit
//               releases the int8 stage / hands the accumulator to the epilogue.
//   warps 6..9  epilogue: tcgen05.ld 32x32b, exact >>8, fp64 scales, fused
//               store / residual add / SiLU / SwiGLU -- overlapping the next
//               tile's main loop (double-buffered accumulators).
#include <cuda.h>  // CUtensorMap (types only; the encoder comes from cudaGetDriverEntryPoint)

#include <algorithm>
#include <cstdlib>

#include "qt_common.cuh"
#include "qt_epilogue.cuh"
#include "qt_kernels.h"

namespace qt {

constexpr int T5_BM = 128, T5_BN = 256, T5_BKB = 64;  // BK = 128 int4 = 64 packed bytes
constexpr int T5_PS = 3, T5_IS = 3, T5_ACC = 2;       // packed stages, int8 stages, TMEM accumulators
constexpr int T5_PA = T5_BM * T5_BKB, T5_PB = T5_BN * T5_BKB;  // packed bytes per stage
constexpr int T5_IA = T5_BM * 128, T5_IB = T5_BN * 128;        // int8 bytes per stage
constexpr int T5_CW = 8;                         // converter warps
constexpr int T5_CT = T5_CW * 32;                // converter threads
constexpr int T5_EW0 = 2 + T5_CW;                // first epilogue warp
constexpr int T5_EWN = 8;                        // epilogue warps: 2 per TMEM lane quarter (column halves)
constexpr int T5_ET = T5_EWN * 32;
constexpr int T5_THREADS = (T5_EW0 + T5_EWN) * 32;  // 0 TMA, 1 MMA, converters, epilogue

struct T5Smem {
    // int8 ring first: 1024-byte aligned SW128 atoms
    static constexpr size_t ia = 0;
    static constexpr size_t ib = ia + (size_t)T5_IS * T5_IA;
    static constexpr size_t pa = ib + (size_t)T5_IS * T5_IB;
    static constexpr size_t pb = pa + (size_t)T5_PS * T5_PA;
    static constexpr size_t swb = pb + (size_t)T5_PS * T5_PB;   // per-accumulator weight scales [2][256] f64
    static constexpr size_t bars = swb + (size_t)T5_ACC * T5_BN * 8;
    static constexpr size_t total = bars + 256;
};

QT_DEV uint64_t umma_desc_sw128(uint32_t saddr) {
    // SmemDescriptor (cute/arch/mma_sm100_desc.hpp): start>>4 [0,14), LBO>>4 [16,30)
    // = 1 (ignored for swizzled K-major), SBO>>4 [32,46) = 1024>>4 (8-row atom
    // stride), version [46,48) = 1, base_offset 0, layout [61,64) = 2 (SW128).
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}

// InstrDescriptor: c_format S32 (2) [4,6), a/b format signed int8 (1) [7,10)/[10,13),
// K-major A/B, n_dim = N>>3 [17,23), m_dim = M>>4 [24,29).
constexpr uint32_t t5_idesc() {
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(T5_BN >> 3) << 17) | ((uint32_t)(T5_BM >> 4) << 24);
}

QT_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
QT_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }

QT_DEV void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accum) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
        : "memory");
}

QT_DEV void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
                 : "memory");
}

QT_DEV void tmem_ld32(uint32_t taddr, uint32_t* r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

// one packed 16-byte chunk (32 k of one row) -> two swizzled int8 16-byte chunks
QT_DEV void convert_chunk(const uint8_t* packed, uint8_t* i8, int row, int q) {
    const uint4 w = *reinterpret_cast<const uint4*>(packed + (size_t)row * T5_BKB + q * 16);
    uint4 o0, o1;
    unpack_x16(w.x, o0.x, o0.y);
    unpack_x16(w.y, o0.z, o0.w);
    unpack_x16(w.z, o1.x, o1.y);
    unpack_x16(w.w, o1.z, o1.w);
    uint8_t* atom = i8 + (size_t)(row >> 3) * 1024 + (row & 7) * 128;
    const int c0 = 2 * q, c1 = 2 * q + 1, sw = row & 7;
    *reinterpret_cast<uint4*>(atom + ((c0 ^ sw) << 4)) = o0;
    *reinterpret_cast<uint4*>(atom + ((c1 ^ sw) << 4)) = o1;
}

// unpack one packed 16-byte chunk (32 k of one row) already in registers -> two
// swizzled int8 16-byte chunks
QT_DEV void store_converted(const uint4 w, uint8_t* i8, int row, int q) {
    uint4 o0, o1;
    unpack_x16(w.x, o0.x, o0.y);
    unpack_x16(w.y, o0.z, o0.w);
    unpack_x16(w.z, o1.x, o1.y);
    unpack_x16(w.w, o1.z, o1.w);
    uint8_t* atom = i8 + (size_t)(row >> 3) * 1024 + (row & 7) * 128;
    const int c0 = 2 * q, c1 = 2 * q + 1, sw = row & 7;
    *reinterpret_cast<uint4*>(atom + ((c0 ^ sw) << 4)) = o0;
    *reinterpret_cast<uint4*>(atom + ((c1 ^ sw) << 4)) = o1;
}

// Epilogue warps (T5_EWN of them, first warp ew0): warp & 3 = TMEM lane quarter (32 rows),
// (warp - ew0) / 4 = column half.  Shared by the packed-int4 and the int8-operand kernels.
// Work unit u (u0, u0 + ustep, ... < units): tile t = u % tiles, k slice u / tiles; the
// tile's M tile is (t % mtp) * cl + rank (cl = cluster size along M) and its N tile t / mtp.
template <int EPI, int BN = T5_BN>
QT_DEV void t5_epilogue_g(int ew0, int warp, int lane, uint32_t tmem, int u0, int ustep, int units, int tiles,
                          int mtp, int cl, int rank, int M, int N, const double* __restrict__ sa,
                          const double* __restrict__ sw, double* sws, void* __restrict__ out, int ldo,
                          int* __restrict__ acc_dbg, int ksplit, int* __restrict__ ws, float* __restrict__ pmax,
                          int pmax_ld, uint64_t* tfull, uint64_t* tempty, bool pair = false) {
    // ---------------- epilogue: 8 warps; warp & 3 = TMEM lane quarter (32 rows), and
    // (warp - ew0) / 4 = column half -- the per-element fp64 scale math is split 2 ways
    pdl_wait();  // scales / residual come from upstream kernels
    pdl_launch_dependents();
    const int q = warp & 3;
    const int et = threadIdx.x - ew0 * 32;
    const int jh = ((warp - ew0) >> 2) * (BN / 64);  // first 32-column chunk of this half
    int tl = 0;
    for (int u = u0; u < units; u += ustep, ++tl) {
        const int t = u % tiles, sl = u / tiles;
        const int acc = tl % T5_ACC;
        const int m0 = ((t % mtp) * cl + rank) * T5_BM, n0 = (t / mtp) * BN;
        double* swt = sws + acc * BN;
        for (int i = et; i < BN; i += T5_ET) swt[i] = n0 + i < N ? sw[n0 + i] : 0.0;
        if (EPI == QT_EPI_RESADD && ksplit == 1) {
            // pull this thread's residual row segment (256 fp64) toward L2 while the
            // tile's MMAs run: the read-modify-write below then hits L2, not HBM
            const int mr = m0 + q * 32 + lane;
            const int c0 = jh * 32;
            if (mr < M && n0 + c0 < N) {
                const char* rp =
                    reinterpret_cast<const char*>(static_cast<const double*>(out) + (size_t)mr * ldo + n0 + c0);
                const int nb = min(BN / 2, N - n0 - c0) * 8;
                for (int c = 0; c < nb; c += 128) asm volatile("prefetch.global.L2 [%0];\n" ::"l"(rp + c));
            }
        }
        asm volatile("bar.sync 2, %0;\n" ::"n"(T5_ET) : "memory");
        mbar_wait(&tfull[acc], (tl / T5_ACC) & 1);
        tc_fence_after();
        const int m = m0 + q * 32 + lane;
        const double a_s = m < M ? sa[m] : 0.0;
        const uint32_t tacc = tmem + (uint32_t)(acc * BN) + ((uint32_t)(q * 32) << 16);
        float mx = 0.f;  // max |v| over this thread's (row, column half) of the tile
#pragma unroll 1
        for (int j = jh; j < jh + BN / 64; ++j) {
            uint32_t r[32];
            tmem_ld32(tacc + (uint32_t)(j * 32), r);
            if (j == jh + BN / 64 - 1) {
                // accumulator fully read: hand it back to the MMA issuer
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if (pair) mbar_arrive_cluster(&tempty[acc], 0);  // the pair's MMA waits on the leader's
                    else mbar_arrive(&tempty[acc]);
                }
            }
            const int nb = n0 + j * 32;
            if (m >= M || nb >= N) continue;
            if (ksplit > 1) {  // raw partial sums of this k slice
                int* wr = ws + ((size_t)sl * M + m) * N + nb;
                if (nb + 32 <= N && (N & 3) == 0) {  // the row's 128 B as 16-B stores (full sectors)
                    int4* w4 = reinterpret_cast<int4*>(wr);
#pragma unroll
                    for (int e = 0; e < 32; e += 4)
                        w4[e / 4] = make_int4((int)r[e] >> 8, (int)r[e + 1] >> 8, (int)r[e + 2] >> 8, (int)r[e + 3] >> 8);
                } else {
#pragma unroll
                    for (int e = 0; e < 32; ++e)
                        if (nb + e < N) wr[e] = (int)r[e] >> 8;
                }
                continue;
            }
            if (acc_dbg) {
#pragma unroll
                for (int e = 0; e < 32; ++e)
                    if (nb + e < N) acc_dbg[(size_t)m * N + nb + e] = (int)r[e] >> 8;
            }
            if (nb + 32 <= N) {
                epi_row32<EPI>(out, ldo, m, nb, r, a_s, swt + j * 32, mx);
            } else {
#pragma unroll
                for (int e = 0; e < 32; e += 2)
                    if (nb + e < N)
                        mx = fmaxf(mx, epi_store<EPI>(out, ldo, m, nb + e,
                                                      (double)((int)r[e] >> 8) * (a_s * swt[j * 32 + e]),
                                                      (double)((int)r[e + 1] >> 8) * (a_s * swt[j * 32 + e + 1]),
                                                      N));
            }
        }
        // partial row max for the next site's dynamic quantizer: slot (n tile, column half)
        if (pmax && ksplit == 1 && m < M) pmax[(size_t)m * pmax_ld + (t / mtp) * 2 + jh / (BN / 64)] = mx;
        asm volatile("bar.sync 2, %0;\n" ::"n"(T5_ET) : "memory");  // swt reuse
    }
}

template <int EPI>
QT_DEV void t5_epilogue(int ew0, int warp, int lane, uint32_t tmem, int units, int tiles, int mt_n, int M, int N,
                        const double* __restrict__ sa, const double* __restrict__ sw, double* sws,
                        void* __restrict__ out, int ldo, int* __restrict__ acc_dbg, int ksplit, int* __restrict__ ws,
                        float* __restrict__ pmax, int pmax_ld, uint64_t* tfull, uint64_t* tempty) {
    t5_epilogue_g<EPI>(ew0, warp, lane, tmem, blockIdx.x, gridDim.x, units, tiles, mt_n, 1, 0, M, N, sa, sw, sws, out,
                       ldo, acc_dbg, ksplit, ws, pmax, pmax_ld, tfull, tempty);
}

template <int EPI>
__global__ void __launch_bounds__(T5_THREADS, 1) k_gemm_tc05(const uint8_t* __restrict__ A, int lda,
                                                              const double* __restrict__ sa,
                                                              const uint8_t* __restrict__ W, int ldw,
                                                              const double* __restrict__ sw, int M, int N, int K,
                                                              void* __restrict__ out, int ldo,
                                                              int* __restrict__ acc_dbg, int ksplit,
                                                              int* __restrict__ ws, float* __restrict__ pmax,
                                                              int pmax_ld) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* pfull = reinterpret_cast<uint64_t*>(smem + T5Smem::bars);
    uint64_t* pempty = pfull + T5_PS;
    uint64_t* ifull = pempty + T5_PS;
    uint64_t* iempty = ifull + T5_IS;
    uint64_t* tfull = iempty + T5_IS;
    uint64_t* tempty = tfull + T5_ACC;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + T5_ACC);
    double* sws = reinterpret_cast<double*>(smem + T5Smem::swb);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int KB = K / 128;
    const int art = lda >> 4, wrt = ldw >> 4;  // row blocks per k-block (tiled, k-block-major)
    const int mt_n = (M + T5_BM - 1) / T5_BM, nt_n = (N + T5_BN - 1) / T5_BN;
    const int tiles = mt_n * nt_n;
    // work unit u = slice * tiles + tile; slice s covers k blocks [s*KB/ksplit, (s+1)*KB/ksplit).
    // ksplit > 1 (few tiles, e.g. decode batches of 17..256 tokens): raw int32 partial sums go
    // to ws[s][m][n] and k_splitk_epilogue reduces them in fixed order and applies the epilogue.
    const int units = tiles * ksplit;
    const int a_rbs_total = (M + 15) / 16, w_rbs_total = (N + 15) / 16;

    if (threadIdx.x == 0) {
        for (int s = 0; s < T5_PS; ++s) {
            mbar_init(&pfull[s], 1);
            mbar_init(&pempty[s], T5_CW);
        }
        for (int s = 0; s < T5_IS; ++s) {
            mbar_init(&ifull[s], T5_CW);
            mbar_init(&iempty[s], 1);
        }
        for (int s = 0; s < T5_ACC; ++s) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], T5_EWN);
        }
        mbar_fence_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                     "n"(T5_ACC * T5_BN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    // tile t -> (m tile fastest): CTAs running concurrently share weight tiles in L2
    if (warp == 0) {
        // ---------------- TMA producer
        if (lane == 0) {
            pdl_wait();  // activation codes come from the upstream kernel
            int it = 0;
            for (int u = blockIdx.x; u < units; u += gridDim.x) {
                const int t = u % tiles, sl = u / tiles;
                const int a_rb0 = (t % mt_n) * (T5_BM / 16), w_rb0 = (t / mt_n) * (T5_BN / 16);
                const int a_rbs = min(T5_BM / 16, a_rbs_total - a_rb0), w_rbs = min(T5_BN / 16, w_rbs_total - w_rb0);
                for (int kb = sl * KB / ksplit; kb < (sl + 1) * KB / ksplit; ++kb, ++it) {
                    const int s = it % T5_PS;
                    if (it >= T5_PS) mbar_wait(&pempty[s], ((it / T5_PS) - 1) & 1);
                    mbar_arrive_expect_tx(&pfull[s], (uint32_t)(a_rbs + w_rbs) * 1024u);
                    // one bulk copy per operand: the stage's row blocks are contiguous
                    bulk_g2s(smem + T5Smem::pa + (size_t)s * T5_PA, A + ((size_t)kb * art + a_rb0) * 1024,
                             (uint32_t)a_rbs * 1024u, &pfull[s]);
                    bulk_g2s(smem + T5Smem::pb + (size_t)s * T5_PB, W + ((size_t)kb * wrt + w_rb0) * 1024,
                             (uint32_t)w_rbs * 1024u, &pfull[s]);
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (one thread)
        if (lane == 0) {
            const uint32_t idesc = t5_idesc();
            int it = 0, tl = 0;
            for (int u = blockIdx.x; u < units; u += gridDim.x, ++tl) {
                const int sl = u / tiles, kb0 = sl * KB / ksplit, kb1 = (sl + 1) * KB / ksplit;
                const int acc = tl % T5_ACC;
                if (tl >= T5_ACC) mbar_wait(&tempty[acc], ((tl / T5_ACC) - 1) & 1);
                tc_fence_after();
                const uint32_t tacc = tmem + (uint32_t)(acc * T5_BN);
                for (int kb = kb0; kb < kb1; ++kb, ++it) {
                    const int s = it % T5_IS;
                    mbar_wait(&ifull[s], (it / T5_IS) & 1);
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(smem + T5Smem::ia + (size_t)s * T5_IA);
                    const uint32_t b0 = smem_u32(smem + T5Smem::ib + (size_t)s * T5_IB);
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        mma_i8(tacc, umma_desc_sw128(a0 + 32 * k), umma_desc_sw128(b0 + 32 * k), idesc,
                               (kb != kb0) || (k != 0));
                    mma_commit(&iempty[s]);
                }
                mma_commit(&tfull[acc]);
            }
        }
        __syncwarp();
    } else if (warp < T5_EW0) {
        // ---------------- converters: packed int4 -> swizzled int8 (T5_CT threads); every
        // thread first loads all of its packed chunks of the stage, then unpacks and stores
        constexpr int CA = (T5_BM * 4) / T5_CT, CB = (T5_BN * 4) / T5_CT;
        const int ct = threadIdx.x - 64;
        int it = 0;
        for (int u = blockIdx.x; u < units; u += gridDim.x) {
            const int sl = u / tiles;
            for (int kb = sl * KB / ksplit; kb < (sl + 1) * KB / ksplit; ++kb, ++it) {
                const int ps = it % T5_PS, is = it % T5_IS;
                mbar_wait(&pfull[ps], (it / T5_PS) & 1);
                const uint8_t* pa = smem + T5Smem::pa + (size_t)ps * T5_PA;
                const uint8_t* pb = smem + T5Smem::pb + (size_t)ps * T5_PB;
                // rows past the valid row blocks convert stale bytes; never stored
                uint4 wa[CA], wb[CB];
#pragma unroll
                for (int i = 0; i < CA; ++i) {
                    const int c = ct + T5_CT * i;
                    wa[i] = *reinterpret_cast<const uint4*>(pa + (size_t)(c >> 2) * T5_BKB + (c & 3) * 16);
                }
#pragma unroll
                for (int i = 0; i < CB; ++i) {
                    const int c = ct + T5_CT * i;
                    wb[i] = *reinterpret_cast<const uint4*>(pb + (size_t)(c >> 2) * T5_BKB + (c & 3) * 16);
                }
                // the packed stage is in registers: order these generic-proxy reads before the
                // TMA (async proxy) refill of the stage, then release it
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(&pempty[ps]);
                if (it >= T5_IS) mbar_wait(&iempty[is], ((it / T5_IS) - 1) & 1);
                uint8_t* ia = smem + T5Smem::ia + (size_t)is * T5_IA;
                uint8_t* ib = smem + T5Smem::ib + (size_t)is * T5_IB;
#pragma unroll
                for (int i = 0; i < CA; ++i) {
                    const int c = ct + T5_CT * i;
                    store_converted(wa[i], ia, c >> 2, c & 3);
                }
#pragma unroll
                for (int i = 0; i < CB; ++i) {
                    const int c = ct + T5_CT * i;
                    store_converted(wb[i], ib, c >> 2, c & 3);
                }
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(&ifull[is]);
            }
        }
    } else {
        t5_epilogue<EPI>(T5_EW0, warp, lane, tmem, units, tiles, mt_n, M, N, sa, sw, sws, out, ldo, acc_dbg, ksplit, ws,
                         pmax, pmax_ld, tfull, tempty);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(T5_ACC * T5_BN));
    }
}

// ============================================================== int8-operand variant
// Both operands arrive as int8 (16 x the int4 code, k in natural order) row-major in
// HBM: the weights converted once at load (k_w4t_to_i8), the activations written by
// the quantizer next to the packed codes.  TMA tensor loads (SWIZZLE_128B) put them
// straight into the UMMA canonical K-major layout, so there are no converter warps:
//   warp 0      TMA producer (2D tensor loads, 4-stage 48 KB ring)
//   warp 1      TMEM allocator + MMA issuer (same UMMA as k_gemm_tc05)
//   warps 2..9  epilogue (t5_epilogue)
// stages of the int8 TMA ring: 4 x 48 KB at N = 256; 6 x 32 KB at N = 128 (decode batches: more
// CTAs, each with as many bytes in flight)
template <int BN>
constexpr int t8_stages() { return BN == 256 ? 4 : 6; }
constexpr int T8_EW0 = 2;
constexpr int T8_THREADS = (T8_EW0 + T5_EWN) * 32;

template <int BN>
struct T8Smem {
    static constexpr int S = t8_stages<BN>();
    static constexpr size_t ia = 0;
    static constexpr size_t ib = ia + (size_t)S * T5_IA;
    static constexpr size_t swb = ib + (size_t)S * BN * 128;
    static constexpr size_t bars = swb + (size_t)T5_ACC * BN * 8;
    static constexpr size_t total = bars + 256;
};
template <int BN>
constexpr uint32_t t8_idesc() {
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(T5_BM >> 4) << 24);
}

QT_DEV void tma_load_2d(void* dst, const CUtensorMap* tm, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
            smem_u32(dst)),
        "l"(tm), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

QT_DEV uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
    return r;
}

QT_DEV void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

template <int EPI, int BN = T5_BN>
__global__ void __launch_bounds__(T8_THREADS, 1) k_gemm_tc05_i8(const __grid_constant__ CUtensorMap tmA,
                                                                 const __grid_constant__ CUtensorMap tmB,
                                                                 const double* __restrict__ sa,
                                                                 const double* __restrict__ sw, int M, int N, int K,
                                                                 void* __restrict__ out, int ldo,
                                                                 int* __restrict__ acc_dbg, float* __restrict__ pmax,
                                                                 int pmax_ld, int ksplit, int* __restrict__ ws) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + T8Smem<BN>::bars);
    uint64_t* empty = full + T8Smem<BN>::S;
    uint64_t* tfull = empty + T8Smem<BN>::S;
    uint64_t* tempty = tfull + T5_ACC;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + T5_ACC);
    double* sws = reinterpret_cast<double*>(smem + T8Smem<BN>::swb);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int KB = K / 128;
    const int mt_n = (M + T5_BM - 1) / T5_BM, nt_n = (N + BN - 1) / BN;
    const int tiles = mt_n * nt_n;
    // work unit u: tile u % tiles, k slice u / tiles (split-K for decode batches, ksplit > 1:
    // int32 partials to ws, reduced in fixed order by k_splitk_epilogue)
    const int units = tiles * ksplit, kbs = (KB + ksplit - 1) / ksplit;
    if (threadIdx.x == 0) {
        for (int s = 0; s < T8Smem<BN>::S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < T5_ACC; ++s) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], T5_EWN);
        }
        mbar_fence_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                     "n"(T5_ACC * BN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (warp == 0) {
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmA) : "memory");
            asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmB) : "memory");
            pdl_wait();  // activation codes come from the upstream kernel
            int it = 0;
            for (int u = blockIdx.x; u < units; u += gridDim.x) {
                const int t = u % tiles, k0 = (u / tiles) * kbs, k1 = min(KB, k0 + kbs);
                const int m0 = (t % mt_n) * T5_BM, n0 = (t / mt_n) * BN;
                for (int kb = k0; kb < k1; ++kb, ++it) {
                    const int s = it % T8Smem<BN>::S;
                    if (it >= T8Smem<BN>::S) mbar_wait(&empty[s], ((it / T8Smem<BN>::S) - 1) & 1);
                    mbar_arrive_expect_tx(&full[s], (uint32_t)(T5_IA + (BN * 128)));
                    tma_load_2d(smem + T8Smem<BN>::ia + (size_t)s * T5_IA, &tmA, kb * 128, m0, &full[s]);
                    tma_load_2d(smem + T8Smem<BN>::ib + (size_t)s * (BN * 128), &tmB, kb * 128, n0, &full[s]);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t idesc = t8_idesc<BN>();
            int it = 0, tl = 0;
            for (int u = blockIdx.x; u < units; u += gridDim.x, ++tl) {
                const int k0 = (u / tiles) * kbs, k1 = min(KB, k0 + kbs);
                const int acc = tl % T5_ACC;
                if (tl >= T5_ACC) mbar_wait(&tempty[acc], ((tl / T5_ACC) - 1) & 1);
                tc_fence_after();
                const uint32_t tacc = tmem + (uint32_t)(acc * BN);
                for (int kb = k0; kb < k1; ++kb, ++it) {
                    const int s = it % T8Smem<BN>::S;
                    mbar_wait(&full[s], (it / T8Smem<BN>::S) & 1);
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(smem + T8Smem<BN>::ia + (size_t)s * T5_IA);
                    const uint32_t b0 = smem_u32(smem + T8Smem<BN>::ib + (size_t)s * (BN * 128));
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        mma_i8(tacc, umma_desc_sw128(a0 + 32 * k), umma_desc_sw128(b0 + 32 * k), idesc,
                               (kb != k0) || (k != 0));
                    mma_commit(&empty[s]);
                }
                mma_commit(&tfull[acc]);
            }
        }
        __syncwarp();
    } else {
        t5_epilogue_g<EPI, BN>(T8_EW0, warp, lane, tmem, blockIdx.x, gridDim.x, units, tiles, mt_n, 1, 0, M, N, sa, sw,
                           sws, out, ldo, ksplit > 1 ? nullptr : acc_dbg, ksplit, ws, pmax, pmax_ld, tfull, tempty);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(T5_ACC * BN));
    }
}

// ============================================================== 2-SM (CTA pair) variant
// A cluster of two CTAs on one TPC computes a 256 x 256 tile with tcgen05.mma.cta_group::2
// (M = 256): each CTA stages its own 128 activation rows and HALF of the 256 weight rows, so
// per SM the operand ingress -- TMA writes plus UMMA shared-memory reads -- is two thirds of
// the single-CTA 128 x 256 tile's (which saturates shared-memory bandwidth, not the tensor
// pipe).  Both CTAs' TMA loads complete on the leader's full barrier; the leader alone issues
// the MMAs, whose commits arrive (multicast) on both CTAs' stage / accumulator barriers; each
// CTA's epilogue reads its own 128 TMEM lanes and arrives on the leader's accumulator-empty
// barrier.
constexpr int T2_S = 6;                                   // stages (32 KB per CTA each)
constexpr int T2_IA = 128 * 128, T2_IB = 128 * 128;       // per-CTA bytes per stage: A half, B half
constexpr int T2_THREADS = (T8_EW0 + T5_EWN) * 32;

struct T2Smem {
    static constexpr size_t ia = 0;
    static constexpr size_t ib = ia + (size_t)T2_S * T2_IA;
    static constexpr size_t swb = ib + (size_t)T2_S * T2_IB;
    static constexpr size_t bars = swb + (size_t)T5_ACC * T5_BN * 8;
    static constexpr size_t total = bars + 256;
};

// InstrDescriptor for M = 256 (cta_group::2), N = 256, s8 x s8 -> s32, K-major
constexpr uint32_t t2_idesc() {
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(T5_BN >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
}

QT_DEV uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}

QT_DEV void tma_load_2d_pair(void* dst, const CUtensorMap* tm, int c0, int c1, uint32_t leader_bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3}], [%4];\n" ::"r"(smem_u32(dst)),
        "l"(tm), "r"(c0), "r"(c1), "r"(leader_bar)
        : "memory");
}

QT_DEV void mma_i8_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accum) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
        : "memory");
}

QT_DEV void mma_commit_pair(uint64_t* bar) {  // arrive on the barrier at this offset in both CTAs
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
            smem_u32(bar)),
        "h"((uint16_t)0x3)
        : "memory");
}

template <int EPI>
__global__ void __launch_bounds__(T2_THREADS, 1) k_gemm_tc05_i8x2(const __grid_constant__ CUtensorMap tmA,
                                                                   const __grid_constant__ CUtensorMap tmB,
                                                                   const double* __restrict__ sa,
                                                                   const double* __restrict__ sw, int M, int N,
                                                                   int K, void* __restrict__ out, int ldo,
                                                                   int* __restrict__ acc_dbg,
                                                                   float* __restrict__ pmax, int pmax_ld, int ksplit,
                                                                   int* __restrict__ ws) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + T2Smem::bars);
    uint64_t* empty = full + T2_S;
    uint64_t* tfull = empty + T2_S;
    uint64_t* tempty = tfull + T5_ACC;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + T5_ACC);
    double* sws = reinterpret_cast<double*>(smem + T2Smem::swb);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rank = (int)cluster_rank();
    const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
    const int KB = K / 128;
    const int mtp = (M + 255) / 256, nt_n = (N + T5_BN - 1) / T5_BN;
    const int tiles = mtp * nt_n;
    // work unit u: tile u % tiles, k slice u / tiles (split-K, ksplit > 1: int32 partials to ws,
    // reduced in fixed order by k_splitk_epilogue)
    const int units = tiles * ksplit, kbs = (KB + ksplit - 1) / ksplit;
    if (threadIdx.x == 0) {
        for (int s = 0; s < T2_S; ++s) {
            mbar_init(&full[s], 1);   // the leader's arrive.expect_tx (both CTAs' bytes)
            mbar_init(&empty[s], 1);  // the leader's multicast MMA commit
        }
        for (int s = 0; s < T5_ACC; ++s) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], 2 * T5_EWN);  // both CTAs' epilogue warps (leader's copy is used)
        }
        mbar_fence_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                     "n"(T5_ACC * T5_BN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();  // both CTAs' barriers and TMEM exist before any cross-CTA signal
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (warp == 0) {
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmA) : "memory");
            asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmB) : "memory");
            pdl_wait();  // activation codes come from the upstream kernel
            int it = 0;
            for (int u = cid; u < units; u += ncl) {
                const int t = u % tiles, k0 = (u / tiles) * kbs, k1 = min(KB, k0 + kbs);
                const int m0 = (t % mtp) * 256 + rank * 128, n0 = (t / mtp) * T5_BN + rank * 128;
                for (int kb = k0; kb < k1; ++kb, ++it) {
                    const int s = it % T2_S;
                    if (it >= T2_S) mbar_wait(&empty[s], ((it / T2_S) - 1) & 1);
                    if (rank == 0) mbar_arrive_expect_tx(&full[s], (uint32_t)(2 * (T2_IA + T2_IB)));
                    const uint32_t lb = mapa_shared(smem_u32(&full[s]), 0);
                    tma_load_2d_pair(smem + T2Smem::ia + (size_t)s * T2_IA, &tmA, kb * 128, m0, lb);
                    tma_load_2d_pair(smem + T2Smem::ib + (size_t)s * T2_IB, &tmB, kb * 128, n0, lb);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && rank == 0) {
            const uint32_t idesc = t2_idesc();
            int it = 0, tl = 0;
            for (int u = cid; u < units; u += ncl, ++tl) {
                const int k0 = (u / tiles) * kbs, k1 = min(KB, k0 + kbs);
                const int acc = tl % T5_ACC;
                if (tl >= T5_ACC) mbar_wait(&tempty[acc], ((tl / T5_ACC) - 1) & 1);
                tc_fence_after();
                const uint32_t tacc = tmem + (uint32_t)(acc * T5_BN);
                for (int kb = k0; kb < k1; ++kb, ++it) {
                    const int s = it % T2_S;
                    mbar_wait(&full[s], (it / T2_S) & 1);
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(smem + T2Smem::ia + (size_t)s * T2_IA);
                    const uint32_t b0 = smem_u32(smem + T2Smem::ib + (size_t)s * T2_IB);
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        mma_i8_pair(tacc, umma_desc_sw128(a0 + 32 * k), umma_desc_sw128(b0 + 32 * k), idesc,
                                    (kb != k0) || (k != 0));
                    mma_commit_pair(&empty[s]);
                }
                mma_commit_pair(&tfull[acc]);
            }
        }
        __syncwarp();
    } else {
        t5_epilogue_g<EPI>(T8_EW0, warp, lane, tmem, cid, ncl, units, tiles, mtp, 2, rank, M, N, sa, sw, sws, out,
                           ldo, ksplit > 1 ? nullptr : acc_dbg, ksplit, ws, pmax, pmax_ld, tfull, tempty, true);
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();  // no CTA leaves while its peer may still signal into it
    if (warp == 1) {
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(T5_ACC * T5_BN));
    }
}

// packed tiled int4 (w4t layout, rows_pad rows) -> row-major int8 [rows_pad x K], 16 x code,
// k in natural order (the int8-operand GEMM's weight copy)
__global__ void k_w4t_to_i8(const uint8_t* __restrict__ tiled, int rows_pad, int K, int8_t* __restrict__ out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;  // one packed byte pair-of-k
    const long long nb = (long long)rows_pad * (K / 2);
    if (i >= nb) return;
    const int row = (int)(i / (K / 2)), kb = (int)(i % (K / 2));
    const uint8_t b = tiled[w4t_offset(row, kb, rows_pad)];
    char2 v;
    v.x = (char)(uint8_t)(b << 4);
    v.y = (char)(uint8_t)(b & 0xF0);
    reinterpret_cast<char2*>(out)[i] = v;
}

// Split-K reduction + epilogue: y = (sum over slices, fixed order) * s_a[m] * s_w[n],
// then the same epilogue as the row-wise path.  One thread per output pair.
template <int EPI>
__global__ void __launch_bounds__(256) k_splitk_epilogue(const int* __restrict__ ws, int ksplit, int M, int N,
                                                         const double* __restrict__ sa, const double* __restrict__ sw,
                                                         void* __restrict__ out, int ldo, int* __restrict__ acc_dbg) {
    pdl_launch_dependents();
    pdl_wait();
    const long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * 2;
    if (i >= (long long)M * N) return;
    const int m = (int)(i / N), n = (int)(i % N);
    int s0 = 0, s1 = 0;
    for (int s = 0; s < ksplit; ++s) {
        const int* p = ws + ((size_t)s * M + m) * N + n;
        s0 += p[0];
        if (n + 1 < N) s1 += p[1];
    }
    if (acc_dbg) {
        acc_dbg[(size_t)m * N + n] = s0;
        if (n + 1 < N) acc_dbg[(size_t)m * N + n + 1] = s1;
    }
    const double a_s = sa[m];
    epi_store<EPI>(out, ldo, m, n, (double)s0 * (a_s * sw[n]), n + 1 < N ? (double)s1 * (a_s * sw[n + 1]) : 0.0, N);
}

}  // namespace qt

extern "C" int qt_tc05_splitk(int M, int N, int K) {
    // slices so that tiles x slices covers the SMs, >= 4 k blocks per slice
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int tiles = ((N + qt::T5_BN - 1) / qt::T5_BN) * ((M + qt::T5_BM - 1) / qt::T5_BM);
    const int KB = K / 128;
    if (tiles >= sms / 2) return 1;
    int s = (sms + tiles - 1) / tiles;
    s = std::min(s, std::max(1, KB / 4));
    return std::max(1, s);
}

extern "C" int qt_launch_w4a4_tc05(int epi, const uint8_t* A, int lda, const double* sa, const uint8_t* W, int ldw,
                                   const double* sw, int M, int N, int K, void* out, int ldo, int* acc_dbg,
                                   int* ws, cudaStream_t st) {
    return qt_launch_w4a4_tc05_ex(epi, A, lda, sa, W, ldw, sw, M, N, K, out, ldo, acc_dbg, ws, nullptr, 0, nullptr, st);
}

// pmax (may be null): per-row partial max |v| of the fp32 outputs, pmax[m * pmax_ld + p],
// p < *n_part = 2 x N tiles; *n_part = 0 when this launch produced none (split-K path).
extern "C" int qt_launch_w4a4_tc05_ex(int epi, const uint8_t* A, int lda, const double* sa, const uint8_t* W,
                                      int ldw, const double* sw, int M, int N, int K, void* out, int ldo,
                                      int* acc_dbg, int* ws, float* pmax, int pmax_ld, int* n_part,
                                      cudaStream_t st) {
    using namespace qt;
    if (n_part) *n_part = 0;
    if (M <= 0) return 0;
    if (K % 128 || lda % 16 || ldw % 16 || M > lda || N > ldw) return -1;  // lda/ldw = padded rows
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int tiles = ((N + T5_BN - 1) / T5_BN) * ((M + T5_BM - 1) / T5_BM);
    const int ksplit = ws ? qt_tc05_splitk(M, N, K) : 1;
    const dim3 grid(std::min(tiles * ksplit, sms));
    const int parts = 2 * ((N + T5_BN - 1) / T5_BN);
    if (pmax && (ksplit > 1 || parts > pmax_ld)) pmax = nullptr;
    if (pmax && n_part) *n_part = parts;
    const size_t smem = T5Smem::total;
#define QT_T5(E)                                                                                                \
    do {                                                                                                        \
        auto kfn = k_gemm_tc05<E>;                                                                              \
        cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);                      \
        int rc = launch_pdl(kfn, grid, dim3(T5_THREADS), smem, st, A, lda, sa, W, ldw, sw, M, N, K, out, ldo,   \
                            ksplit > 1 ? nullptr : acc_dbg, ksplit, ws, pmax, pmax_ld);                          \
        if (rc || ksplit == 1) return rc;                                                                       \
        const long long pairs = ((long long)M * N + 1) / 2;                                                     \
        return launch_pdl(k_splitk_epilogue<E>, dim3((unsigned)((pairs + 255) / 256)), dim3(256), 0, st,      \
                          (const int*)ws, ksplit, M, N, sa, sw, out, ldo, acc_dbg);                              \
    } while (0)
    switch (epi) {
        case QT_EPI_STORE: QT_T5(QT_EPI_STORE);
        case QT_EPI_RESADD: QT_T5(QT_EPI_RESADD);
        case QT_EPI_SILU: QT_T5(QT_EPI_SILU);
        case QT_EPI_SWIGLU: QT_T5(QT_EPI_SWIGLU);
    }
#undef QT_T5
    return -1;
}

// ---------------------------------------------------------------- int8-operand launcher
typedef CUresult (*qt_encode_fn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static qt_encode_fn qt_encoder() {
    static qt_encode_fn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return (qt_encode_fn) nullptr;
        return reinterpret_cast<qt_encode_fn>(p);
    }();
    return fn;
}

// int8 row-major [rows x K] with row stride ld bytes; box 128 k x box_rows rows, SW128
static int qt_tmap_i8(CUtensorMap* tm, const int8_t* base, int rows, int K, int ld, int box_rows) {
    qt_encode_fn enc = qt_encoder();
    if (!enc) return -1;
    const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)ld};
    const cuuint32_t box[2] = {128, (cuuint32_t)box_rows};
    const cuuint32_t estr[2] = {1, 1};
    return enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int8_t*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS
               ? 0
               : -1;
}

extern "C" int qt_launch_w4t_to_i8(const uint8_t* tiled, int rows_pad, int K, int8_t* out, cudaStream_t st) {
    const long long nb = (long long)rows_pad * (K / 2);
    if (nb <= 0) return 0;
    qt::k_w4t_to_i8<<<(unsigned)((nb + 255) / 256), 256, 0, st>>>(tiled, rows_pad, K, out);
    return (int)cudaGetLastError();
}

// A8: int8 activations [>= M rows x K], row stride lda8; W8: int8 weights [w_rows x K], stride ldw8.
// M >= 8192: the 2-SM (CTA pair, cta_group::2) kernel on 256 x 256 tiles; else the single-CTA one.
// k slices of the single-CTA kernel (decode batches, M <= 512): only when the tiles fill
// less than half the SMs (the N = d_model projections), as many slices as keep one wave,
// at most 6 and >= 4 k blocks each -- measured per shape and slice count at M = 32..256
// (tools/bench_decode_gemm.py): splitting the wide projections only added the int32
// partials' round trip.  ks_force > 0 overrides (measurement).
#ifndef QT_I8_NARROW_M
#define QT_I8_NARROW_M 256  // up to this many tokens the single-CTA kernel uses N = 128 tiles (A/B:
                           // C5 decode GEMM class 2.29 -> 2.04 ms/step at B = 64, 3.28 -> 2.94 at 256)
#endif
// tile width of the single-CTA int8 kernel: 128 for decode batches (twice the CTAs streaming
// the weights, 6 stages in flight each), 256 for prefill
static int qt_i8_bn(int M) { return M <= QT_I8_NARROW_M ? 128 : qt::T5_BN; }

static int qt_tc05_i8_single_splitk(int M, int N, int K, int ks_force = 0) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int KB = K / 128, bn = qt_i8_bn(M);
    const int tiles = ((M + qt::T5_BM - 1) / qt::T5_BM) * ((N + bn - 1) / bn);
    auto eff = [&](int ks) {  // slices actually formed (no empty slice)
        ks = std::max(1, std::min(ks, KB));
        const int kbs = (KB + ks - 1) / ks;
        return (KB + kbs - 1) / kbs;
    };
    if (ks_force > 0) return eff(ks_force);
    if (M > 512 || 2 * tiles > sms) return 1;
    return eff(std::min({6, sms / tiles, KB / 4}));
}

int qt_tc05_i8_splitk(int M, int N, int K) {
    // the 2-SM kernel's k slices: enough work units for every CTA pair, >= 4 k blocks per slice
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    if (M < 8192) return qt_tc05_i8_single_splitk(M, N, K);
    const int tiles = ((M + 255) / 256) * ((N + qt::T5_BN - 1) / qt::T5_BN);
    const int pairs = sms / 2, KB = K / 128;
    if (tiles >= pairs) return 1;
    const int ks = std::max(1, std::min((pairs + tiles - 1) / tiles, KB / 4));
    const int kbs = (KB + ks - 1) / ks;
    return (KB + kbs - 1) / kbs;  // no empty slice
}

extern "C" int qt_launch_w4a4_tc05_i8_ex(int epi, const int8_t* A8, int lda8, const double* sa, const int8_t* W8,
                                         int w_rows, int ldw8, const double* sw, int M, int N, int K, void* out,
                                         int ldo, int* acc_dbg, float* pmax, int pmax_ld, int* n_part, int* ws,
                                         int flags, cudaStream_t st);

extern "C" int qt_launch_w4a4_tc05_i8(int epi, const int8_t* A8, int lda8, const double* sa, const int8_t* W8,
                                      int w_rows, int ldw8, const double* sw, int M, int N, int K, void* out, int ldo,
                                      int* acc_dbg, float* pmax, int pmax_ld, int* n_part, int* ws, cudaStream_t st) {
    return qt_launch_w4a4_tc05_i8_ex(epi, A8, lda8, sa, W8, w_rows, ldw8, sw, M, N, K, out, ldo, acc_dbg, pmax,
                                     pmax_ld, n_part, ws, 0, st);
}

// flags bit 0: the single-CTA 128 x 256 kernel at any M (A/B measurements, qt_w4a4_gemm_i8);
// bits 8..15: k-slice count override of the single-CTA kernel (needs ws; measurement)
extern "C" int qt_launch_w4a4_tc05_i8_ex(int epi, const int8_t* A8, int lda8, const double* sa, const int8_t* W8,
                                         int w_rows, int ldw8, const double* sw, int M, int N, int K, void* out,
                                         int ldo, int* acc_dbg, float* pmax, int pmax_ld, int* n_part, int* ws,
                                         int flags, cudaStream_t st) {
    using namespace qt;
    const bool force_single = flags & 1;
    const int ks_force = (flags >> 8) & 0xFF;
    if (n_part) *n_part = 0;
    if (M <= 0) return 0;
    if (K % 128 || lda8 % 16 || ldw8 % 16 || N > w_rows) return -1;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    // CTA pairs only pay for the largest token counts (measured, tools/bench_gemm.py: pair 2880 vs
    // single 2774 TOPS at 8192^3, but 1582 vs 2004 on the 7B QKV GEMM at M = 1896)
    const bool pair = M >= 8192 && !force_single && ks_force == 0;
    const int bn = pair ? T5_BN : qt_i8_bn(M);
    const int nt_n = (N + bn - 1) / bn;
    const int parts = 2 * nt_n;
    if (pmax && parts > pmax_ld) pmax = nullptr;
    if (pmax && n_part) *n_part = parts;
    CUtensorMap ta, tb;
    if (qt_tmap_i8(&ta, A8, M, K, lda8, T5_BM) || qt_tmap_i8(&tb, W8, w_rows, K, ldw8, pair ? 128 : bn))
        return -2;
    if (pair) {
        const int tiles = ((M + 255) / 256) * nt_n;
        const int ksplit = ws ? qt_tc05_i8_splitk(M, N, K) : 1;
        if (ksplit > 1) {
            pmax = nullptr;
            if (n_part) *n_part = 0;
        }
        const dim3 grid(2 * std::min(tiles * ksplit, sms / 2));
        const size_t smem = T2Smem::total;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = grid;
        cfg.blockDim = dim3(T2_THREADS);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = g_pdl_block ? 1 : 2;
        g_pdl_block = false;
#define QT_T2(E)                                                                                                 \
    do {                                                                                                         \
        auto kfn = k_gemm_tc05_i8x2<E>;                                                                          \
        cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);                       \
        int rc = (int)cudaLaunchKernelEx(&cfg, kfn, ta, tb, sa, sw, M, N, K, out, ldo, acc_dbg, pmax, pmax_ld,   \
                                         ksplit, ws);                                                            \
        if (rc || ksplit == 1) return rc;                                                                        \
        const long long pairs2 = ((long long)M * N + 1) / 2;                                                     \
        return launch_pdl(k_splitk_epilogue<E>, dim3((unsigned)((pairs2 + 255) / 256)), dim3(256), 0, st,       \
                          (const int*)ws, ksplit, M, N, sa, sw, out, ldo, acc_dbg);                               \
    } while (0)
        switch (epi) {
            case QT_EPI_STORE: QT_T2(QT_EPI_STORE);
            case QT_EPI_RESADD: QT_T2(QT_EPI_RESADD);
            case QT_EPI_SILU: QT_T2(QT_EPI_SILU);
            case QT_EPI_SWIGLU: QT_T2(QT_EPI_SWIGLU);
        }
#undef QT_T2
        return -1;
    }
    const int ksplit = ws ? qt_tc05_i8_single_splitk(M, N, K, ks_force) : 1;
    if (ksplit > 1) {
        pmax = nullptr;
        if (n_part) *n_part = 0;
    }
    const int units = ((M + T5_BM - 1) / T5_BM) * nt_n * ksplit;
    const dim3 grid(std::min(units, sms));
    const size_t smem = bn == 128 ? T8Smem<128>::total : T8Smem<T5_BN>::total;
#define QT_T8(E)                                                                                                 \
    do {                                                                                                         \
        auto kfn = bn == 128 ? k_gemm_tc05_i8<E, 128> : k_gemm_tc05_i8<E, T5_BN>;                                \
        cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);                       \
        int rc = launch_pdl(kfn, grid, dim3(T8_THREADS), smem, st, ta, tb, sa, sw, M, N, K, out, ldo, acc_dbg,    \
                            pmax, pmax_ld, ksplit, ws);                                                          \
        if (rc || ksplit == 1) return rc;                                                                        \
        const long long pairs1 = ((long long)M * N + 1) / 2;                                                     \
        return launch_pdl(k_splitk_epilogue<E>, dim3((unsigned)((pairs1 + 255) / 256)), dim3(256), 0, st,       \
                          (const int*)ws, ksplit, M, N, sa, sw, out, ldo, acc_dbg);                               \
    } while (0)
    switch (epi) {
        case QT_EPI_STORE: QT_T8(QT_EPI_STORE);
        case QT_EPI_RESADD: QT_T8(QT_EPI_RESADD);
        case QT_EPI_SILU: QT_T8(QT_EPI_SILU);
        case QT_EPI_SWIGLU: QT_T8(QT_EPI_SWIGLU);
    }
#undef QT_T8
    return -1;
}
