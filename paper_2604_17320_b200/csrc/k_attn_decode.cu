// k_attn_decode.cu -- K6 decode attention over the paged int4 KV cache, with the decode
// step's RoPE + K5 KV quantize-and-append fused in.
//
// Reference: decode_step (model.cpp:455-562): q/k RoPE at next_position (model.cpp:494-495),
// kv_quantize of the new K / V rows appended to the cache (model.cpp:499-501,
// quant.cpp:117-119), then per query head an unmasked max-subtracted softmax of
// q . k^ / sqrt(d_head) over every cached row and out = sum_j p_j v^_j (model.cpp:515-535).
//
// B200 layout of the work (k_attn_dec_w): one warp per (page, kv head, sequence) -- G <= 2:
// a CTA holds up to 4 kv heads of one page; G > 2 (GQA, C4): a CTA is one kv head of one
// page with one warp per pair of query heads, sharing the page's V copy -- so every cached
// K / V byte is read from HBM once.  Each (sequence, query head, page) leaves one (max, sum,
// unnormalised o) partial; k_attn_merge_quant merges the pages in fixed order and quantizes
// the attn_out site.
#include <algorithm>
#include <type_traits>

#include "qt_common.cuh"
#include "qt_kernels.h"

namespace qt {

constexpr int AD_MAX_G = 8;  // query heads per kv head

// ---------------------------------------------------------------- K6 on integer tensor cores
// One WARP per (page, kv head, sequence) for G <= 2 (a CTA is up to 4 kv heads of the same
// page, no block barrier), one warp per (page, pair of query heads) for G > 2 (a CTA is one kv
// head, its warps share the V copy; two block barriers).  The page's V code block and scales
// arrive by cp.async.bulk into shared memory; its K codes go straight into the MMA lanes'
// registers (each warp load instruction covers 8 whole 64 B rows).  Both are issued before the
// programmatic-dependency wait.
//
// Both products run as exact integer MMAs (mma.sync m16n8k32 s8.s8.s32) on the codes as
// stored: the fp32 operand (q, then p * s_v) is written as a fixed-point integer Q =
// rint(x * 2^F) (|Q| < 2^30, F from the head's max |x|) in four balanced base-256 digits, one
// MMA column per digit: S = sum_d Q_d * c_d is exact in int32 per digit, and a score's only
// roundings are the fixed-point step (2^-31 of the head's max |q|) and the final fp32 one --
// tighter than an fp32 dot product (round 2's fp32 CUDA-core kernel, replaced: C5 B = 256
// attention 5.32 -> 2.53 ms/step, C4 0.487 -> 0.412).
//   QK: A = K codes (16 keys x 32 dims, 16 * code in s8 as unpack_x16 gives), B = q digits.
//   PV: A = V^T (16 channels x 32 keys), built by a 4 x 4 byte transpose of 4 keys' code
//       words (PRMT) then unpack_x16; B = (p * s_v) digits.
// Balanced digits of Q: U = Q + 0x80808080 has bytes d_j + 128, so (U ^ 0x80808080) holds
// the four signed digits d_j directly.  The exact integer digit-pair sums are recombined and
// rounded once in fp32 (hi * 2^16 + lo by one FMA).
constexpr int AW_MAXW = 4;  // warps (kv heads) per CTA
// Two register budgets (A/B at C2 / C5 B = 64 / C5 B = 256, decode attention chain ms per
// step): 96 registers, 5 CTAs per SM by shared memory -- 0.361 / 0.859 / 2.797; capped at 80
// for 6 CTAs per SM -- 0.387 / 0.842 / 2.537 (7: 0.412 / 0.873 / 2.535).  Latency decides a
// grid of less than one full wave, residency a larger one.
constexpr int AW_MINB_WIDE = 6;
// (G > 2 splits the heads over warps: one warp running all G = 7 heads of C4 -- 4 MMA column
// tiles and 7 softmaxes serially -- measured 0.613 ms/step against 0.412 split)
template <int DH, int HW>
struct AwSmem {  // the page's V slice (shared by the warps of one kv head) + per-warp scratch
    static constexpr int CB = kPage * (DH / 2);   // (the K codes go straight to registers)
    static constexpr size_t vc = 0, ks = CB, vs = ks + kPage * 4, bar = vs + kPage * 4;
    static constexpr size_t sh_total = (bar + 8 + 127) / 128 * 128;
    static constexpr size_t sc = 0;                      // [HW][64] scores
    static constexpr size_t ql = sc + HW * kPage * 4;    // [HW][4 digits][DH] q digits, MMA-B order
    static constexpr size_t wl = ql + HW * 4 * DH;       // [HW][4 digits][64] (p * s_v) digits
    static constexpr size_t w_total = (wl + HW * 4 * kPage + 127) / 128 * 128;
};
QT_DEV uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, %3;\n" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
    return r;
}
// position of dim d (word d / 8, nibble d % 8) in a digit row: the MMA-B fragment's bytes
// (even nibbles of a word, then odd ones) contiguous
QT_DEV int aw_qpos(int d) { return (d & ~7) | ((d & 1) << 2) | ((d >> 1) & 3); }
// position of key k = 32 s + 16 h + t + 4 i in a digit row: 32 s + 16 h + 4 t + i
QT_DEV int aw_kpos(int k) { return (k & 48) | ((k & 3) << 2) | ((k >> 2) & 3); }
// fixed-point exponent: |x| * 2^F < 2^30 for every |x| <= mx (F <= 100: 2^F and the
// recombination factor 2^-(F + 4) stay normal fp32 numbers)
QT_DEV int aw_fexp(float mx) {
    if (!(mx > 0.f)) return 0;
    int e;
    frexpf(mx, &e);
    return min(30 - e, 100);
}
QT_DEV float aw_pow2(int e) { return __int_as_float((127 + e) << 23); }  // 2^e, -126 <= e <= 127
// the four signed digits of rint(x * 2^F) (x * 2^F is exact: a power-of-two scaling)
QT_DEV uint32_t aw_digits(float x, float two_f) {
    const int Q = __float2int_rn(x * two_f);
    return ((uint32_t)Q + 0x80808080u) ^ 0x80808080u;
}
// hi * 2^16 + lo (the digit pairs' partial sums, exact ints) rounded once to fp32, scaled
QT_DEV float aw_comb(int lo, int hi, float scale) { return fmaf((float)hi, 65536.f, (float)lo) * scale; }

template <int DH, int G, int MINB>
__global__ void __launch_bounds__(AW_MAXW * 32, MINB) k_attn_dec_w(const float* __restrict__ qkv, int ldq, int H, int Hkv,
                                                             const int* __restrict__ kv_len, uint8_t* __restrict__ pool,
                                                             long long page_bytes, const int* __restrict__ pt,
                                                             int max_pages, const double2* __restrict__ rope,
                                                             const int* __restrict__ pos, float inv_sqrt,
                                                             float* __restrict__ part_ml, float* __restrict__ part_o) {
    constexpr bool SPLIT = G > 2;       // one kv head per CTA, one MMA column tile per warp
    constexpr int HW = SPLIT ? 2 : G;   // query heads per warp
    using S = AwSmem<DH, HW>;
    constexpr int CB = S::CB;
    constexpr int NT = SPLIT ? 1 : (G + 1) / 2;  // the warp's n8 tiles: two heads x four digits each
    constexpr int KS = DH / 32;      // QK k-steps; also the 32-bit code words a lane reads per key
    constexpr int MT = DH / 16;      // PV m-tiles (channels)
    constexpr int WPG = DH / 64;     // code words per key a lane transposes in PV
    extern __shared__ __align__(128) uint8_t sm_all[];
    pdl_launch_dependents();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int kh = SPLIT ? blockIdx.y : blockIdx.y * (blockDim.x >> 5) + warp;
    const int hb = SPLIT ? 2 * warp : 0;  // the warp's first query head within its kv head
    if (kh >= Hkv) {
        pdl_wait();
        return;
    }
    uint8_t* sm = sm_all + (SPLIT ? 0 : (size_t)warp * (S::sh_total + S::w_total));
    uint8_t* smw = SPLIT ? sm_all + S::sh_total + (size_t)warp * S::w_total : sm + S::sh_total;
    const int p = blockIdx.x, nsplit = gridDim.x, b = blockIdx.z;
    const bool fused = rope != nullptr;
    const int old_len = kv_len[b];
    const int len = old_len + (fused ? 1 : 0);
    const int r0 = p * kPage;
    const int n_rows = min(kPage, len - r0);
    const size_t pidx0 = ((size_t)b * H + (size_t)kh * G) * nsplit + p;
    if (n_rows <= 0) {  // nothing cached in this page: an empty partial per head
        pdl_wait();     // the partial buffers are still read by the previous layer's merge
#pragma unroll
        for (int gl = 0; gl < HW; ++gl)
            if (hb + gl < G)
                for (int c = lane; c < DH; c += 32) part_o[(pidx0 + (size_t)(hb + gl) * nsplit) * DH + c] = 0.f;
        if (lane < HW && hb + lane < G) {
            part_ml[(pidx0 + (size_t)(hb + lane) * nsplit) * 2] = -1e30f;
            part_ml[(pidx0 + (size_t)(hb + lane) * nsplit) * 2 + 1] = 0.f;
        }
        return;
    }
    uint8_t* vc = sm + S::vc;
    float* ksc = reinterpret_cast<float*>(sm + S::ks);
    float* vsc = reinterpret_cast<float*>(sm + S::vs);
    float* sc = reinterpret_cast<float*>(smw + S::sc);
    uint8_t* ql = smw + S::ql;
    uint8_t* wl = smw + S::wl;
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + S::bar);
    const size_t cbh = (size_t)Hkv * CB;
    const uint8_t* page_c = pool + (long long)pt[b * max_pages + p] * page_bytes;
    const bool owner = !SPLIT || warp == 0;  // issues the page copy, appends the new row
    if (owner && lane == 0) {
        mbar_init(bar, 1);
        mbar_fence_init();
        mbar_arrive_expect_tx(bar, (uint32_t)(CB + 2 * kPage * 4));
        const uint8_t* page = page_c;
        bulk_g2s(vc, page + cbh + (size_t)kh * CB, CB, bar);
        bulk_g2s(ksc, page + 2 * cbh + (size_t)kh * kPage * 4, kPage * 4, bar);
        bulk_g2s(vsc, page + 2 * cbh + ((size_t)Hkv + kh) * kPage * 4, kPage * 4, bar);
    }
    // the lane's K code words (keys 16 mt + g (+ 8), words KS * t ..), straight from the cache:
    // one warp instruction reads 8 whole 64 B rows
    uint32_t kw[4][2][KS];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
            const uint8_t* src = page_c + (size_t)kh * CB + (size_t)(16 * mt + g + 8 * hf) * (DH / 2) + t * KS * 4;
            // (ld.global.cg: the rows are read once, no L1 allocation)
            if constexpr (KS == 4) {
                const uint4 w4 = __ldcg(reinterpret_cast<const uint4*>(src));
                kw[mt][hf][0] = w4.x; kw[mt][hf][1] = w4.y; kw[mt][hf][2] = w4.z; kw[mt][hf][3] = w4.w;
            } else {
                const uint2 w2 = __ldcg(reinterpret_cast<const uint2*>(src));
                kw[mt][hf][0] = w2.x; kw[mt][hf][1] = w2.y;
            }
        }
    // the RoPE cos / sin of the lane's q pairs and new-K pairs (the table and the position are
    // final before the upstream chain): loaded before the wait, off the q -> RoPE path
    constexpr int PPL = DH / 64;  // dim pairs per lane per head
    constexpr int E = DH / 32;
    // (ld.global.cg: an invariant .nc load is scheduled below the wait by the compiler / ptxas)
    double2 cq[PPL], ckr[E / 2];
    if (fused) {
        const double2* rt = rope + (size_t)pos[b] * (DH / 2);
#pragma unroll
        for (int j = 0; j < PPL; ++j) cq[j] = __ldcg(rt + lane + 32 * j);
#pragma unroll
        for (int j = 0; j < E / 2; ++j) ckr[j] = __ldcg(rt + lane * E / 2 + j);
    }
    if (SPLIT) __syncthreads();  // the barrier is initialised before the other warps wait on it
    pdl_wait();  // q (and the new token's k / v) come from the upstream GEMV
    qkv = pdl_fresh(qkv);

    // q of the warp's heads (RoPE'd here in the decode step: fp64, rounded to fp32 like the
    // prefill's k_rope_kv_append) -> fixed-point digits in MMA-B order
    const float* qrow = qkv + (size_t)b * ldq;
    int F[HW];
#pragma unroll
    for (int gl = 0; gl < HW; ++gl) {
        const int gh = hb + gl;
        F[gl] = 0;
        if (gh >= G) continue;
        float2 v[PPL];
        float mx = 0.f;
#pragma unroll
        for (int j = 0; j < PPL; ++j) {
            const int pr = lane + 32 * j;
            v[j] = *reinterpret_cast<const float2*>(qrow + (size_t)(kh * G + gh) * DH + 2 * pr);
            if (fused) {
                const double2 cs = cq[j];
                const double a = v[j].x, bb = v[j].y;
                v[j].x = (float)__dsub_rn(__dmul_rn(a, cs.x), __dmul_rn(bb, cs.y));
                v[j].y = (float)__dadd_rn(__dmul_rn(a, cs.y), __dmul_rn(bb, cs.x));
            }
            mx = fmaxf(mx, fmaxf(fabsf(v[j].x), fabsf(v[j].y)));
        }
        F[gl] = aw_fexp(warp_max(mx));
        const float two_f = aw_pow2(F[gl]);
#pragma unroll
        for (int j = 0; j < PPL; ++j) {
            const int d = 2 * (lane + 32 * j);
            const uint32_t L0 = aw_digits(v[j].x, two_f), L1 = aw_digits(v[j].y, two_f);
            uint8_t* row = ql + (size_t)gl * 4 * DH;
#pragma unroll
            for (int dg = 0; dg < 4; ++dg) {
                row[dg * DH + aw_qpos(d)] = (uint8_t)(L0 >> (8 * dg));
                row[dg * DH + aw_qpos(d + 1)] = (uint8_t)(L1 >> (8 * dg));
            }
        }
    }
    // the new row (decode step): its K (RoPE'd) then its V -- kv_quantize in fp64, appended
    const int new_r = old_len - r0;  // row within this page
    const bool has_new = fused && new_r >= 0 && new_r < n_rows;
    uint32_t new_word[2] = {0u, 0u};
    float new_scale[2] = {0.f, 0.f};
    if (has_new) {
        uint8_t* page = pool + (long long)pt[b * max_pages + p] * page_bytes;
#pragma unroll
        for (int kv = 0; kv < 2; ++kv) {
            if (kv == 1 && !owner) break;  // the other warps only need the K row (in registers)
            const float* src = qrow + (kv == 0 ? H * DH : (H + Hkv) * DH) + kh * DH + lane * E;
            double val[E];
#pragma unroll
            for (int j = 0; j < E; ++j) val[j] = (double)src[j];
            if (kv == 0) {
#pragma unroll
                for (int j = 0; j < E; j += 2) {
                    const double2 cs = ckr[j / 2];
                    const double a = val[j], bb = val[j + 1];
                    val[j] = __dsub_rn(__dmul_rn(a, cs.x), __dmul_rn(bb, cs.y));
                    val[j + 1] = __dadd_rn(__dmul_rn(a, cs.y), __dmul_rn(bb, cs.x));
                }
            }
            double mx = 0.0;
#pragma unroll
            for (int j = 0; j < E; ++j) mx = fmax(mx, fabs(val[j]));
            mx = warp_max(mx);
            const double s = q_scale(mx, 7), inv_s = 1.0 / s;
            uint32_t w = 0;
#pragma unroll
            for (int j = 0; j < E; ++j) w |= (uint32_t)(q_code_r(val[j], s, inv_s, 7) & 0xF) << (4 * j);
            new_word[kv] = w;
            new_scale[kv] = (float)s;
            if (!owner) continue;
            // append to the cache (model.cpp:499-501)
            uint8_t* dst = page + (kv == 0 ? 0 : cbh) + (size_t)kh * CB + (size_t)new_r * (DH / 2) + lane * E / 2;
            if (E == 4) *reinterpret_cast<uint16_t*>(dst) = (uint16_t)w;
            else *dst = (uint8_t)w;
            if (lane == 0)
                reinterpret_cast<float*>(page + 2 * cbh)[(kv == 0 ? 0 : Hkv * kPage) + kh * kPage + new_r] =
                    (float)s;
        }
    }
    if (has_new) {  // the new K row replaces its stale register copy: word w of the row is the
                    // 8 / E lanes' pieces from lane w * 8 / E on
#pragma unroll
        for (int s2 = 0; s2 < KS; ++s2) {
            const int w = KS * t + s2;
            uint32_t word = 0;
#pragma unroll
            for (int q = 0; q < 8 / E; ++q)
                word |= (__shfl_sync(0xffffffffu, new_word[0], w * (8 / E) + q) & ((1u << (4 * E)) - 1u)) << (4 * E * q);
#pragma unroll
            for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                for (int hf = 0; hf < 2; ++hf)
                    if (new_r == 16 * mt + 8 * hf + g) kw[mt][hf][s2] = word;
        }
    }
    mbar_wait(bar, 0);     // the page's V codes and scales have landed
    if (has_new && owner) {  // ... and the new row replaces its (stale) shared copy
        {
            uint8_t* d = vc + (size_t)new_r * (DH / 2) + lane * E / 2;
            if (E == 4) *reinterpret_cast<uint16_t*>(d) = (uint16_t)new_word[1];
            else *d = (uint8_t)new_word[1];
        }
        if (lane == 0) {
            ksc[new_r] = new_scale[0];
            vsc[new_r] = new_scale[1];
        }
    }
    if (SPLIT) __syncthreads();  // the patched row is visible to every warp of the kv head
    else __syncwarp();

    // ---- scores: S[key][head] for the 64 keys (4 m-tiles of 16 keys)
    {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            const int hq = 2 * nt + (g >> 2);  // the B column's head (within the warp's) and digit
            uint32_t bq[KS][2];
#pragma unroll
            for (int s = 0; s < KS; ++s) {
                const uint2 v = hb + hq < G ? *reinterpret_cast<const uint2*>(ql + (size_t)(hq * 4 + (g & 3)) * DH +
                                                                         8 * (KS * t + s))
                                       : make_uint2(0u, 0u);
                bq[s][0] = v.x;
                bq[s][1] = v.y;
            }
            const int ho = 2 * nt + (t >> 1);  // the accumulator columns' head
            const int Fo = (2 * nt + 1 < HW && (t >> 1)) ? F[(2 * nt + 1) % HW] : F[2 * nt];
            const float qsc = aw_pow2(-(Fo + 4)) * inv_sqrt;
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) {
                int acc[4] = {0, 0, 0, 0};
#pragma unroll
                for (int s = 0; s < KS; ++s) {
                    uint32_t a[4];
                    unpack_x16(kw[mt][0][s], a[0], a[2]);
                    unpack_x16(kw[mt][1][s], a[1], a[3]);
                    mma_s8_16832(acc, a, bq[s]);
                }
                const int P0 = acc[0] + (acc[1] << 8), P1 = acc[2] + (acc[3] << 8);  // digits 2(t&1), +1
                const int U0 = __shfl_xor_sync(0xffffffffu, P0, 1), U1 = __shfl_xor_sync(0xffffffffu, P1, 1);
                if (!(t & 1) && hb + ho < G) {
                    const int k0 = 16 * mt + g;
                    sc[ho * kPage + k0] = aw_comb(P0, U0, qsc) * ksc[k0];
                    sc[ho * kPage + k0 + 8] = aw_comb(P1, U1, qsc) * ksc[k0 + 8];
                }
            }
        }
    }
    __syncwarp();
    // ---- softmax per head over the page's rows; p * s_v -> fixed-point digits
    float m_h[HW], l_h[HW], osc[HW];
#pragma unroll
    for (int gh = 0; gh < HW; ++gh) {  // (the warp's heads)
        m_h[gh] = l_h[gh] = osc[gh] = 0.f;
        if (hb + gh >= G) continue;
        const bool ok0 = lane < n_rows, ok1 = lane + 32 < n_rows;
        const float s0 = ok0 ? sc[gh * kPage + lane] : -1e30f, s1 = ok1 ? sc[gh * kPage + lane + 32] : -1e30f;
        const float m = warp_max(fmaxf(s0, s1));
        const float p0 = ok0 ? expf(s0 - m) : 0.f, p1 = ok1 ? expf(s1 - m) : 0.f;
        const float w0 = p0 * (ok0 ? vsc[lane] : 0.f), w1 = p1 * (ok1 ? vsc[lane + 32] : 0.f);
        m_h[gh] = m;
        l_h[gh] = warp_sum(p0 + p1);
        const int Fw = aw_fexp(warp_max(fmaxf(w0, w1)));
        osc[gh] = aw_pow2(-(Fw + 4));
        const float two_w = aw_pow2(Fw);
        const uint32_t L0 = aw_digits(w0, two_w), L1 = aw_digits(w1, two_w);
        uint8_t* row = wl + (size_t)gh * 4 * kPage;
#pragma unroll
        for (int dg = 0; dg < 4; ++dg) {
            row[dg * kPage + aw_kpos(lane)] = (uint8_t)(L0 >> (8 * dg));
            row[dg * kPage + aw_kpos(lane + 32)] = (uint8_t)(L1 >> (8 * dg));
        }
    }
    __syncwarp();
    // ---- P . V: o[channel][head]; A = V^T by 4 x 4 byte transposes of 4 keys' code words
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
        const int hq = 2 * nt + (g >> 2);
        int acc[MT][4];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) acc[mt][0] = acc[mt][1] = acc[mt][2] = acc[mt][3] = 0;
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            uint32_t bw[2];
            bw[0] = hb + hq < G ? *reinterpret_cast<const uint32_t*>(wl + (size_t)(hq * 4 + (g & 3)) * kPage + 32 * s + 4 * t) : 0u;
            bw[1] = hb + hq < G ? *reinterpret_cast<const uint32_t*>(wl + (size_t)(hq * 4 + (g & 3)) * kPage + 32 * s + 16 + 4 * t) : 0u;
            // R[hf][ww][e]: channel (word WPG * g + ww, nibble e) of keys 32 s + 16 hf + t + 4 i
            uint32_t R[2][WPG][8];
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
                uint32_t w[4][WPG];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const uint8_t* src = vc + (size_t)(32 * s + 16 * hf + t + 4 * i) * (DH / 2) + g * WPG * 4;
                    if constexpr (WPG == 2) {
                        const uint2 v2 = *reinterpret_cast<const uint2*>(src);
                        w[i][0] = v2.x;
                        w[i][1] = v2.y;
                    } else {
                        w[i][0] = *reinterpret_cast<const uint32_t*>(src);
                    }
                }
#pragma unroll
                for (int ww = 0; ww < WPG; ++ww) {
                    const uint32_t t0 = prmt(w[0][ww], w[1][ww], 0x5140), t1 = prmt(w[0][ww], w[1][ww], 0x7362);
                    const uint32_t t2 = prmt(w[2][ww], w[3][ww], 0x5140), t3 = prmt(w[2][ww], w[3][ww], 0x7362);
                    const uint32_t T[4] = {prmt(t0, t2, 0x5410), prmt(t0, t2, 0x7632), prmt(t1, t3, 0x5410),
                                           prmt(t1, t3, 0x7632)};  // T[c] = byte c of the 4 keys
#pragma unroll
                    for (int c = 0; c < 4; ++c) unpack_x16(T[c], R[hf][ww][2 * c], R[hf][ww][2 * c + 1]);
                }
            }
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
                // rows g / g + 8 of m-tile mt: channel 8 WPG g + mt / 8 WPG g + DH / 16 + mt
                constexpr int HALF = DH / 16;  // == 8 WPG / 2 ... channel offset of row g + 8
                const int e0 = mt, e1 = HALF + mt;  // nibble index within the lane's 8 * WPG channels
                uint32_t a[4];
                a[0] = R[0][e0 >> 3][e0 & 7];
                a[1] = R[0][e1 >> 3][e1 & 7];
                a[2] = R[1][e0 >> 3][e0 & 7];
                a[3] = R[1][e1 >> 3][e1 & 7];
                mma_s8_16832(acc[mt], a, bw);
            }
        }
        const int ho = 2 * nt + (t >> 1);
        const float oscale = (2 * nt + 1 < HW && (t >> 1)) ? osc[(2 * nt + 1) % HW] : osc[2 * nt];
        float o[2][MT];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
            const int P0 = acc[mt][0] + (acc[mt][1] << 8), P1 = acc[mt][2] + (acc[mt][3] << 8);
            const int U0 = __shfl_xor_sync(0xffffffffu, P0, 1), U1 = __shfl_xor_sync(0xffffffffu, P1, 1);
            o[0][mt] = aw_comb(P0, U0, oscale);
            o[1][mt] = aw_comb(P1, U1, oscale);
        }
        if (!(t & 1) && hb + ho < G) {  // channels 8 WPG g .. 8 WPG g + 8 WPG - 1 (rows g, then g + 8)
            float* dst = part_o + (pidx0 + (size_t)(hb + ho) * nsplit) * DH + 8 * WPG * g;
#pragma unroll
            for (int hf = 0; hf < 2; ++hf)
#pragma unroll
                for (int c = 0; c < MT; c += 4)
                    *reinterpret_cast<float4*>(dst + hf * MT + c) =
                        make_float4(o[hf][c], o[hf][c + 1], o[hf][c + 2], o[hf][c + 3]);
        }
    }
#pragma unroll
    for (int gh = 0; gh < HW; ++gh)
        if (lane == gh && hb + gh < G) {
            part_ml[(pidx0 + (size_t)(hb + gh) * nsplit) * 2] = m_h[gh];
            part_ml[(pidx0 + (size_t)(hb + gh) * nsplit) * 2 + 1] = l_h[gh];
        }
}

// Merge the split partials of every head of one sequence (fixed split order) and,
// optionally, quantize the concatenated attention row (the attn_out site,
// model.cpp:394/539) in the same kernel.  grid B, 1024 threads: warp w merges heads
// w, w+32, ...; lane c holds channels c*CPL.. of that head.
template <int DH, int MAXH>
__global__ void __launch_bounds__(1024) k_attn_merge_quant(const float* __restrict__ part_ml,
                                                           const float* __restrict__ part_o, int npg, int H,
                                                           float* __restrict__ out, int ldo,
                                                           uint8_t* __restrict__ codes, int ld_codes,
                                                           double* __restrict__ scales, int mode, double static_scale,
                                                           int d_pad, int qmax, int8_t* __restrict__ codes8, int ld8) {
    constexpr int CPL = DH / 32;
    __shared__ double red[32];
    pdl_launch_dependents();
    pdl_wait();
    const int b = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int HPW = (MAXH + 31) / 32;  // heads per warp
    float o[HPW][CPL];
    double mx = 0.0;
#pragma unroll
    for (int hh = 0; hh < HPW; ++hh) {
        const int h = warp + 32 * hh;
#pragma unroll
        for (int c = 0; c < CPL; ++c) o[hh][c] = 0.f;
        if (h >= H) continue;
        const size_t base = ((size_t)b * H + h) * npg;
        float M = -1e30f;
        float L = 0.f;
        if (npg <= 32) {
            // lane p holds split p's (m, l): one load per lane, then the loop only loads o
            // (independent of M, so it pipelines) and takes (m, l) by shuffle
            // (o of up to 8 pages per batch as one vector load each, all issued together with
            // the (m, l) load: one L2 round trip per 8 pages instead of one per 4 pages and
            // channel; the accumulation order is unchanged)
            using VecT = typename std::conditional<CPL == 4, float4, float2>::type;
            float2 mlv = make_float2(-1e30f, 0.f);
            if (lane < npg) mlv = __ldcg(reinterpret_cast<const float2*>(part_ml + (base + lane) * 2));
            constexpr int PB = 8;
            VecT ov[PB];
#pragma unroll
            for (int j = 0; j < PB; ++j)
                if (j < npg) ov[j] = __ldcg(reinterpret_cast<const VecT*>(part_o + (base + j) * DH + lane * CPL));
            M = warp_max(mlv.x);
            for (int p0 = 0; p0 < npg; p0 += PB) {
#pragma unroll
                for (int j = 0; j < PB; ++j) {
                    const int p = p0 + j;
                    if (p >= npg) break;
                    const float mp = __shfl_sync(0xffffffffu, mlv.x, p), lp = __shfl_sync(0xffffffffu, mlv.y, p);
                    const float a = lp == 0.f ? 0.f : expf(mp - M);
                    L += lp * a;
                    const float* v = reinterpret_cast<const float*>(&ov[j]);
#pragma unroll
                    for (int c = 0; c < CPL; ++c) o[hh][c] += v[c] * a;
                    if (p + PB < npg)  // the next batch's page, into the slot just consumed
                        ov[j] = __ldcg(reinterpret_cast<const VecT*>(part_o + (base + p + PB) * DH + lane * CPL));
                }
            }
        } else {
            for (int p = lane; p < npg; p += 32) M = fmaxf(M, part_ml[(base + p) * 2]);
            M = warp_max(M);
#pragma unroll 4
            for (int p = 0; p < npg; ++p) {
                const float2 mlp = *reinterpret_cast<const float2*>(part_ml + (base + p) * 2);
                float ov[CPL];
#pragma unroll
                for (int c = 0; c < CPL; ++c) ov[c] = part_o[(base + p) * DH + lane * CPL + c];
                const float a = mlp.y == 0.f ? 0.f : expf(mlp.x - M);
                L += mlp.y * a;
#pragma unroll
                for (int c = 0; c < CPL; ++c) o[hh][c] += ov[c] * a;
            }
        }
        const float il = 1.f / L;
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
            o[hh][c] *= il;
            mx = fmax(mx, fabs((double)o[hh][c]));
            if (out) out[(size_t)b * ldo + h * DH + lane * CPL + c] = o[hh][c];
        }
    }
    if (!codes) return;
    double s;
    if (mode == 0) {
        s = static_scale;
    } else {
        mx = block_max1(mx, red);
        s = q_scale(mx, qmax);
    }
    const double inv_s = 1.0 / s;
#pragma unroll
    for (int hh = 0; hh < HPW; ++hh) {
        const int h = warp + 32 * hh;
        if (h >= H) continue;
        int c[CPL];
#pragma unroll
        for (int e = 0; e < CPL; ++e) c[e] = q_code_r((double)o[hh][e], s, inv_s, qmax);
        const int k0 = h * DH + lane * CPL;
        if (CPL == 4) {
            *reinterpret_cast<uint16_t*>(codes + w4t_offset(b, k0 / 2, ld_codes)) =
                (uint16_t)((c[0] & 0xF) | ((c[1] & 0xF) << 4) | ((c[2] & 0xF) << 8) | ((c[3] & 0xF) << 12));
            if (codes8)  // the int8-operand GEMM's copy: 16 x code, row-major
                *reinterpret_cast<uint32_t*>(codes8 + (size_t)b * ld8 + k0) =
                    (uint32_t)((c[0] << 4) & 0xFF) | ((uint32_t)((c[1] << 4) & 0xFF) << 8) |
                    ((uint32_t)((c[2] << 4) & 0xFF) << 16) | ((uint32_t)((c[3] << 4) & 0xFF) << 24);
        } else {
            codes[w4t_offset(b, k0 / 2, ld_codes)] = (uint8_t)((c[0] & 0xF) | ((c[1] & 0xF) << 4));
            if (codes8)
                *reinterpret_cast<uint16_t*>(codes8 + (size_t)b * ld8 + k0) =
                    (uint16_t)(((c[0] << 4) & 0xFF) | (((c[1] << 4) & 0xFF) << 8));
        }
    }
    // zero the K padding of this row
    for (int k = H * DH + threadIdx.x * 2; k < d_pad; k += blockDim.x * 2) {
        codes[w4t_offset(b, k / 2, ld_codes)] = 0;
        if (codes8) *reinterpret_cast<uint16_t*>(codes8 + (size_t)b * ld8 + k) = 0;
    }
    if (threadIdx.x == 0) scales[b] = s;
}

template <int DH, int G>
static int launch_dec_w(int nsplit, int Hkv, int B, cudaStream_t st, const float* qkv, int ldq, int H,
                        const int* kv_len, uint8_t* pool, long long page_bytes, const int* pt, int max_pages,
                        const double2* rope, const int* pos, float inv_sqrt, float* part_ml, float* part_o) {
    constexpr bool SPLIT = G > 2;
    using S = AwSmem<DH, SPLIT ? 2 : G>;
    // G <= 2: up to 4 kv heads per CTA, one warp each; G > 2: one kv head, one warp per 2 heads
    const int wpc = SPLIT ? (G + 1) / 2 : std::min(AW_MAXW, Hkv);
    const size_t smem = SPLIT ? S::sh_total + (size_t)wpc * S::w_total : (size_t)wpc * (S::sh_total + S::w_total);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int gy = SPLIT ? Hkv : (Hkv + wpc - 1) / wpc;
    const long long ctas = (long long)nsplit * gy * B;
    auto kfn = ctas > (long long)5 * sms ? k_attn_dec_w<DH, G, AW_MINB_WIDE> : k_attn_dec_w<DH, G, 1>;
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    return launch_pdl(kfn, dim3(nsplit, gy, B), dim3(32 * wpc), smem, st, qkv, ldq, H, Hkv,
                      kv_len, pool, page_bytes, pt, max_pages, rope, pos, inv_sqrt, part_ml, part_o);
}


}  // namespace qt

using namespace qt;

extern "C" {

int qt_attn_decode_plan(int B, int H, int Hkv, int pages, int sms, int* pps, int* nsplit) {
    if (pages < 1 || B < 1 || Hkv < 1 || H % Hkv) return -1;
    (void)sms;
    *pps = 1;  // k_attn_dec_w: one page per warp (per split)
    *nsplit = pages;
    return 0;
}

int qt_launch_attn_decode(const float* qkv, int ldq, int H, int Hkv, int dh, const int* kv_len, int B,
                          uint8_t* pool, long long page_bytes, const int* pt, int max_pages, int pps, int nsplit,
                          const double* rope, const int* pos, float* part_ml, float* part_o, float* out, int ldo,
                          uint8_t* codes, int ld_codes, double* scales, int qmode, double static_scale, int d_pad,
                          int bits, int8_t* codes8, int ld8, cudaStream_t st) {
    if (B <= 0) return 0;
    if (H > 64 || Hkv < 1 || H % Hkv || H / Hkv > AD_MAX_G || pps != 1 || nsplit < 1) return -1;
    // (splits past a sequence's pages write empty partials: only pages holding cached rows are read)
    const int G = H / Hkv;
    const float inv_sqrt = (float)(1.0 / sqrt((double)dh));
    const double2* rt = reinterpret_cast<const double2*>(rope);
    int rc = -1;
#define QT_AD(D, GG)                                                                                          \
    if (dh == D && G == GG)                                                                                   \
        rc = launch_dec_w<D, GG>(nsplit, Hkv, B, st, qkv, ldq, H, kv_len, pool, page_bytes, pt, max_pages, rt, pos, \
                                 inv_sqrt, part_ml, part_o);
    QT_AD(128, 1) QT_AD(128, 2) QT_AD(128, 4) QT_AD(128, 7) QT_AD(128, 8)
    QT_AD(64, 1) QT_AD(64, 2) QT_AD(64, 4) QT_AD(64, 7) QT_AD(64, 8)
#undef QT_AD
    if (rc) return rc;
    const int qmax = (1 << (bits - 1)) - 1;
    if (dh == 128) {
        auto mk = H > 32 ? k_attn_merge_quant<128, 64> : k_attn_merge_quant<128, 32>;
        return launch_pdl(mk, dim3(B), dim3(1024), 0, st, (const float*)part_ml, (const float*)part_o, nsplit, H,
                          out, ldo, codes, ld_codes, scales, qmode, static_scale, d_pad, qmax, codes8, ld8);
    }
    auto mk = H > 32 ? k_attn_merge_quant<64, 64> : k_attn_merge_quant<64, 32>;
    return launch_pdl(mk, dim3(B), dim3(1024), 0, st, (const float*)part_ml, (const float*)part_o, nsplit, H, out,
                      ldo, codes, ld_codes, scales, qmode, static_scale, d_pad, qmax, codes8, ld8);
}

}  // extern "C"
