// k_attn.cu -- attention over the paged int4 KV cache.
//
//   K7  prefill attention with the reference mask (model.cpp:35-44,272-292,385):
//       visual queries see only visual keys (bidirectional); text queries see
//       every visual key plus causal text.  Keys/values are the dequantised
//       int4 rows k^ = code * s (model.cpp:371-372).  Optionally emits the row
//       max / sum so K3a can rebuild normalised probabilities.
//   K3a QUOTA attention-received metrics (selector.cpp:40-49): per visual key
//       i and head h, column sums of softmax probabilities over text queries
//       (m^inter) and over visual queries (m^intra).  Deterministic: partial
//       sums per (seq, head, key) in fixed order, no float atomics.
//   K6  decode attention (model.cpp:515-535): one query row per sequence over
//       all cached rows, unmasked, 128-bit coalesced int4 loads dequantised in
//       registers, split over pages + a fixed-order merge.
//
// Tensor-core math (mma.sync m16n8k16 f16->f32) uses hi/lo fp16 splits of the
// fp32 operand (q, or p * s_v); int4 codes are exact in fp16, so products are
// accurate to ~2^-22 relative -- well inside the 1e-3 score tolerance.
#include "qt_common.cuh"
#include "qt_kernels.h"

namespace qt {

constexpr int AT_Q = 64;   // query rows per CTA (16 per warp)
constexpr int AT_K = 64;   // key rows per tile == kPage

struct PageRef {
    const uint8_t* codes;  // K codes for (kv head) rows of this page: [kPage][dh/2]
    const float* scales;   // [kPage]
};

// Page p of (seq b): K codes at page + kh*kPage*dh/2, V codes after Hkv*kPage*dh/2,
// K scales after 2*Hkv*kPage*dh/2, V scales after those.
QT_DEV const uint8_t* page_base(const uint8_t* pool, long long page_bytes, const int* pt, int max_pages, int b,
                                int j) {
    return pool + (long long)pt[b * max_pages + j / kPage] * page_bytes;
}

// Load one 64-key tile of K and V (both row layout [key][dh] fp16 codes, row
// stride DH + 8) plus scales into shared memory.
template <int DH>
QT_DEV void load_kv_tile(const uint8_t* page, int Hkv, int kh, int nkeys, __half* Ks, __half* Vt, float* ks,
                         float* vs, bool need_v) {
    constexpr int KLD = DH + 8;
    const size_t cb = (size_t)Hkv * kPage * (DH / 2);
    const uint8_t* kc = page + (size_t)kh * kPage * (DH / 2);
    const uint8_t* vc = page + cb + (size_t)kh * kPage * (DH / 2);
    const float* ksc = reinterpret_cast<const float*>(page + 2 * cb) + kh * kPage;
    const float* vsc = reinterpret_cast<const float*>(page + 2 * cb) + Hkv * kPage + kh * kPage;
    // 16-byte chunks: AT_K * DH/2 / 16 per matrix
    constexpr int CH = AT_K * (DH / 2) / 16;
    for (int c = threadIdx.x; c < CH; c += blockDim.x) {
        const int row = c / (DH / 32), col = (c % (DH / 32)) * 32;  // 32 codes per chunk
        uint4 w = row < nkeys ? *reinterpret_cast<const uint4*>(kc + (size_t)c * 16) : make_uint4(0, 0, 0, 0);
        uint32_t* dst = reinterpret_cast<uint32_t*>(Ks + row * KLD + col);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint32_t word = (&w.x)[q];
#pragma unroll
            for (int bb = 0; bb < 4; ++bb) dst[q * 4 + bb] = nib2_to_h2((word >> (8 * bb)) & 0xFF);
        }
        if (need_v) {  // row-major like K; the PV MMA reads it transposed with ldmatrix.trans
            uint4 v = row < nkeys ? *reinterpret_cast<const uint4*>(vc + (size_t)c * 16) : make_uint4(0, 0, 0, 0);
            uint32_t* vd = reinterpret_cast<uint32_t*>(Vt + row * KLD + col);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                uint32_t word = (&v.x)[q];
#pragma unroll
                for (int bb = 0; bb < 4; ++bb) vd[q * 4 + bb] = nib2_to_h2((word >> (8 * bb)) & 0xFF);
            }
        }
    }
    for (int r = threadIdx.x; r < AT_K; r += blockDim.x) {
        ks[r] = r < nkeys ? ksc[r] : 0.f;
        if (need_v) vs[r] = r < nkeys ? vsc[r] : 0.f;
    }
}

// Raw int4 tile of one page for kv head kh: K codes [AT_K][DH/2], V codes, K and V
// scales -- issued as cp.async 16-byte copies (rows >= nkeys zero-filled), no registers.
template <int DH>
QT_DEV void load_kv_raw_async(const uint8_t* page, int Hkv, int kh, int nkeys, uint8_t* raw) {
    constexpr int CB = AT_K * (DH / 2);  // code bytes per matrix
    const size_t cb = (size_t)Hkv * kPage * (DH / 2);
    const uint8_t* kc = page + (size_t)kh * kPage * (DH / 2);
    const uint8_t* vc = page + cb + (size_t)kh * kPage * (DH / 2);
    const uint8_t* ksc = page + 2 * cb + (size_t)kh * kPage * 4;
    const uint8_t* vsc = page + 2 * cb + ((size_t)Hkv * kPage + kh * kPage) * 4;
    for (int c = threadIdx.x; c < CB / 16; c += blockDim.x) {
        const bool ok = c / (DH / 32) < nkeys;
        cp_async16(raw + c * 16, kc + (size_t)c * 16, ok);
        cp_async16(raw + CB + c * 16, vc + (size_t)c * 16, ok);
    }
    for (int c = threadIdx.x; c < 2 * (AT_K * 4 / 16); c += blockDim.x) {  // 16 chunks of 4 scales each
        const int m = c / (AT_K * 4 / 16), q = c % (AT_K * 4 / 16);
        cp_async16(raw + 2 * CB + c * 16, (m ? vsc : ksc) + q * 16, q * 4 < nkeys);
    }
    cp_async_commit();
}

// Dequantise the raw tile (smem) into the fp16 K / V tiles and the scale arrays.
template <int DH>
QT_DEV void dequant_kv_raw(const uint8_t* raw, int nkeys, __half* Ks, __half* Vt, float* ks, float* vs) {
    constexpr int KLD = DH + 8;
    constexpr int CB = AT_K * (DH / 2);
    for (int c = threadIdx.x; c < CB / 16; c += blockDim.x) {
        const int row = c / (DH / 32), col = (c % (DH / 32)) * 32;
        const uint4 w = *reinterpret_cast<const uint4*>(raw + c * 16);
        const uint4 v = *reinterpret_cast<const uint4*>(raw + CB + c * 16);
        uint32_t* kd = reinterpret_cast<uint32_t*>(Ks + row * KLD + col);
        uint32_t* vd = reinterpret_cast<uint32_t*>(Vt + row * KLD + col);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
#pragma unroll
            for (int bb = 0; bb < 4; ++bb) {
                kd[q * 4 + bb] = nib2_to_h2(((&w.x)[q] >> (8 * bb)) & 0xFF);
                vd[q * 4 + bb] = nib2_to_h2(((&v.x)[q] >> (8 * bb)) & 0xFF);
            }
        }
    }
    const float* sc = reinterpret_cast<const float*>(raw + 2 * CB);
    for (int r = threadIdx.x; r < AT_K; r += blockDim.x) {
        ks[r] = r < nkeys ? sc[r] : 0.f;
        vs[r] = r < nkeys ? sc[AT_K + r] : 0.f;
    }
}

// Q fragments (hi/lo) for 16 query rows of one head: qf[s][0..3] hi, ql lo.
template <int DH>
QT_DEV void load_q_frags(const float* qkv, int ldq, int tok0, int rows_valid, int h, uint32_t (*qh)[4],
                         uint32_t (*ql)[4]) {
    const int lane = threadIdx.x & 31, g = lane >> 2, tig = lane & 3;
#pragma unroll
    for (int s = 0; s < DH / 16; ++s) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int row = g + ((r & 1) ? 8 : 0);
            const int col = s * 16 + ((r & 2) ? 8 : 0) + 2 * tig;
            float2 v = make_float2(0.f, 0.f);
            if (row < rows_valid) v = *reinterpret_cast<const float2*>(qkv + (size_t)(tok0 + row) * ldq + h * DH + col);
            split_h2(v.x, v.y, qh[s][r], ql[s][r]);
        }
    }
}

// S(16 x 64) = Q(16 x DH) . K^T with hi/lo split of Q.
template <int DH>
QT_DEV void qk_tile(const uint32_t (*qh)[4], const uint32_t (*ql)[4], const __half* Ks, float (*sc)[4]) {
    constexpr int KLD = DH + 8;
    const int lane = threadIdx.x & 31, g = lane >> 2, tig = lane & 3;
#pragma unroll
    for (int t = 0; t < AT_K / 8; ++t) {
        sc[t][0] = sc[t][1] = sc[t][2] = sc[t][3] = 0.f;
#pragma unroll
        for (int s = 0; s < DH / 16; ++s) {
            uint32_t b[2];
            const __half* kr = Ks + (t * 8 + g) * KLD + s * 16 + 2 * tig;
            b[0] = *reinterpret_cast<const uint32_t*>(kr);
            b[1] = *reinterpret_cast<const uint32_t*>(kr + 8);
            mma_f16_16816(sc[t], qh[s], b);
            mma_f16_16816(sc[t], ql[s], b);
        }
    }
}

// ============================================================== K7
#ifndef QT_ATTN_MINB
#define QT_ATTN_MINB 2  // 3 caps at 168 registers with spills; 2: 255, no spills (prefill -0.15 ms)
#endif
template <int DH>
__global__ void __launch_bounds__(128, QT_ATTN_MINB) k_attn_prefill(const float* __restrict__ qkv, int ldq, int H, int Hkv,
                                                      const int* __restrict__ seq_off, const int* __restrict__ vis,
                                                      const int* __restrict__ seq_len,
                                                      const uint8_t* __restrict__ pool, long long page_bytes,
                                                      const int* __restrict__ pt, int max_pages, float inv_sqrt,
                                                      float* __restrict__ out, int ldo, float2* __restrict__ ml,
                                                      float* __restrict__ pmax, int pmax_ld) {
    constexpr int KLD = DH + 8;
    __shared__ __align__(16) __half Ks[AT_K * KLD];
    __shared__ __align__(16) __half Vt[AT_K * KLD];  // V, row layout (read with ldmatrix.trans)
    __shared__ float ks[AT_K], vs[AT_K];
    __shared__ __align__(16) uint8_t raw[AT_K * DH + 2 * AT_K * 4];  // next tile's int4 codes + scales
    const int b = blockIdx.z, h = blockIdx.y;
    const int S = seq_len[b], V = vis[b];
    const int q0 = blockIdx.x * AT_Q;
    if (q0 >= S) return;
    const int kh = h / (H / Hkv);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, tig = lane & 3;
    const int tok0 = seq_off[b];
    const int wq0 = q0 + warp * 16;  // first query row of this warp (index in sequence)
    const float sl2 = inv_sqrt * 1.4426950408889634f;  // 1/sqrt(dh) * log2(e)

    uint32_t qh[DH / 16][4], ql[DH / 16][4];
    load_q_frags<DH>(qkv, ldq, tok0 + wq0, S - wq0, h, qh, ql);

    float o[DH / 8][4];
#pragma unroll
    for (int t = 0; t < DH / 8; ++t) o[t][0] = o[t][1] = o[t][2] = o[t][3] = 0.f;
    float mrow[2] = {-1e30f, -1e30f}, lrow[2] = {0.f, 0.f};
    const int qi[2] = {wq0 + g, wq0 + g + 8};

    const int kend = max(V, min(S, q0 + AT_Q));
    // two-stage: the raw int4 codes of tile k0 + AT_K stream in (cp.async) while tile k0 computes
    load_kv_raw_async<DH>(page_base(pool, page_bytes, pt, max_pages, b, 0), Hkv, kh, min(AT_K, S), raw);
    for (int k0 = 0; k0 < kend; k0 += AT_K) {
        cp_async_wait<0>();
        __syncthreads();  // raw holds tile k0; every warp is done with tile k0 - AT_K
        dequant_kv_raw<DH>(raw, min(AT_K, S - k0), Ks, Vt, ks, vs);
        __syncthreads();  // raw free, tile k0 ready
        if (k0 + AT_K < kend)
            load_kv_raw_async<DH>(page_base(pool, page_bytes, pt, max_pages, b, k0 + AT_K), Hkv, kh,
                                  min(AT_K, S - k0 - AT_K), raw);
        // scores in log2 units: s2 = q.k * (scale_k / sqrt(dh) * log2 e), p = 2^(s2 - m2)
        // warp-uniform tile classification against the reference mask (model.cpp:35-44):
        // `none` -> no (query, key) pair of this warp's 16 rows x 64 keys is allowed;
        // `full` -> every pair is allowed and in range, so the per-element test is skipped
        const int klast = k0 + AT_K - 1, qlast = wq0 + 15;
        const bool none = wq0 >= S || (qlast < V && k0 >= V);
        const bool full = qlast < S && klast < S &&
                          (qlast < V ? klast < V : (wq0 >= V && (klast < V || klast <= wq0)));
        if (none) continue;  // no MMA needed (the block-wide syncs stay uniform)
        float sc[AT_K / 8][4];
        qk_tile<DH>(qh, ql, Ks, sc);
        // scale, mask, row max
        float tmax[2] = {-1e30f, -1e30f};
#pragma unroll
        for (int t = 0; t < AT_K / 8; ++t) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int r = e >> 1;
                const int kj = k0 + t * 8 + 2 * tig + (e & 1);
                const int q = qi[r];
                const bool ok = full || (q < S && kj < S && (q < V ? kj < V : (kj < V || kj <= q)));
                float s = ok ? sc[t][e] * (ks[t * 8 + 2 * tig + (e & 1)] * sl2) : -1e30f;
                sc[t][e] = s;
                tmax[r] = fmaxf(tmax[r], s);
            }
        }
        float alpha[2];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            tmax[r] = fmaxf(tmax[r], __shfl_xor_sync(0xffffffffu, tmax[r], 1));
            tmax[r] = fmaxf(tmax[r], __shfl_xor_sync(0xffffffffu, tmax[r], 2));
            const float mn = fmaxf(mrow[r], tmax[r]);
            alpha[r] = exp2f(mrow[r] - mn);
            mrow[r] = mn;
        }
        float psum[2] = {0.f, 0.f};
        uint32_t ph[AT_K / 16][4], pl[AT_K / 16][4];
#pragma unroll
        for (int t = 0; t < AT_K / 8; ++t) {
            float p[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int r = e >> 1;
                p[e] = sc[t][e] <= -1e30f ? 0.f : exp2f(sc[t][e] - mrow[r]);
                psum[r] += p[e];
                p[e] *= vs[t * 8 + 2 * tig + (e & 1)];
            }
            // A fragment of step u = t/2: tile 2u -> regs 0,1; tile 2u+1 -> regs 2,3
            const int u = t >> 1, hi2 = (t & 1) * 2;
            split_h2(p[0], p[1], ph[u][hi2 + 0], pl[u][hi2 + 0]);
            split_h2(p[2], p[3], ph[u][hi2 + 1], pl[u][hi2 + 1]);
        }
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            psum[r] += __shfl_xor_sync(0xffffffffu, psum[r], 1);
            psum[r] += __shfl_xor_sync(0xffffffffu, psum[r], 2);
            lrow[r] = lrow[r] * alpha[r] + psum[r];
        }
#pragma unroll
        for (int t = 0; t < DH / 8; ++t) {
            o[t][0] *= alpha[0];
            o[t][1] *= alpha[0];
            o[t][2] *= alpha[1];
            o[t][3] *= alpha[1];
#pragma unroll
            for (int u = 0; u < AT_K / 16; ++u) {
                uint32_t bb[2];
                // B fragment (keys u*16.., channels t*8..) of row-major V: 8x8 halves of rows
                // u*16 + lane (lanes 0..15), transposed on load
                const __half* vr = Vt + (u * 16 + (lane & 15)) * KLD + t * 8;
                asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0, %1}, [%2];\n"
                             : "=r"(bb[0]), "=r"(bb[1])
                             : "r"(smem_u32(vr)));
                mma_f16_16816(o[t], ph[u], bb);
                mma_f16_16816(o[t], pl[u], bb);
            }
        }
    }
    // finalize
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int q = qi[r];
        const bool ok = q < S;
        float mx = 0.f;  // max |out| of this (row, head): the attn_out quantizer's partial row max
        if (ok) {
            const float inv_l = 1.f / lrow[r];
            float* orow = out + (size_t)(tok0 + q) * ldo + h * DH;
#pragma unroll
            for (int t = 0; t < DH / 8; ++t) {
                float2 v = make_float2(o[t][2 * r] * inv_l, o[t][2 * r + 1] * inv_l);
                *reinterpret_cast<float2*>(orow + t * 8 + 2 * tig) = v;
                mx = fmaxf(mx, fmaxf(fabsf(v.x), fabsf(v.y)));
            }
            // row max back in natural-log units for the QUOTA column sums (k_attn_colsum uses expf)
            if (ml && tig == 0) ml[(size_t)(tok0 + q) * H + h] = make_float2(mrow[r] * 0.69314718055994531f, lrow[r]);
        }
        if (pmax) {  // the quad of lanes sharing the row
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
            if (ok && tig == 0) pmax[(size_t)(tok0 + q) * pmax_ld + h] = mx;
        }
    }
}

// ============================================================== K3a
// grid (ceil(Vmax/64), H, B).  colsum[(b*H + h)*vstride + i] for i < V.
template <int DH>
__global__ void __launch_bounds__(128) k_attn_colsum(const float* __restrict__ qkv, int ldq, int H, int Hkv,
                                                     const int* __restrict__ seq_off, const int* __restrict__ vis,
                                                     const int* __restrict__ seq_len,
                                                     const uint8_t* __restrict__ pool, long long page_bytes,
                                                     const int* __restrict__ pt, int max_pages, float inv_sqrt,
                                                     const float2* __restrict__ ml, int vstride,
                                                     float* __restrict__ inter, float* __restrict__ intra) {
    constexpr int KLD = DH + 8;
    __shared__ __align__(16) __half Ks[AT_K * KLD];
    __shared__ float ks[AT_K], vs_unused[AT_K];
    __shared__ float red[2][4][AT_K];
    const int b = blockIdx.z, h = blockIdx.y;
    const int S = seq_len[b], V = vis[b];
    const int k0 = blockIdx.x * AT_K;
    if (k0 >= V) return;
    const int kh = h / (H / Hkv);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, tig = lane & 3;
    const int tok0 = seq_off[b];
    const uint8_t* page = page_base(pool, page_bytes, pt, max_pages, b, k0);
    load_kv_tile<DH>(page, Hkv, kh, min(AT_K, V - k0), Ks, nullptr, ks, vs_unused, false);
    __syncthreads();

    float ci[AT_K / 8][2], ca[AT_K / 8][2];  // inter (text q), intra (visual q)
#pragma unroll
    for (int t = 0; t < AT_K / 8; ++t) ci[t][0] = ci[t][1] = ca[t][0] = ca[t][1] = 0.f;

    for (int q0 = warp * 16; q0 < S; q0 += 64) {
        uint32_t qh[DH / 16][4], ql[DH / 16][4];
        load_q_frags<DH>(qkv, ldq, tok0 + q0, S - q0, h, qh, ql);
        float sc[AT_K / 8][4];
        qk_tile<DH>(qh, ql, Ks, sc);
        float mr[2], il[2];
        bool valid[2], isvis[2];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int q = q0 + g + 8 * r;
            valid[r] = q < S;
            isvis[r] = q < V;
            float2 v = valid[r] ? ml[(size_t)(tok0 + q) * H + h] : make_float2(0.f, 1.f);
            mr[r] = v.x;
            il[r] = 1.f / v.y;
        }
#pragma unroll
        for (int t = 0; t < AT_K / 8; ++t) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int r = e >> 1, c = e & 1;
                if (!valid[r]) continue;
                const float s = sc[t][e] * ks[t * 8 + 2 * tig + c] * inv_sqrt;
                const float p = expf(s - mr[r]) * il[r];
                if (isvis[r]) ca[t][c] += p;
                else ci[t][c] += p;
            }
        }
    }
    // reduce over g (lanes differing in bits 2..4), then over warps
#pragma unroll
    for (int t = 0; t < AT_K / 8; ++t)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
#pragma unroll
            for (int o = 4; o < 32; o <<= 1) {
                ci[t][c] += __shfl_xor_sync(0xffffffffu, ci[t][c], o);
                ca[t][c] += __shfl_xor_sync(0xffffffffu, ca[t][c], o);
            }
            if (g == 0) {
                red[0][warp][t * 8 + 2 * tig + c] = ci[t][c];
                red[1][warp][t * 8 + 2 * tig + c] = ca[t][c];
            }
        }
    __syncthreads();
    for (int i = threadIdx.x; i < AT_K; i += blockDim.x) {
        if (k0 + i >= V) continue;
        const float si = ((red[0][0][i] + red[0][1][i]) + red[0][2][i]) + red[0][3][i];
        const float sa = ((red[1][0][i] + red[1][1][i]) + red[1][2][i]) + red[1][3][i];
        inter[((size_t)b * H + h) * vstride + k0 + i] = si;
        intra[((size_t)b * H + h) * vstride + k0 + i] = sa;
    }
}

// ============================================================== K6 merge by the last arrival
// Called by every page CTA of (b, h) after its partial is written (128 threads).
// The last CTA to arrive for (b, h) merges the head's page partials in fixed page
// order -- the same arithmetic as k_attn_merge_quant -- into the fp32 attention
// row and the head's max |o|; the last head of sequence b to finish then
// quantizes the whole row for the attn_out site.  Both arrival counters
// (cnt[b*H + h], cnt[B*H + b]) are reset by their last arrival, so the kernel
// replays from a CUDA graph.  Replaces the separate merge launch.
template <int DH>
QT_DEV void attn_dec_arrive(int b, int h, int H, int npg, const float* part_ml, const float* part_o, unsigned* cnt,
                            float* row, float* hmax, uint8_t* codes, int ld_codes, double* scales, int qmode,
                            double static_scale, int d_pad, int qmax) {
    __shared__ unsigned s_last;
    __shared__ float s_red[4];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int B = gridDim.z;
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(&cnt[b * H + h], 1u) == (unsigned)npg - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (tid == 0) cnt[b * H + h] = 0;
    const size_t base = ((size_t)b * H + h) * npg;
    float M = -1e30f;
    for (int p = lane; p < npg; p += 32) M = fmaxf(M, part_ml[(base + p) * 2]);
    M = warp_max(M);
    float L = 0.f, o = 0.f;
    for (int p0 = 0; p0 < npg; p0 += 4) {  // 4 pages' loads in flight, summed in page order
        float2 ml4[4];
        float ov[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int p = p0 + j;
            ml4[j] = p < npg ? *reinterpret_cast<const float2*>(part_ml + (base + p) * 2) : make_float2(-1e30f, 0.f);
            ov[j] = p < npg && tid < DH ? part_o[(base + p) * DH + tid] : 0.f;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (ml4[j].y == 0.f) continue;
            const float a = expf(ml4[j].x - M);
            L += ml4[j].y * a;
            o += ov[j] * a;
        }
    }
    o *= 1.f / L;
    const int HD = H * DH;
    if (tid < DH) row[(size_t)b * HD + h * DH + tid] = o;
    float mx = tid < DH ? fabsf(o) : 0.f;
    mx = warp_max(mx);
    if (lane == 0) s_red[warp] = mx;
    __syncthreads();
    if (tid == 0) hmax[b * H + h] = fmaxf(fmaxf(s_red[0], s_red[1]), fmaxf(s_red[2], s_red[3]));
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(&cnt[B * H + b], 1u) == (unsigned)H - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (tid == 0) cnt[B * H + b] = 0;
    double s = static_scale;
    if (qmode != 0) {
        float m2 = 0.f;
        for (int i = lane; i < H; i += 32) m2 = fmaxf(m2, hmax[b * H + i]);
        s = q_scale((double)warp_max(m2), qmax);
    }
    const double inv_s = 1.0 / s;
    for (int w = tid; w < d_pad / 8; w += blockDim.x) {
        int c[8];
        if (w * 8 < HD) {
            const float4 a = *reinterpret_cast<const float4*>(row + (size_t)b * HD + w * 8);
            const float4 bq = *reinterpret_cast<const float4*>(row + (size_t)b * HD + w * 8 + 4);
            const float f[8] = {a.x, a.y, a.z, a.w, bq.x, bq.y, bq.z, bq.w};
#pragma unroll
            for (int e = 0; e < 8; ++e) c[e] = q_code_r((double)f[e], s, inv_s, qmax);
        } else {
#pragma unroll
            for (int e = 0; e < 8; ++e) c[e] = 0;
        }
        *reinterpret_cast<uint32_t*>(codes + w4t_offset(b, w * 4, ld_codes)) = pack8(c);
    }
    if (tid == 0) scales[b] = s;
}

// ============================================================== K6
// grid (pages, H, B), 128 threads: one CTA per (64-row page, query head,
// sequence) -- the cache length is read from device memory so the decode step
// replays from a CUDA graph.  Each warp owns 16 rows; 4 lanes per row each
// hold 32 channels (16 bytes of int4 codes), and both of a lane's rows are
// loaded before any math so two 128-bit loads per operand are in flight.
//
// rope != nullptr (the decode step, K5 fused in): q is RoPE'd in registers from
// the raw GEMV output, and the CTAs of the page holding the new row (row
// kv_len) RoPE + quantize that token's K and V (kv_quantize, quant.cpp:117-119)
// and append them before attending -- one launch instead of two.  With GQA the
// group's query-head CTAs write identical bytes.
template <int DH>
__global__ void __launch_bounds__(128) k_attn_decode(const float* __restrict__ qkv, int ldq, int H, int Hkv,
                                                     const int* __restrict__ kv_len, int len_add,
                                                     uint8_t* __restrict__ pool, long long page_bytes,
                                                     const int* __restrict__ pt, int max_pages, float inv_sqrt,
                                                     float* __restrict__ part_ml, float* __restrict__ part_o,
                                                     const double2* __restrict__ rope, const int* __restrict__ pos,
                                                     unsigned* __restrict__ cnt, float* __restrict__ row,
                                                     float* __restrict__ hmax, uint8_t* __restrict__ codes,
                                                     int ld_codes, double* __restrict__ scales, int qmode,
                                                     double static_scale, int d_pad, int qmax) {
    constexpr int CPL = DH / 4;  // channels per lane
    constexpr int R = 2;         // rows per lane
    pdl_launch_dependents();
    // Without the fused append (rope == null) every cached row but the newest (len - 1, written
    // by the K/V append kernel just before) is final since earlier steps, as are kv_len and the
    // page table: those loads are issued before the dependency wait and overlap the upstream
    // kernel; q and the newest row are read after it (the row through L2, not the .nc path,
    // since its 128-byte line may have been cached with the row before it).
    if (rope) pdl_wait();
    const int b = blockIdx.z, h = blockIdx.y, pg = blockIdx.x, npg = gridDim.x;
    const int kh = h / (H / Hkv);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int q4 = lane & 3, quad = lane >> 2;
    const int len = kv_len[b] + len_add;
    const int r0 = pg * kPage;
    const size_t pidx = ((size_t)b * H + h) * npg + pg;
    const double2* rt = rope ? rope + (size_t)pos[b] * (DH / 2) : nullptr;
    if (rope && pg == (len - 1) / kPage && warp < 2) {
        // append the new token's K (warp 0, RoPE'd) or V (warp 1) of kv head kh at row len-1
        constexpr int E = DH / 32;
        const int r = len - 1;
        const bool is_k = warp == 0;
        const float* src = qkv + (size_t)b * ldq + (is_k ? H * DH : (H + Hkv) * DH) + kh * DH;
        double val[E];
#pragma unroll
        for (int j = 0; j < E; ++j) val[j] = (double)src[lane * E + j];
        if (is_k) {
#pragma unroll
            for (int j = 0; j < E; j += 2) {
                const double2 cs = rt[(lane * E + j) / 2];
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
        int c[4] = {0, 0, 0, 0};
#pragma unroll
        for (int j = 0; j < E; ++j) c[j] = q_code_r(val[j], s, inv_s, 7);
        uint8_t* page = pool + (long long)pt[b * max_pages + r / kPage] * page_bytes;
        const size_t cbn = (size_t)Hkv * kPage * (DH / 2);
        uint8_t* dst = page + (is_k ? 0 : cbn) + ((size_t)kh * kPage + r % kPage) * (DH / 2) + lane * E / 2;
        if (E == 4)
            *reinterpret_cast<uint16_t*>(dst) =
                (uint16_t)((c[0] & 0xF) | ((c[1] & 0xF) << 4) | ((c[2] & 0xF) << 8) | ((c[3] & 0xF) << 12));
        else
            *dst = (uint8_t)((c[0] & 0xF) | ((c[1] & 0xF) << 4));
        if (lane == 0)
            reinterpret_cast<float*>(page + 2 * cbn)[(is_k ? 0 : Hkv * kPage) + kh * kPage + r % kPage] = (float)s;
    }
    if (rope) __syncthreads();  // the appended row is visible to the block's loads below
    if (r0 >= len) {
        if (!rope) pdl_wait();  // part buffers are still read by the previous layer's merge
        if (threadIdx.x < DH) part_o[pidx * DH + threadIdx.x] = 0.f;
        if (threadIdx.x == 0) {
            part_ml[pidx * 2] = -1e30f;
            part_ml[pidx * 2 + 1] = 0.f;
        }
        if (cnt) attn_dec_arrive<DH>(b, h, H, npg, part_ml, part_o, cnt, row, hmax, codes, ld_codes, scales, qmode,
                                     static_scale, d_pad, qmax);
        return;
    }
    const uint8_t* page = pool + (long long)pt[b * max_pages + pg] * page_bytes;
    const size_t cb = (size_t)Hkv * kPage * (DH / 2);
    const float* sc = reinterpret_cast<const float*>(page + 2 * cb);
    uint32_t kw[R][CPL / 8], vw[R][CPL / 8];
    float sk[R], sv[R];
    bool valid[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
        const int slot = warp * 16 + quad + 8 * i;
        valid[i] = r0 + slot < len;
        const bool ld = valid[i] && (rope || r0 + slot != len - 1);  // the newest row: after the wait
        const uint8_t* krow = page + ((size_t)kh * kPage + slot) * (DH / 2) + q4 * (CPL / 2);
        if (CPL == 32) {
            uint4 ka = ld ? ldg_nc_v4(krow) : make_uint4(0, 0, 0, 0);
            uint4 va = ld ? ldg_nc_v4(krow + cb) : make_uint4(0, 0, 0, 0);
            kw[i][0] = ka.x; kw[i][1] = ka.y; kw[i][2] = ka.z; kw[i][3] = ka.w;
            vw[i][0] = va.x; vw[i][1] = va.y; vw[i][2] = va.z; vw[i][3] = va.w;
        } else {
            uint2 ka = ld ? *reinterpret_cast<const uint2*>(krow) : make_uint2(0, 0);
            uint2 va = ld ? *reinterpret_cast<const uint2*>(krow + cb) : make_uint2(0, 0);
            kw[i][0] = ka.x; kw[i][1] = ka.y;
            vw[i][0] = va.x; vw[i][1] = va.y;
        }
        sk[i] = ld ? sc[kh * kPage + slot] : 0.f;
        sv[i] = ld ? sc[Hkv * kPage + kh * kPage + slot] : 0.f;
    }
    if (!rope) {
        pdl_wait();  // q and the newest row come from the upstream kernels
#pragma unroll
        for (int i = 0; i < R; ++i) {
            const int slot = warp * 16 + quad + 8 * i;
            if (!(valid[i] && r0 + slot == len - 1)) continue;
            const uint8_t* krow = page + ((size_t)kh * kPage + slot) * (DH / 2) + q4 * (CPL / 2);
            if (CPL == 32) {
                const uint4 ka = __ldcg(reinterpret_cast<const uint4*>(krow));
                const uint4 va = __ldcg(reinterpret_cast<const uint4*>(krow + cb));
                kw[i][0] = ka.x; kw[i][1] = ka.y; kw[i][2] = ka.z; kw[i][3] = ka.w;
                vw[i][0] = va.x; vw[i][1] = va.y; vw[i][2] = va.z; vw[i][3] = va.w;
            } else {
                const uint2 ka = __ldcg(reinterpret_cast<const uint2*>(krow));
                const uint2 va = __ldcg(reinterpret_cast<const uint2*>(krow + cb));
                kw[i][0] = ka.x; kw[i][1] = ka.y;
                vw[i][0] = va.x; vw[i][1] = va.y;
            }
            sk[i] = __ldcg(sc + kh * kPage + slot);
            sv[i] = __ldcg(sc + Hkv * kPage + kh * kPage + slot);
        }
    }
    float q[CPL];
    const float* qp = qkv + (size_t)b * ldq + h * DH + q4 * CPL;
#pragma unroll
    for (int i = 0; i < CPL; i += 4) {
        float4 v = *reinterpret_cast<const float4*>(qp + i);
        q[i] = v.x; q[i + 1] = v.y; q[i + 2] = v.z; q[i + 3] = v.w;
    }
    if (rope) {  // interleaved-pair RoPE of q in fp32 (q only feeds fp32 scores; K keeps the fp64 path)
#pragma unroll
        for (int i = 0; i < CPL; i += 2) {
            const double2 cs = rt[(q4 * CPL + i) / 2];
            const float c = (float)cs.x, sn = (float)cs.y, a = q[i], bb = q[i + 1];
            q[i] = fmaf(a, c, -bb * sn);
            q[i + 1] = fmaf(a, sn, bb * c);
        }
    }
    float s[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
        float d = 0.f;
#pragma unroll
        for (int w = 0; w < CPL / 8; ++w)
#pragma unroll
            for (int e = 0; e < 8; ++e) d = fmaf(q[w * 8 + e], (float)nib(kw[i][w], e), d);
        d += __shfl_xor_sync(0xffffffffu, d, 1);
        d += __shfl_xor_sync(0xffffffffu, d, 2);
        s[i] = valid[i] ? d * sk[i] * inv_sqrt : -1e30f;
    }
    float m = fmaxf(s[0], s[1]);
    float l = 0.f;
    float acc[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) acc[c] = 0.f;
#pragma unroll
    for (int i = 0; i < R; ++i) {
        if (!valid[i]) continue;
        const float p = expf(s[i] - m);
        l += p;
        const float pv = p * sv[i];
#pragma unroll
        for (int w = 0; w < CPL / 8; ++w)
#pragma unroll
            for (int e = 0; e < 8; ++e) acc[w * 8 + e] = fmaf(pv, (float)nib(vw[i][w], e), acc[w * 8 + e]);
    }
    // merge the 8 quads of the warp (lanes with equal q4)
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
        const float mo = __shfl_xor_sync(0xffffffffu, m, o);
        const float lo = __shfl_xor_sync(0xffffffffu, l, o);
        const float mn = fmaxf(m, mo);
        const float a1 = expf(m - mn), a2 = expf(mo - mn);
        l = l * a1 + lo * a2;
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
            const float ao = __shfl_xor_sync(0xffffffffu, acc[c], o);
            acc[c] = acc[c] * a1 + ao * a2;
        }
        m = mn;
    }
    __shared__ float smx[4][2];
    __shared__ float so[4][DH];
    if (quad == 0) {
#pragma unroll
        for (int c = 0; c < CPL; ++c) so[warp][q4 * CPL + c] = acc[c];
        if (q4 == 0) {
            smx[warp][0] = m;
            smx[warp][1] = l;
        }
    }
    __syncthreads();
    if (threadIdx.x < DH) {
        float mm = -1e30f;
        for (int w = 0; w < 4; ++w) mm = fmaxf(mm, smx[w][0]);
        float ll = 0.f, oo = 0.f;
        for (int w = 0; w < 4; ++w) {
            const float a = smx[w][1] > 0.f ? expf(smx[w][0] - mm) : 0.f;
            ll += smx[w][1] * a;
            oo += so[w][threadIdx.x] * a;
        }
        part_o[pidx * DH + threadIdx.x] = oo;
        if (threadIdx.x == 0) {
            part_ml[pidx * 2] = mm;
            part_ml[pidx * 2 + 1] = ll;
        }
    }
    if (cnt) attn_dec_arrive<DH>(b, h, H, npg, part_ml, part_o, cnt, row, hmax, codes, ld_codes, scales, qmode,
                                 static_scale, d_pad, qmax);
}

// Two 64-row pages per CTA (4 rows per lane): half the CTAs and half the partials of
// k_attn_decode.  Unfused path only (rope == nullptr).
template <int DH, int PP = 2>
__global__ void __launch_bounds__(128) k_attn_decode_pp2(const float* __restrict__ qkv, int ldq, int H, int Hkv,
                                                     const int* __restrict__ kv_len, int len_add,
                                                     uint8_t* __restrict__ pool, long long page_bytes,
                                                     const int* __restrict__ pt, int max_pages, float inv_sqrt,
                                                     float* __restrict__ part_ml, float* __restrict__ part_o,
                                                     const double2* __restrict__ rope, const int* __restrict__ pos,
                                                     unsigned* __restrict__ cnt, float* __restrict__ row,
                                                     float* __restrict__ hmax, uint8_t* __restrict__ codes,
                                                     int ld_codes, double* __restrict__ scales, int qmode,
                                                     double static_scale, int d_pad, int qmax) {
    constexpr int CPL = DH / 4;  // channels per lane
    constexpr int R = 2 * PP;    // rows per lane: PP 64-row pages per CTA
    constexpr int WR = 16 * PP;  // rows per warp (64 / WR warps per page)
    pdl_launch_dependents();
    // Without the fused append (rope == null) every cached row but the newest (len - 1, written
    // by the K/V append kernel just before) is final since earlier steps, as are kv_len and the
    // page table: those loads are issued before the dependency wait and overlap the upstream
    // kernel; q and the newest row are read after it (the row through L2, not the .nc path,
    // since its 128-byte line may have been cached with the row before it).
    if (rope) pdl_wait();
    const int b = blockIdx.z, h = blockIdx.y, pg = blockIdx.x, npg = gridDim.x;
    const int kh = h / (H / Hkv);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int q4 = lane & 3, quad = lane >> 2;
    const int len = kv_len[b] + len_add;
    const int r0 = pg * PP * kPage;
    const size_t pidx = ((size_t)b * H + h) * npg + pg;
    const double2* rt = rope ? rope + (size_t)pos[b] * (DH / 2) : nullptr;
    if (rope && pg == (len - 1) / kPage && warp < 2) {
        // append the new token's K (warp 0, RoPE'd) or V (warp 1) of kv head kh at row len-1
        constexpr int E = DH / 32;
        const int r = len - 1;
        const bool is_k = warp == 0;
        const float* src = qkv + (size_t)b * ldq + (is_k ? H * DH : (H + Hkv) * DH) + kh * DH;
        double val[E];
#pragma unroll
        for (int j = 0; j < E; ++j) val[j] = (double)src[lane * E + j];
        if (is_k) {
#pragma unroll
            for (int j = 0; j < E; j += 2) {
                const double2 cs = rt[(lane * E + j) / 2];
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
        int c[4] = {0, 0, 0, 0};
#pragma unroll
        for (int j = 0; j < E; ++j) c[j] = q_code_r(val[j], s, inv_s, 7);
        uint8_t* page = pool + (long long)pt[b * max_pages + r / kPage] * page_bytes;
        const size_t cbn = (size_t)Hkv * kPage * (DH / 2);
        uint8_t* dst = page + (is_k ? 0 : cbn) + ((size_t)kh * kPage + r % kPage) * (DH / 2) + lane * E / 2;
        if (E == 4)
            *reinterpret_cast<uint16_t*>(dst) =
                (uint16_t)((c[0] & 0xF) | ((c[1] & 0xF) << 4) | ((c[2] & 0xF) << 8) | ((c[3] & 0xF) << 12));
        else
            *dst = (uint8_t)((c[0] & 0xF) | ((c[1] & 0xF) << 4));
        if (lane == 0)
            reinterpret_cast<float*>(page + 2 * cbn)[(is_k ? 0 : Hkv * kPage) + kh * kPage + r % kPage] = (float)s;
    }
    if (rope) __syncthreads();  // the appended row is visible to the block's loads below
    if (r0 >= len) {
        if (!rope) pdl_wait();  // part buffers are still read by the previous layer's merge
        if (threadIdx.x < DH) part_o[pidx * DH + threadIdx.x] = 0.f;
        if (threadIdx.x == 0) {
            part_ml[pidx * 2] = -1e30f;
            part_ml[pidx * 2 + 1] = 0.f;
        }
        if (cnt) attn_dec_arrive<DH>(b, h, H, npg, part_ml, part_o, cnt, row, hmax, codes, ld_codes, scales, qmode,
                                     static_scale, d_pad, qmax);
        return;
    }
    const int wrow0 = r0 + warp * WR;  // a warp's 32 rows lie in one page
    // (clamped: a trailing odd page's partner may lie past the table; its rows are all invalid)
    const uint8_t* page = pool + (long long)pt[b * max_pages + min(wrow0 / kPage, max_pages - 1)] * page_bytes;
    const int pofs = wrow0 % kPage;
    const size_t cb = (size_t)Hkv * kPage * (DH / 2);
    const float* sc = reinterpret_cast<const float*>(page + 2 * cb);
    uint32_t kw[R][CPL / 8], vw[R][CPL / 8];
    float sk[R], sv[R];
    bool valid[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
        const int slot = warp * WR + quad + 8 * i;
        valid[i] = r0 + slot < len;
        const bool ld = valid[i] && (rope || r0 + slot != len - 1);  // the newest row: after the wait
        const uint8_t* krow = page + ((size_t)kh * kPage + pofs + quad + 8 * i) * (DH / 2) + q4 * (CPL / 2);
        if (CPL == 32) {
            uint4 ka = ld ? ldg_nc_v4(krow) : make_uint4(0, 0, 0, 0);
            uint4 va = ld ? ldg_nc_v4(krow + cb) : make_uint4(0, 0, 0, 0);
            kw[i][0] = ka.x; kw[i][1] = ka.y; kw[i][2] = ka.z; kw[i][3] = ka.w;
            vw[i][0] = va.x; vw[i][1] = va.y; vw[i][2] = va.z; vw[i][3] = va.w;
        } else {
            uint2 ka = ld ? *reinterpret_cast<const uint2*>(krow) : make_uint2(0, 0);
            uint2 va = ld ? *reinterpret_cast<const uint2*>(krow + cb) : make_uint2(0, 0);
            kw[i][0] = ka.x; kw[i][1] = ka.y;
            vw[i][0] = va.x; vw[i][1] = va.y;
        }
        sk[i] = ld ? sc[kh * kPage + pofs + quad + 8 * i] : 0.f;
        sv[i] = ld ? sc[Hkv * kPage + kh * kPage + pofs + quad + 8 * i] : 0.f;
    }
    if (!rope) {
        pdl_wait();  // q and the newest row come from the upstream kernels
#pragma unroll
        for (int i = 0; i < R; ++i) {
            const int slot = warp * WR + quad + 8 * i;
            if (!(valid[i] && r0 + slot == len - 1)) continue;
            const uint8_t* krow = page + ((size_t)kh * kPage + pofs + quad + 8 * i) * (DH / 2) + q4 * (CPL / 2);
            if (CPL == 32) {
                const uint4 ka = __ldcg(reinterpret_cast<const uint4*>(krow));
                const uint4 va = __ldcg(reinterpret_cast<const uint4*>(krow + cb));
                kw[i][0] = ka.x; kw[i][1] = ka.y; kw[i][2] = ka.z; kw[i][3] = ka.w;
                vw[i][0] = va.x; vw[i][1] = va.y; vw[i][2] = va.z; vw[i][3] = va.w;
            } else {
                const uint2 ka = __ldcg(reinterpret_cast<const uint2*>(krow));
                const uint2 va = __ldcg(reinterpret_cast<const uint2*>(krow + cb));
                kw[i][0] = ka.x; kw[i][1] = ka.y;
                vw[i][0] = va.x; vw[i][1] = va.y;
            }
            sk[i] = __ldcg(sc + kh * kPage + pofs + quad + 8 * i);
            sv[i] = __ldcg(sc + Hkv * kPage + kh * kPage + pofs + quad + 8 * i);
        }
    }
    float q[CPL];
    const float* qp = qkv + (size_t)b * ldq + h * DH + q4 * CPL;
#pragma unroll
    for (int i = 0; i < CPL; i += 4) {
        float4 v = *reinterpret_cast<const float4*>(qp + i);
        q[i] = v.x; q[i + 1] = v.y; q[i + 2] = v.z; q[i + 3] = v.w;
    }
    if (rope) {  // interleaved-pair RoPE of q in fp32 (q only feeds fp32 scores; K keeps the fp64 path)
#pragma unroll
        for (int i = 0; i < CPL; i += 2) {
            const double2 cs = rt[(q4 * CPL + i) / 2];
            const float c = (float)cs.x, sn = (float)cs.y, a = q[i], bb = q[i + 1];
            q[i] = fmaf(a, c, -bb * sn);
            q[i + 1] = fmaf(a, sn, bb * c);
        }
    }
    float s[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
        float d = 0.f;
#pragma unroll
        for (int w = 0; w < CPL / 8; ++w)
#pragma unroll
            for (int e = 0; e < 8; ++e) d = fmaf(q[w * 8 + e], (float)nib(kw[i][w], e), d);
        d += __shfl_xor_sync(0xffffffffu, d, 1);
        d += __shfl_xor_sync(0xffffffffu, d, 2);
        s[i] = valid[i] ? d * sk[i] * inv_sqrt : -1e30f;
    }
    float m = s[0];
#pragma unroll
    for (int i = 1; i < R; ++i) m = fmaxf(m, s[i]);
    float l = 0.f;
    float acc[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) acc[c] = 0.f;
#pragma unroll
    for (int i = 0; i < R; ++i) {
        if (!valid[i]) continue;
        const float p = expf(s[i] - m);
        l += p;
        const float pv = p * sv[i];
#pragma unroll
        for (int w = 0; w < CPL / 8; ++w)
#pragma unroll
            for (int e = 0; e < 8; ++e) acc[w * 8 + e] = fmaf(pv, (float)nib(vw[i][w], e), acc[w * 8 + e]);
    }
    // merge the 8 quads of the warp (lanes with equal q4)
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
        const float mo = __shfl_xor_sync(0xffffffffu, m, o);
        const float lo = __shfl_xor_sync(0xffffffffu, l, o);
        const float mn = fmaxf(m, mo);
        const float a1 = expf(m - mn), a2 = expf(mo - mn);
        l = l * a1 + lo * a2;
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
            const float ao = __shfl_xor_sync(0xffffffffu, acc[c], o);
            acc[c] = acc[c] * a1 + ao * a2;
        }
        m = mn;
    }
    __shared__ float smx[4][2];
    __shared__ float so[4][DH];
    if (quad == 0) {
#pragma unroll
        for (int c = 0; c < CPL; ++c) so[warp][q4 * CPL + c] = acc[c];
        if (q4 == 0) {
            smx[warp][0] = m;
            smx[warp][1] = l;
        }
    }
    __syncthreads();
    if (threadIdx.x < DH) {
        float mm = -1e30f;
        for (int w = 0; w < 4; ++w) mm = fmaxf(mm, smx[w][0]);
        float ll = 0.f, oo = 0.f;
        for (int w = 0; w < 4; ++w) {
            const float a = smx[w][1] > 0.f ? expf(smx[w][0] - mm) : 0.f;
            ll += smx[w][1] * a;
            oo += so[w][threadIdx.x] * a;
        }
        part_o[pidx * DH + threadIdx.x] = oo;
        if (threadIdx.x == 0) {
            part_ml[pidx * 2] = mm;
            part_ml[pidx * 2 + 1] = ll;
        }
    }
    if (cnt) attn_dec_arrive<DH>(b, h, H, npg, part_ml, part_o, cnt, row, hmax, codes, ld_codes, scales, qmode,
                                 static_scale, d_pad, qmax);
}

// Merge the page partials of every head of one sequence (fixed page order) and,
// optionally, quantize the concatenated attention row (the attn_out site,
// model.cpp:394/539) in the same kernel.  grid B, 1024 threads: warp w merges
// heads w, w+32, ...; lane c holds channels c*CPL.. of that head.
template <int DH, int MAXH>
__global__ void __launch_bounds__(1024) k_attn_merge_quant(const float* __restrict__ part_ml,
                                                           const float* __restrict__ part_o, int npg, int H,
                                                           float* __restrict__ out, int ldo,
                                                           uint8_t* __restrict__ codes, int ld_codes,
                                                           double* __restrict__ scales, int mode, double static_scale,
                                                           int d_pad, int qmax) {
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
            // lane p holds page p's (m, l): one load per lane, then the page loop only loads o
            // (independent of M, so it pipelines) and takes (m, l) by shuffle -- same sums
            float2 mlv = make_float2(-1e30f, 0.f);
            if (lane < npg) mlv = *reinterpret_cast<const float2*>(part_ml + (base + lane) * 2);
            M = warp_max(mlv.x);
#pragma unroll 4
            for (int p = 0; p < npg; ++p) {
                float ov[CPL];
#pragma unroll
                for (int c = 0; c < CPL; ++c) ov[c] = part_o[(base + p) * DH + lane * CPL + c];
                const float mp = __shfl_sync(0xffffffffu, mlv.x, p), lp = __shfl_sync(0xffffffffu, mlv.y, p);
                const float a = lp == 0.f ? 0.f : expf(mp - M);
                L += lp * a;
#pragma unroll
                for (int c = 0; c < CPL; ++c) o[hh][c] += ov[c] * a;
            }
        } else {
            for (int p = lane; p < npg; p += 32) M = fmaxf(M, part_ml[(base + p) * 2]);
            M = warp_max(M);
            // branch-free so the loads of consecutive pages overlap; an empty page (l = 0,
            // o = 0, m = -1e30) contributes exactly 0, as a skipped iteration would
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
        } else {
            codes[w4t_offset(b, k0 / 2, ld_codes)] = (uint8_t)((c[0] & 0xF) | ((c[1] & 0xF) << 4));
        }
    }
    // zero the K padding of this row
    for (int k = H * DH + threadIdx.x * 2; k < d_pad; k += blockDim.x * 2) codes[w4t_offset(b, k / 2, ld_codes)] = 0;
    if (threadIdx.x == 0) scales[b] = s;
}

}  // namespace qt

using namespace qt;

extern "C" {

int qt_launch_attn_prefill(const float* qkv, int ldq, int H, int Hkv, int dh, const int* seq_off, const int* vis,
                           const int* seq_len, int B, int smax, const uint8_t* pool, long long page_bytes,
                           const int* pt, int max_pages, float* out, int ldo, float* ml, float* pmax, int pmax_ld,
                           cudaStream_t st) {
    if (B <= 0 || smax <= 0) return 0;
    if (pmax && H > pmax_ld) return -1;
    const dim3 grid((smax + AT_Q - 1) / AT_Q, H, B);
    const float inv_sqrt = (float)(1.0 / sqrt((double)dh));
    if (dh == 128)
        k_attn_prefill<128><<<grid, 128, 0, st>>>(qkv, ldq, H, Hkv, seq_off, vis, seq_len, pool, page_bytes, pt,
                                                  max_pages, inv_sqrt, out, ldo, reinterpret_cast<float2*>(ml), pmax, pmax_ld);
    else if (dh == 64)
        k_attn_prefill<64><<<grid, 128, 0, st>>>(qkv, ldq, H, Hkv, seq_off, vis, seq_len, pool, page_bytes, pt,
                                                 max_pages, inv_sqrt, out, ldo, reinterpret_cast<float2*>(ml), pmax, pmax_ld);
    else
        return -1;
    return (int)cudaGetLastError();
}

int qt_launch_attn_colsum(const float* qkv, int ldq, int H, int Hkv, int dh, const int* seq_off, const int* vis,
                          const int* seq_len, int B, int vmax, const uint8_t* pool, long long page_bytes,
                          const int* pt, int max_pages, const float* ml, int vstride, float* inter, float* intra,
                          cudaStream_t st) {
    if (B <= 0 || vmax <= 0) return 0;
    const dim3 grid((vmax + AT_K - 1) / AT_K, H, B);
    const float inv_sqrt = (float)(1.0 / sqrt((double)dh));
    const float2* m2 = reinterpret_cast<const float2*>(ml);
    if (dh == 128)
        k_attn_colsum<128><<<grid, 128, 0, st>>>(qkv, ldq, H, Hkv, seq_off, vis, seq_len, pool, page_bytes, pt,
                                                 max_pages, inv_sqrt, m2, vstride, inter, intra);
    else if (dh == 64)
        k_attn_colsum<64><<<grid, 128, 0, st>>>(qkv, ldq, H, Hkv, seq_off, vis, seq_len, pool, page_bytes, pt,
                                                max_pages, inv_sqrt, m2, vstride, inter, intra);
    else
        return -1;
    return (int)cudaGetLastError();
}

int qt_launch_attn_decode(const float* qkv, int ldq, int H, int Hkv, int dh, const int* kv_len, int len_add, int B,
                          uint8_t* pool, long long page_bytes, const int* pt, int max_pages, int n_pages,
                          float* part_ml, float* part_o, float* out, int ldo, uint8_t* codes, int ld_codes,
                          double* scales, int qmode, double static_scale, int d_pad, int bits, const double* rope,
                          const int* pos, unsigned* counters, float* row, float* hmax, cudaStream_t st) {
    const double2* rt = reinterpret_cast<const double2*>(rope);
    if (counters && (!row || !hmax || !codes || (H * dh) % 8)) return -1;
    if (B <= 0) return 0;
    if (H > 64) return -1;
    // two 64-row pages per CTA (unfused path, dh = 128): half the CTAs, half the partials
    const int ppc = !rope && !counters && dh == 128 ? 2 : 1;
    const bool pp2 = ppc > 1;
    if (pp2) n_pages = (n_pages + ppc - 1) / ppc;
    const dim3 grid(n_pages, H, B);
    const float inv_sqrt = (float)(1.0 / sqrt((double)dh));
    const int qmax = (1 << (bits - 1)) - 1;
    int rc;
    if (dh == 128) {
        rc = pp2 ? launch_pdl(k_attn_decode_pp2<128, 2>, grid, dim3(128), 0, st, qkv, ldq, H, Hkv, kv_len, len_add, pool,
                              page_bytes, pt, max_pages, inv_sqrt, part_ml, part_o, rt, pos, counters, row, hmax,
                              codes, ld_codes, scales, qmode, static_scale, d_pad, qmax)
                 : launch_pdl(k_attn_decode<128>, grid, dim3(128), 0, st, qkv, ldq, H, Hkv, kv_len, len_add, pool,
                              page_bytes, pt, max_pages, inv_sqrt, part_ml, part_o, rt, pos, counters, row, hmax,
                              codes, ld_codes, scales, qmode, static_scale, d_pad, qmax);
        if (rc || counters) return rc;  // counters: merged + quantized by the last arrivals
        auto mk = H > 32 ? k_attn_merge_quant<128, 64> : k_attn_merge_quant<128, 32>;
        return launch_pdl(mk, dim3(B), dim3(1024), 0, st, (const float*)part_ml, (const float*)part_o, n_pages, H, out,
                          ldo, codes, ld_codes, scales, qmode, static_scale, d_pad, qmax);
    }
    if (dh == 64) {
        rc = launch_pdl(k_attn_decode<64>, grid, dim3(128), 0, st, qkv, ldq, H, Hkv, kv_len, len_add, pool,
                        page_bytes, pt, max_pages, inv_sqrt, part_ml, part_o, rt, pos, counters, row, hmax, codes,
                        ld_codes, scales, qmode, static_scale, d_pad, qmax);
        if (rc || counters) return rc;  // counters: merged + quantized by the last arrivals
        auto mk = H > 32 ? k_attn_merge_quant<64, 64> : k_attn_merge_quant<64, 32>;
        return launch_pdl(mk, dim3(B), dim3(1024), 0, st, (const float*)part_ml, (const float*)part_o, n_pages, H, out,
                          ldo, codes, ld_codes, scales, qmode, static_scale, d_pad, qmax);
    }
    return -1;
}

}  // extern "C"
