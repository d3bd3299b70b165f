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
//   (K6, decode attention, is k_attn_decode.cu)
//
// Tensor-core math (mma.sync m16n8k16 f16->f32) uses hi/lo fp16 splits of the
// fp32 operand (q, or p * s_v); int4 codes are exact in fp16, so products are
// accurate to ~2^-22 relative -- well inside the 1e-3 score tolerance.
#include "qt_common.cuh"
#include "qt_kernels.h"

namespace qt {

#ifndef QT_ATTN_QW
#define QT_ATTN_QW 4  // prefill attention warps per CTA (16 query rows each)
#endif
constexpr int AT_QW = QT_ATTN_QW;
constexpr int AT_Q = 16 * AT_QW;  // query rows per CTA
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
        for (int q = 0; q < 4; ++q) word_to_h2_pairs((&w.x)[q], dst + q * 4);
        if (need_v) {  // row-major like K; the PV MMA reads it transposed with ldmatrix.trans
            uint4 v = row < nkeys ? *reinterpret_cast<const uint4*>(vc + (size_t)c * 16) : make_uint4(0, 0, 0, 0);
            uint32_t* vd = reinterpret_cast<uint32_t*>(Vt + row * KLD + col);
#pragma unroll
            for (int q = 0; q < 4; ++q) word_to_h2_pairs((&v.x)[q], vd + q * 4);
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
            word_to_h2_pairs((&w.x)[q], kd + q * 4);
            word_to_h2_pairs((&v.x)[q], vd + q * 4);
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
__global__ void __launch_bounds__(32 * AT_QW, AT_QW > 4 ? 1 : QT_ATTN_MINB) k_attn_prefill(const float* __restrict__ qkv, int ldq, int H, int Hkv,
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
                                                     float* __restrict__ inter, float* __restrict__ intra,
                                                     float* __restrict__ probs, int p_rows, int p_ld) {
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
                // LayerActivationRecord blocks (model.cpp:382-384): p[h][query][visual key]
                const int kk = k0 + t * 8 + 2 * tig + c;
                if (probs && kk < V) probs[(((size_t)b * H + h) * p_rows + q0 + g + 8 * r) * p_ld + kk] = p;
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

}  // namespace qt

using namespace qt;

extern "C" {

int qt_launch_attn_prefill(const float* qkv, int ldq, int H, int Hkv, int dh, const int* seq_off, const int* vis,
                           const int* seq_len, int B, int smax, const uint8_t* pool, long long page_bytes,
                           const int* pt, int max_pages, float* out, int ldo, float* ml, float* pmax, int pmax_ld,
                           cudaStream_t st) {
    if (B <= 0 || smax <= 0) return 0;
    if (pmax && H > pmax_ld) return -1;
    const float inv_sqrt = (float)(1.0 / sqrt((double)dh));
    const dim3 grid((smax + AT_Q - 1) / AT_Q, H, B);
    if (dh == 128)
        k_attn_prefill<128><<<grid, 32 * AT_QW, 0, st>>>(qkv, ldq, H, Hkv, seq_off, vis, seq_len, pool, page_bytes, pt,
                                                  max_pages, inv_sqrt, out, ldo, reinterpret_cast<float2*>(ml), pmax, pmax_ld);
    else if (dh == 64)
        k_attn_prefill<64><<<grid, 32 * AT_QW, 0, st>>>(qkv, ldq, H, Hkv, seq_off, vis, seq_len, pool, page_bytes, pt,
                                                 max_pages, inv_sqrt, out, ldo, reinterpret_cast<float2*>(ml), pmax, pmax_ld);
    else
        return -1;
    return (int)cudaGetLastError();
}

int qt_launch_attn_colsum(const float* qkv, int ldq, int H, int Hkv, int dh, const int* seq_off, const int* vis,
                          const int* seq_len, int B, int vmax, const uint8_t* pool, long long page_bytes,
                          const int* pt, int max_pages, const float* ml, int vstride, float* inter, float* intra,
                          float* probs, int p_rows, int p_ld, cudaStream_t st) {
    if (B <= 0 || vmax <= 0) return 0;
    const dim3 grid((vmax + AT_K - 1) / AT_K, H, B);
    const float inv_sqrt = (float)(1.0 / sqrt((double)dh));
    const float2* m2 = reinterpret_cast<const float2*>(ml);
    if (dh == 128)
        k_attn_colsum<128><<<grid, 128, 0, st>>>(qkv, ldq, H, Hkv, seq_off, vis, seq_len, pool, page_bytes, pt,
                                                 max_pages, inv_sqrt, m2, vstride, inter, intra, probs, p_rows, p_ld);
    else if (dh == 64)
        k_attn_colsum<64><<<grid, 128, 0, st>>>(qkv, ldq, H, Hkv, seq_off, vis, seq_len, pool, page_bytes, pt,
                                                max_pages, inv_sqrt, m2, vstride, inter, intra, probs, p_rows, p_ld);
    else
        return -1;
    return (int)cudaGetLastError();
}

}  // extern "C"
