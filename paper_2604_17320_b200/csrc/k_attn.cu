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

// ---------------------------------------------------------------- tcgen05 helpers (kind::f16)
QT_DEV float ex2_approx(float x) {  // 2^x, flush-to-zero (x < -126 -> 0)
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;\n" : "=f"(r) : "f"(x));
    return r;
}
QT_DEV uint64_t ta_desc(uint32_t saddr) {  // K-major SWIZZLE_128B smem descriptor (SBO 1024)
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}
// kind::f16 instruction descriptor: F32 accumulate, F16 A / B, K-major, N, M = 128
constexpr uint32_t ta_idesc(int n) { return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24); }  // M = 128
QT_DEV void ta_mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
QT_DEV void ta_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
                 : "memory");
}
QT_DEV void ta_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
QT_DEV void ta_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
QT_DEV void ta_fence_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
QT_DEV void ta_ld32(uint32_t taddr, float* v) {
    uint32_t r[32];
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
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
QT_DEV void ta_st32(uint32_t taddr, const float* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n" ::"r"(taddr),
        "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]),
        "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]),
        "f"(v[17]), "f"(v[18]), "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]),
        "f"(v[25]), "f"(v[26]), "f"(v[27]), "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31])
        : "memory");
}
// byte offset of 16-byte chunk c of row r in a [rows][128 B] SWIZZLE_128B tile
QT_DEV uint32_t ta_sw(int r, int c) { return (uint32_t)(r * 128 + ((c ^ (r & 7)) << 4)); }

// ============================================================== K7 on tcgen05, warp-specialised (d_head 128)
// One CTA per (128-query tile, head, sequence), 9 warps:
//   warps 0-3  softmax: thread i owns query row i = TMEM lane i (tcgen05.ld of S, the
//              reference mask, online softmax in log2 units with a lazy max, P = p * s_v
//              split hi + lo fp16 into the UMMA A tile, O rescale when the max rises by > 8)
//   warps 4-7  producer: the int4 K / V codes of the next tiles by cp.async into a 3-deep raw
//              ring, dequantised to fp16 (exact) into double-buffered K [key][dh] and V^T
//              [dh][key] UMMA tiles -- K one tile ahead of V: K(t) then V(t - 1)
//   warp 8     TMEM owner + MMA issuer: S(t) = Q K^T (Q hi + lo) into a double-buffered S,
//              then O += P(t-1) V(t-1) -- tile t's S product runs while tile t-1's softmax does
// mbarriers: k_full / k_empty and v_full / v_empty (producer <-> MMA; a K buffer is free once
// its S product is done, a V buffer once its P.V is -- so the next K tile never waits for a
// P.V), ks_full (producer -> softmax: the tile's K / V scales, a 4-deep ring), s_full (MMA ->
// softmax), p_full (softmax -> MMA), pv_done (MMA -> softmax: P buffer free, O updated).
constexpr int TW_Q = 128, TW_K = 64;
constexpr int TW_SW = 8, TW_PW = 4;                // softmax warps (2 threads per query row), producer warps
constexpr int TW_MW = TW_SW + TW_PW;              // the MMA warp
constexpr int TW_THREADS = (TW_MW + 1) * 32;
struct TwSmem {
    static constexpr size_t qh = 0;                 // [2 sub-tiles][128 rows][128 B]
    static constexpr size_t ql = qh + 32768;
    static constexpr size_t kt = ql + 32768;        // [2 bufs][2 sub-tiles][64 keys][128 B]
    static constexpr size_t vt = kt + 2 * 16384;    // [2 bufs][128 dh][128 B]
    static constexpr size_t ph = vt + 2 * 16384;    // [2 bufs][128 q][128 B]
    static constexpr size_t pl = ph + 2 * 16384;
    static constexpr size_t raw = pl + 2 * 16384;   // [3] x (K codes 4 KB, V codes 4 KB, scales 512 B)
    static constexpr size_t raw_sz = 2 * 4096 + 512;
    static constexpr size_t kvs = raw + 3 * raw_sz; // [4 tiles] ks[64], then [4 tiles] vs[64]
    static constexpr size_t xch = kvs + 2048;       // [2 tiles][2 halves][128] tile max, then [2][128] l, [2][128] max |o|
    static constexpr size_t bars = xch + 4096;
    static constexpr size_t total = bars + 256;
};

template <int DH>
QT_DEV void tw_load_raw(const uint8_t* page, int Hkv, int kh, int nkeys, uint8_t* raw, int p, int np) {
    constexpr int CB = TW_K * (DH / 2);
    const size_t cb = (size_t)Hkv * kPage * (DH / 2);
    const uint8_t* kc = page + (size_t)kh * kPage * (DH / 2);
    const uint8_t* vc = page + cb + (size_t)kh * kPage * (DH / 2);
    const uint8_t* ksc = page + 2 * cb + (size_t)kh * kPage * 4;
    const uint8_t* vsc = page + 2 * cb + ((size_t)Hkv * kPage + kh * kPage) * 4;
    for (int c = p; c < CB / 16; c += np) {
        const bool ok = c / (DH / 32) < nkeys;
        cp_async16(raw + c * 16, kc + (size_t)c * 16, ok);
        cp_async16(raw + CB + c * 16, vc + (size_t)c * 16, ok);
    }
    for (int c = p; c < 2 * (TW_K * 4 / 16); c += np) {
        const int m = c / (TW_K * 4 / 16), q = c % (TW_K * 4 / 16);
        cp_async16(raw + 2 * CB + c * 16, (m ? vsc : ksc) + q * 16, q * 4 < nkeys);
    }
    cp_async_commit();
}

__global__ void __launch_bounds__(TW_THREADS, 1) k_attn_prefill_ws(const float* __restrict__ qkv, int ldq, int H,
                                                                    int Hkv, const int* __restrict__ seq_off,
                                                                    const int* __restrict__ vis,
                                                                    const int* __restrict__ seq_len,
                                                                    const uint8_t* __restrict__ pool,
                                                                    long long page_bytes, const int* __restrict__ pt,
                                                                    int max_pages, float inv_sqrt,
                                                                    float* __restrict__ out, int ldo,
                                                                    float2* __restrict__ ml, float* __restrict__ pmax,
                                                                    int pmax_ld) {
    constexpr int DH = 128;
    extern __shared__ __align__(1024) uint8_t sm[];
    const int b = blockIdx.z, h = blockIdx.y;
    const int S = seq_len[b], V = vis[b];
    const int q0 = blockIdx.x * TW_Q;
    if (q0 >= S) return;
    const int kh = h / (H / Hkv);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int tok0 = seq_off[b];
    const int kend = max(V, min(S, q0 + TW_Q));
    const int T = (kend + TW_K - 1) / TW_K;
    uint64_t* k_full = reinterpret_cast<uint64_t*>(sm + TwSmem::bars);
    uint64_t* k_empty = k_full + 2;
    uint64_t* v_full = k_empty + 2;
    uint64_t* v_empty = v_full + 2;
    uint64_t* s_full = v_empty + 2;
    uint64_t* p_full = s_full + 2;
    uint64_t* pv_done = p_full + 2;
    uint64_t* ks_full = pv_done + 2;  // [4]
    uint32_t* tslot = reinterpret_cast<uint32_t*>(ks_full + 4);
    float* ksb = reinterpret_cast<float*>(sm + TwSmem::kvs);  // [4][64] K scales, then [4][64] V scales
    float* vsb = ksb + 4 * TW_K;

    if (tid == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(&k_full[i], TW_PW * 32);
            mbar_init(&k_empty[i], 1);
            mbar_init(&v_full[i], TW_PW * 32);
            mbar_init(&v_empty[i], 1);
            mbar_init(&s_full[i], 1);
            mbar_init(&p_full[i], TW_SW * 32);
            mbar_init(&pv_done[i], 1);
        }
        for (int i = 0; i < 4; ++i) mbar_init(&ks_full[i], TW_PW * 32);
        mbar_fence_init();
    }
    if (warp == TW_MW) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"r"(smem_u32(tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (warp >= TW_SW && warp < TW_MW)  // the first three tiles' codes in flight while Q is staged
        for (int j = 0; j < 3; ++j) {
            if (j < T)
                tw_load_raw<DH>(page_base(pool, page_bytes, pt, max_pages, b, j * TW_K), Hkv, kh,
                                min(TW_K, S - j * TW_K), sm + TwSmem::raw + (size_t)j * TwSmem::raw_sz,
                                tid - TW_SW * 32, TW_PW * 32);
            else
                cp_async_commit();  // (empty group: the wait counts below stay regular)
        }
    if (warp < 4) {  // Q row -> hi / lo fp16 (rows past S are zero)
        const int q = q0 + tid;
        const float* qr = qkv + (size_t)(tok0 + min(q, S - 1)) * ldq + h * DH;
        const bool ok = q < S;
#pragma unroll 4
        for (int c = 0; c < 16; ++c) {
            const float4 a = ok ? *reinterpret_cast<const float4*>(qr + c * 8) : make_float4(0.f, 0.f, 0.f, 0.f);
            const float4 bb = ok ? *reinterpret_cast<const float4*>(qr + c * 8 + 4) : make_float4(0.f, 0.f, 0.f, 0.f);
            uint32_t hi[4], lo[4];
            split_h2(a.x, a.y, hi[0], lo[0]);
            split_h2(a.z, a.w, hi[1], lo[1]);
            split_h2(bb.x, bb.y, hi[2], lo[2]);
            split_h2(bb.z, bb.w, hi[3], lo[3]);
            const uint32_t off = (uint32_t)(c >> 3) * 16384 + ta_sw(tid, c & 7);
            *reinterpret_cast<uint4*>(sm + TwSmem::qh + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
            *reinterpret_cast<uint4*>(sm + TwSmem::ql + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
        }
        ta_fence_async();
    }
    ta_fence_before();
    __syncthreads();
    ta_fence_after();
    const uint32_t tmem = *tslot;
    const uint32_t tO = tmem + 128;  // S buffers at columns 0 and 64

    if (warp == TW_MW) {
        // ---------------- MMA issuer
        if (lane == 0) {
            const uint32_t qh = smem_u32(sm + TwSmem::qh), ql = smem_u32(sm + TwSmem::ql);
            for (int t = 0; t <= T; ++t) {
                if (t < T) {  // S(t) = Qhi K^T + Qlo K^T into S[t & 1]
                    const int bf = t & 1;
                    mbar_wait(&k_full[bf], (uint32_t)(t >> 1) & 1u);
                    ta_fence_after();
                    const uint32_t kt = smem_u32(sm + TwSmem::kt + (size_t)bf * 16384);
                    const uint32_t tS = tmem + (uint32_t)(bf * 64);
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        ta_mma(tS, ta_desc(qh + (k >> 2) * 16384 + (k & 3) * 32),
                               ta_desc(kt + (k >> 2) * 8192 + (k & 3) * 32), ta_idesc(TW_K), k != 0);
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        ta_mma(tS, ta_desc(ql + (k >> 2) * 16384 + (k & 3) * 32),
                               ta_desc(kt + (k >> 2) * 8192 + (k & 3) * 32), ta_idesc(TW_K), 1);
                    ta_commit(&s_full[bf]);
                    ta_commit(&k_empty[bf]);
                }
                if (t >= 1) {  // O += Phi V + Plo V of tile t - 1
                    const int u = t - 1, c = u & 1;
                    mbar_wait(&v_full[c], (uint32_t)(u >> 1) & 1u);
                    mbar_wait(&p_full[c], (uint32_t)(u >> 1) & 1u);
                    ta_fence_after();
                    const uint32_t ph = smem_u32(sm + TwSmem::ph + (size_t)c * 16384);
                    const uint32_t pl = smem_u32(sm + TwSmem::pl + (size_t)c * 16384);
                    const uint32_t vt = smem_u32(sm + TwSmem::vt + (size_t)c * 16384);
#pragma unroll
                    for (int k = 0; k < TW_K / 16; ++k)
                        ta_mma(tO, ta_desc(ph + k * 32), ta_desc(vt + k * 32), ta_idesc(DH), (u != 0) || (k != 0));
#pragma unroll
                    for (int k = 0; k < TW_K / 16; ++k)
                        ta_mma(tO, ta_desc(pl + k * 32), ta_desc(vt + k * 32), ta_idesc(DH), 1);
                    ta_commit(&pv_done[c]);
                    ta_commit(&v_empty[c]);
                }
            }
        }
        __syncwarp();
    } else if (warp >= TW_SW) {
        // ---------------- producer: K(t) then V(t - 1) per step
        const int p = tid - TW_SW * 32;
        for (int it = 0; it <= T; ++it) {
            if (it < T) {  // K(it): raw(it) has landed (groups raw(0 .. it + 1) issued so far)
                const int j = it, bf = j & 1;
                if (j == 0) cp_async_wait<2>();
                else cp_async_wait<1>();
                asm volatile("bar.sync 1, %0;\n" ::"n"(TW_PW * 32) : "memory");
                if (j >= 2) mbar_wait(&k_empty[bf], (uint32_t)((j - 2) >> 1) & 1u);
                const uint8_t* raw = sm + TwSmem::raw + (size_t)(j % 3) * TwSmem::raw_sz;
                const uint32_t* kw = reinterpret_cast<const uint32_t*>(raw);
                uint8_t* ktb = sm + TwSmem::kt + (size_t)bf * 16384;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int wi = p + 128 * i;  // K: word (key, w) in row order
                    const int key = wi >> 4, w = wi & 15;
                    uint32_t hp[4];
                    word_to_h2_pairs(kw[wi], hp);
                    *reinterpret_cast<uint4*>(ktb + (size_t)(w >> 3) * 8192 + ta_sw(key, w & 7)) =
                        *reinterpret_cast<const uint4*>(hp);
                }
                if (p < TW_K) {  // the tile's scales, a 4-deep ring (overwritten at K(j + 4), after S(j + 2),
                                 // so after softmax(j))
                    const int nk = min(TW_K, S - j * TW_K);
                    const float* sc = reinterpret_cast<const float*>(raw + 8192);
                    ksb[(j & 3) * TW_K + p] = p < nk ? sc[p] * (inv_sqrt * 1.4426950408889634f) : 0.f;  // s_k / sqrt(dh) * log2 e
                    vsb[(j & 3) * TW_K + p] = p < nk ? sc[TW_K + p] : 0.f;
                }
                ta_fence_async();
                mbar_arrive(&k_full[bf]);
                mbar_arrive(&ks_full[j & 3]);
            }
            if (it >= 1) {  // V(it - 1)
                const int j = it - 1, bf = j & 1;
                if (j >= 2) mbar_wait(&v_empty[bf], (uint32_t)((j - 2) >> 1) & 1u);
                const uint8_t* raw = sm + TwSmem::raw + (size_t)(j % 3) * TwSmem::raw_sz;
                const uint32_t* vw = reinterpret_cast<const uint32_t*>(raw + 4096);
                uint8_t* vtb = sm + TwSmem::vt + (size_t)bf * 16384;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int key = p & 63, w = (p >> 6) + 2 * i;  // V: a warp covers 32 keys of one word
                    uint32_t hp[4];
                    word_to_h2_pairs(vw[key * 16 + w], hp);
#pragma unroll
                    for (int jj = 0; jj < 4; ++jj) {
                        const int c = 8 * w + 2 * jj;
                        uint8_t* base = vtb + (key & 7) * 2;
                        *reinterpret_cast<uint16_t*>(base + ta_sw(c, key >> 3)) = (uint16_t)(hp[jj] & 0xFFFF);
                        *reinterpret_cast<uint16_t*>(base + ta_sw(c + 1, key >> 3)) = (uint16_t)(hp[jj] >> 16);
                    }
                }
                ta_fence_async();
                mbar_arrive(&v_full[bf]);
                // raw(j) fully read by every producer thread: its slot takes raw(j + 3)
                asm volatile("bar.sync 1, %0;\n" ::"n"(TW_PW * 32) : "memory");
                if (j + 3 < T)
                    tw_load_raw<DH>(page_base(pool, page_bytes, pt, max_pages, b, (j + 3) * TW_K), Hkv, kh,
                                    min(TW_K, S - (j + 3) * TW_K), sm + TwSmem::raw + (size_t)(j % 3) * TwSmem::raw_sz,
                                    p, 128);
                else
                    cp_async_commit();
            }
        }
    } else {
        // ---------------- softmax: query row r = TMEM lane r (warps w and w + 4 share lane quarter
        // w), half hf of the tile's 64 keys and of O's 128 columns per thread
        const int r = tid & 127, hf = tid >> 7;
        const int q = q0 + r;
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        float* xch = reinterpret_cast<float*>(sm + TwSmem::xch);  // [2][2][128]
        constexpr int HK = TW_K / 2;  // keys per thread
        float m_used = -1e30f, l = 0.f;
        for (int t = 0; t < T; ++t) {
            const int bf = t & 1;
            const uint32_t ph = (uint32_t)(t >> 1) & 1u;
            const int k0 = t * TW_K + hf * HK;
            mbar_wait(&s_full[bf], ph);
            mbar_wait(&ks_full[t & 3], (uint32_t)(t >> 2) & 1u);  // this tile's scales
            ta_fence_after();
            float s[HK];
            ta_ld32(tmem + (uint32_t)(bf * 64 + hf * HK) + lane_off, s);
            const float* ks = ksb + (t & 3) * TW_K + hf * HK;
            const float* vs = vsb + (t & 3) * TW_K + hf * HK;
            // every (query, key) pair of the tile allowed and in range: no per-element mask
            const int klast = t * TW_K + TW_K - 1, qlast = q0 + TW_Q - 1;
            const bool full = qlast < S && klast < S &&
                              (qlast < V ? klast < V : (q0 >= V && (klast < V || klast <= q0)));
            float tmax = -1e30f;
            if (full) {
#pragma unroll
                for (int j = 0; j < HK; ++j) {
                    s[j] *= ks[j];
                    tmax = fmaxf(tmax, s[j]);
                }
            } else {
#pragma unroll
                for (int j = 0; j < HK; ++j) {
                    const int kj = k0 + j;
                    const bool ok = q < S && kj < S && (q < V ? kj < V : (kj < V || kj <= q));
                    s[j] = ok ? s[j] * ks[j] : -1e30f;
                    tmax = fmaxf(tmax, s[j]);
                }
            }
            // the row's tile max from both halves (the two threads then decide identically)
            xch[(bf * 2 + hf) * 128 + r] = tmax;
            asm volatile("bar.sync 2, %0;\n" ::"n"(TW_SW * 32) : "memory");
            tmax = fmaxf(tmax, xch[(bf * 2 + (hf ^ 1)) * 128 + r]);
            const bool raise = tmax > m_used + 8.f;
            const float fac = raise ? exp2f(m_used - tmax) : 1.f;
            if (raise) {
                l *= fac;
                m_used = tmax;
            }
            if (t >= 1 && __any_sync(0xffffffffu, raise)) {  // O holds tiles < t: rescale after PV(t-1)
                mbar_wait(&pv_done[(t - 1) & 1], (uint32_t)((t - 1) >> 1) & 1u);
                ta_fence_after();
#pragma unroll 1
                for (int c = hf * 64; c < hf * 64 + 64; c += 32) {
                    float o[32];
                    ta_ld32(tO + lane_off + c, o);
#pragma unroll
                    for (int i = 0; i < 32; ++i) o[i] *= fac;
                    ta_st32(tO + lane_off + c, o);
                }
                asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
            }
            if (t >= 2) mbar_wait(&pv_done[bf], (uint32_t)((t - 2) >> 1) & 1u);  // P buffer free
            uint8_t* phb = sm + TwSmem::ph + (size_t)bf * 16384;
            uint8_t* plb = sm + TwSmem::pl + (size_t)bf * 16384;
            float psum = 0.f;
#pragma unroll
            for (int c = 0; c < HK / 8; ++c) {
                uint32_t hi[4], lo[4];
#pragma unroll
                for (int e = 0; e < 8; e += 2) {
                    const int j = 8 * c + e;
                    // masked scores (-1e30) underflow to exactly 0 (ex2.approx of < -126 flushes)
                    const float p0 = ex2_approx(s[j] - m_used);
                    const float p1 = ex2_approx(s[j + 1] - m_used);
                    psum += p0 + p1;
                    split_h2(p0 * vs[j], p1 * vs[j + 1], hi[e / 2], lo[e / 2]);
                }
                const int chunk = hf * (HK / 8) + c;
                *reinterpret_cast<uint4*>(phb + ta_sw(r, chunk)) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
                *reinterpret_cast<uint4*>(plb + ta_sw(r, chunk)) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
            }
            l += psum;
            ta_fence_async();
            ta_fence_before();
            mbar_arrive(&p_full[bf]);
        }
        // finalize: O / l over this half's 64 columns; l and the row max |out| combined across the
        // two halves; (m, l) for the QUOTA sums
        xch[512 + hf * 128 + r] = l;
        mbar_wait(&pv_done[(T - 1) & 1], (uint32_t)((T - 1) >> 1) & 1u);
        ta_fence_after();
        asm volatile("bar.sync 2, %0;\n" ::"n"(TW_SW * 32) : "memory");
        const float lt = xch[512 + r] + xch[512 + 128 + r];  // half 0 + half 1, fixed order
        const bool ok = q < S;
        const float inv_l = lt > 0.f ? 1.f / lt : 0.f;
        float* orow = out + (size_t)(tok0 + min(q, S - 1)) * ldo + h * DH;
        float mx = 0.f;
#pragma unroll 1
        for (int c = hf * 64; c < hf * 64 + 64; c += 32) {
            float o[32];
            ta_ld32(tO + lane_off + c, o);
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                o[i] *= inv_l;
                mx = fmaxf(mx, fabsf(o[i]));
            }
            if (ok)
#pragma unroll
                for (int i = 0; i < 32; i += 8) st_v8f32(orow + c + i, o + i);
        }
        xch[768 + hf * 128 + r] = mx;
        asm volatile("bar.sync 2, %0;\n" ::"n"(TW_SW * 32) : "memory");
        if (ok && hf == 0) {
            if (ml) ml[(size_t)(tok0 + q) * H + h] = make_float2(m_used * 0.69314718055994531f, lt);
            if (pmax) pmax[(size_t)(tok0 + q) * pmax_ld + h] = fmaxf(mx, xch[768 + 128 + r]);
        }
    }
    ta_fence_before();
    __syncthreads();
    if (warp == TW_MW) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" ::"r"(tmem));
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
    // d_head 128: the warp-specialised tcgen05 kernel at every batch length (A/B against the
    // mma.sync kernel from 0 / 256 / 512 tokens: equal within noise below 512, faster above);
    // d_head 64 (configs[0]): the mma.sync kernel
    if (dh == 128) {
        const dim3 gws((smax + TW_Q - 1) / TW_Q, H, B);
        cudaFuncSetAttribute(k_attn_prefill_ws, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TwSmem::total);
        k_attn_prefill_ws<<<gws, TW_THREADS, TwSmem::total, st>>>(qkv, ldq, H, Hkv, seq_off, vis, seq_len, pool,
                                                                 page_bytes, pt, max_pages, inv_sqrt, out, ldo,
                                                                 reinterpret_cast<float2*>(ml), pmax, pmax_ld);
        return (int)cudaGetLastError();
    }
    const dim3 grid((smax + AT_Q - 1) / AT_Q, H, B);
    if (dh == 64)
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
