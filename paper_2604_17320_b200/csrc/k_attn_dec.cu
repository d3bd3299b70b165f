// k_attn_dec.cu -- the decode attention block as ONE kernel (model.cpp:479-539):
//
//   per (sequence b, kv head g) CTA, 8 warps:
//     1. RoPE of q (the group's query heads) and k at next_position, in fp64
//        with the reference's cos/sin table (model.cpp:156-168, 494-496);
//     2. per-(token, head) int4 quantization of k and v (kv_quantize,
//        quant.cpp:117-119) appended at row len into the paged cache;
//     3. attention of each query head over rows 0..len (model.cpp:515-535):
//        every warp owns 32-row blocks, a lane quad owns a row (16 bytes of
//        int4 codes per lane, 128-bit loads), all loads of a block issued
//        before any math, dequantised in registers, online softmax, a fixed
//        order merge across quads and warps -> no split / merge kernels;
//     4. the LAST CTA of sequence b (a per-sequence arrival counter, reset by
//        that CTA) quantizes the whole attention row for the attn_out site
//        (model.cpp:539) -> tiled int4 codes + scale for the O projection.
//
// Replaces k_rope_kv_append + k_attn_decode + k_attn_merge_quant at decode
// (three launches and two HBM round trips of partials).  The attention row
// and the codes are bit-compatible with the unfused path's arithmetic up to
// fp32 summation order.
#include "qt_common.cuh"
#include "qt_kernels.h"

namespace qt {

constexpr int AD_THREADS = 256;

template <int DH>
__global__ void __launch_bounds__(AD_THREADS) k_attn_dec_fused(
    float* __restrict__ qkv, int ldq, int H, int Hkv, const int* __restrict__ pos, const int* __restrict__ kv_len,
    const double2* __restrict__ rope, const int* __restrict__ pt, int max_pages, uint8_t* __restrict__ pool,
    long long page_bytes, float* __restrict__ attn, int d, unsigned* __restrict__ seq_cnt, uint8_t* __restrict__ codes,
    int ld_codes, double* __restrict__ scales, int qmode, double static_scale, int d_pad, int qmax) {
    constexpr int CPL = DH / 4;  // channels per lane (4 lanes per row)
    constexpr int R = 4;         // rows per lane quad per block
    extern __shared__ __align__(16) float smf[];
    float* sm_ml = smf;                 // [8][2]
    float* sm_o = smf + 16;             // [8][DH]
    float* qs = sm_o + 8 * DH;          // [DH] roped query of the current head
    int* spt = reinterpret_cast<int*>(qs + DH);  // page table of this sequence
    __shared__ double red[32];
    __shared__ int s_last;
    pdl_launch_dependents();
    pdl_wait();
    const int kh = blockIdx.x, b = blockIdx.y;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int q4 = lane & 3, quad = lane >> 2;
    const int hpg = H / Hkv;
    const int p = pos[b];
    const int r = kv_len[b];  // row of the new token
    const int len = r + 1;
    const double2* rt = rope + (size_t)p * (DH / 2);
    float* row = qkv + (size_t)b * ldq;
    const size_t cb = (size_t)Hkv * kPage * (DH / 2);
    for (int j = threadIdx.x; j < (len + kPage - 1) / kPage; j += AD_THREADS) spt[j] = pt[b * max_pages + j];
    // ---- 2. K (warp 0) and V (warp 1) of this kv head: RoPE k, quantize, append
    if (warp < 2) {
        constexpr int E = DH / 32;
        const bool is_k = warp == 0;
        const float* src = row + (is_k ? H * DH : (H + Hkv) * DH) + kh * DH;
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
        const double s = q_scale(mx, qmax), inv_s = 1.0 / s;
        int c[4] = {0, 0, 0, 0};
#pragma unroll
        for (int j = 0; j < E; ++j) c[j] = q_code_r(val[j], s, inv_s, qmax);
        uint8_t* page = pool + (long long)pt[b * max_pages + r / kPage] * page_bytes;
        uint8_t* dst = page + (is_k ? 0 : cb) + ((size_t)kh * kPage + r % kPage) * (DH / 2) + lane * E / 2;
        if (E == 4) {
            *reinterpret_cast<uint16_t*>(dst) =
                (uint16_t)((c[0] & 0xF) | ((c[1] & 0xF) << 4) | ((c[2] & 0xF) << 8) | ((c[3] & 0xF) << 12));
        } else {
            *dst = (uint8_t)((c[0] & 0xF) | ((c[1] & 0xF) << 4));
        }
        if (lane == 0) {
            float* sc = reinterpret_cast<float*>(page + 2 * cb) + (is_k ? 0 : Hkv * kPage);
            sc[kh * kPage + r % kPage] = (float)s;
        }
    }
    __syncthreads();  // the new row and the page table are visible to the block
    const float inv_sqrt = (float)(1.0 / sqrt((double)DH));
    for (int hh = 0; hh < hpg; ++hh) {
        const int h = kh * hpg + hh;
        // ---- 1. RoPE of q_h (fp64, rounded to fp32 like the unfused path)
        if (threadIdx.x < DH / 2) {
            const int i = threadIdx.x;
            const double a = (double)row[h * DH + 2 * i], bb = (double)row[h * DH + 2 * i + 1];
            const double2 cs = rt[i];
            qs[2 * i] = (float)__dsub_rn(__dmul_rn(a, cs.x), __dmul_rn(bb, cs.y));
            qs[2 * i + 1] = (float)__dadd_rn(__dmul_rn(a, cs.y), __dmul_rn(bb, cs.x));
        }
        __syncthreads();
        float q[CPL];
#pragma unroll
        for (int c = 0; c < CPL; ++c) q[c] = qs[q4 * CPL + c];
        // ---- 3. attention over rows 0..len
        float m = -1e30f, lsum = 0.f;
        float o[CPL];
#pragma unroll
        for (int c = 0; c < CPL; ++c) o[c] = 0.f;
        for (int r0 = warp * 32; r0 < len; r0 += 256) {
            uint32_t kw[R][CPL / 8], vw[R][CPL / 8];
            float sk[R], sv[R];
#pragma unroll
            for (int i = 0; i < R; ++i) {
                const int rr = r0 + quad + 8 * i;
                const bool valid = rr < len;
                const uint8_t* pg = pool + (long long)spt[valid ? rr / kPage : 0] * page_bytes;
                const int slot = valid ? rr % kPage : 0;
                const uint8_t* krow = pg + ((size_t)kh * kPage + slot) * (DH / 2) + q4 * (CPL / 2);
                if (CPL == 32) {
                    const uint4 ka = valid ? *reinterpret_cast<const uint4*>(krow) : make_uint4(0, 0, 0, 0);
                    const uint4 va = valid ? *reinterpret_cast<const uint4*>(krow + cb) : make_uint4(0, 0, 0, 0);
                    kw[i][0] = ka.x; kw[i][1] = ka.y; kw[i][2] = ka.z; kw[i][3] = ka.w;
                    vw[i][0] = va.x; vw[i][1] = va.y; vw[i][2] = va.z; vw[i][3] = va.w;
                } else {
                    const uint2 ka = valid ? *reinterpret_cast<const uint2*>(krow) : make_uint2(0, 0);
                    const uint2 va = valid ? *reinterpret_cast<const uint2*>(krow + cb) : make_uint2(0, 0);
                    kw[i][0] = ka.x; kw[i][1] = ka.y;
                    vw[i][0] = va.x; vw[i][1] = va.y;
                }
                const float* scp = reinterpret_cast<const float*>(pg + 2 * cb);
                sk[i] = valid ? scp[kh * kPage + slot] : 0.f;
                sv[i] = valid ? scp[Hkv * kPage + kh * kPage + slot] : 0.f;
            }
#pragma unroll
            for (int i = 0; i < R; ++i) {
                const bool valid = r0 + quad + 8 * i < len;
                float dsum = 0.f;
#pragma unroll
                for (int w = 0; w < CPL / 8; ++w)
#pragma unroll
                    for (int e = 0; e < 8; ++e) dsum = fmaf(q[w * 8 + e], (float)nib(kw[i][w], e), dsum);
                dsum += __shfl_xor_sync(0xffffffffu, dsum, 1);
                dsum += __shfl_xor_sync(0xffffffffu, dsum, 2);
                if (valid) {
                    const float sc = dsum * sk[i] * inv_sqrt;
                    const float mn = fmaxf(m, sc);
                    const float al = expf(m - mn), pr = expf(sc - mn);
                    lsum = lsum * al + pr;
                    const float pv = pr * sv[i];
#pragma unroll
                    for (int w = 0; w < CPL / 8; ++w)
#pragma unroll
                        for (int e = 0; e < 8; ++e) o[w * 8 + e] = fmaf(pv, (float)nib(vw[i][w], e), o[w * 8 + e] * al);
                    m = mn;
                }
            }
        }
        // merge the 8 quads of the warp (fixed butterfly order)
#pragma unroll
        for (int off = 4; off < 32; off <<= 1) {
            const float mo = __shfl_xor_sync(0xffffffffu, m, off);
            const float lo = __shfl_xor_sync(0xffffffffu, lsum, off);
            const float mn = fmaxf(m, mo);
            const float a1 = lsum > 0.f ? expf(m - mn) : 0.f, a2 = lo > 0.f ? expf(mo - mn) : 0.f;
            lsum = lsum * a1 + lo * a2;
#pragma unroll
            for (int c = 0; c < CPL; ++c) {
                const float ao = __shfl_xor_sync(0xffffffffu, o[c], off);
                o[c] = o[c] * a1 + ao * a2;
            }
            m = mn;
        }
        if (quad == 0) {
#pragma unroll
            for (int c = 0; c < CPL; ++c) sm_o[warp * DH + q4 * CPL + c] = o[c];
            if (q4 == 0) {
                sm_ml[warp * 2] = m;
                sm_ml[warp * 2 + 1] = lsum;
            }
        }
        __syncthreads();
        if (threadIdx.x < DH) {
            float mm = -1e30f;
            for (int w = 0; w < 8; ++w)
                if (sm_ml[w * 2 + 1] > 0.f) mm = fmaxf(mm, sm_ml[w * 2]);
            float ll = 0.f, oo = 0.f;
            for (int w = 0; w < 8; ++w) {
                const float a = sm_ml[w * 2 + 1] > 0.f ? expf(sm_ml[w * 2] - mm) : 0.f;
                ll += sm_ml[w * 2 + 1] * a;
                oo += sm_o[w * DH + threadIdx.x] * a;
            }
            attn[(size_t)b * d + h * DH + threadIdx.x] = oo / ll;
        }
        __syncthreads();
    }
    // ---- 4. the last CTA of sequence b quantizes the attention row (attn_out site)
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned old = atomicAdd(&seq_cnt[b], 1u);
        s_last = old == (unsigned)(Hkv - 1);
        if (s_last) seq_cnt[b] = 0;  // ready for the next step / graph replay
        __threadfence();
    }
    __syncthreads();
    if (!s_last) return;
    const float* ar = attn + (size_t)b * d;
    double mx = 0.0;
    for (int n = threadIdx.x; n < d; n += AD_THREADS) mx = fmax(mx, fabs((double)__ldcg(ar + n)));
    double s = static_scale;
    if (qmode == 1) s = q_scale(block_max(mx, red), qmax);
    const double inv_s = 1.0 / s;
    for (int w = threadIdx.x; w * 8 < d_pad; w += AD_THREADS) {
        int c[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) c[e] = w * 8 + e < d ? q_code_r((double)__ldcg(ar + w * 8 + e), s, inv_s, qmax) : 0;
        *reinterpret_cast<uint32_t*>(codes + w4t_offset(b, w * 4, ld_codes)) = pack8(c);
    }
    if (threadIdx.x == 0) scales[b] = s;
}

}  // namespace qt

using namespace qt;

extern "C" int qt_launch_attn_dec_fused(float* qkv, int ldq, int H, int Hkv, int dh, const int* pos,
                                        const int* kv_len, const double* rope, const int* pt, int max_pages,
                                        uint8_t* pool, long long page_bytes, float* attn, int d, unsigned* seq_cnt,
                                        uint8_t* codes, int ld_codes, double* scales, int qmode, double static_scale,
                                        int d_pad, int bits, int B, cudaStream_t st) {
    if (B <= 0) return 0;
    if (H % Hkv) return -1;
    const int qmax = (1 << (bits - 1)) - 1;
    const size_t smem = (size_t)(16 + 9 * dh) * sizeof(float) + (size_t)max_pages * sizeof(int) + 16;
    const dim3 grid(Hkv, B);
    const double2* rt = reinterpret_cast<const double2*>(rope);
    if (dh == 128)
        return launch_pdl(k_attn_dec_fused<128>, grid, dim3(AD_THREADS), smem, st, qkv, ldq, H, Hkv, pos, kv_len, rt,
                          pt, max_pages, pool, page_bytes, attn, d, seq_cnt, codes, ld_codes, scales, qmode,
                          static_scale, d_pad, qmax);
    if (dh == 64)
        return launch_pdl(k_attn_dec_fused<64>, grid, dim3(AD_THREADS), smem, st, qkv, ldq, H, Hkv, pos, kv_len, rt, pt,
                          max_pages, pool, page_bytes, attn, d, seq_cnt, codes, ld_codes, scales, qmode, static_scale,
                          d_pad, qmax);
    return -1;
}
