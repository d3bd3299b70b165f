// k_quant.cu -- memory-bound quantizer kernels (HBM roofline):
//   K1  RMSNorm + symmetric int4 activation quantizer (site_quant), static
//       per-tensor or dynamic per-token scale           model.cpp:31-33,147-154,
//                                                        347-349,394,429-435,442-444
//   K5  RoPE + per-(token, kv-head) int4 KV quantize + paged append
//                                                        model.cpp:156-168,368-374,494-501
//   K3b QUOTA token magnitude / quantization-residual metrics
//                                                        selector.cpp:38,56-66
//   weight quantizer (prepare_quant_env, per output channel) model.cpp:212-237
//
// All quantizer arithmetic is fp64 (the reference's type), so an int4 code
// equals the reference code for the same fp32 input; the fp32 scale handed to
// the GEMM epilogue is the rounded fp64 scale.
#include "qt_common.cuh"
#include "qt_kernels.h"

namespace qt {

// ============================================================== K1
// One CTA per token row.  gain == nullptr: no RMSNorm (attn_out / mlp_mid sites).
// mode 0: static per-tensor scale `static_scale`; mode 1: dynamic per-row
// max|n|/qmax.  codes: packed int4 [M x ld_codes bytes], zero-padded to
// d_pad; scales: fp32 [M] (the scale each row was quantized with).
template <typename TX>
QT_DEV void load8(const TX* p, double* v);
template <>
QT_DEV void load8<float>(const float* p, double* v) {
    float4 a = *reinterpret_cast<const float4*>(p);
    float4 b = *reinterpret_cast<const float4*>(p + 4);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
template <>
QT_DEV void load8<double>(const double* p, double* v) {
#pragma unroll
    for (int j = 0; j < 8; j += 2) {
        double2 a = *reinterpret_cast<const double2*>(p + j);
        v[j] = a.x;
        v[j + 1] = a.y;
    }
}

// Register-resident: each thread owns G groups of 8 consecutive elements
// (words w = tid + j * blockDim), read once from global memory; the RMS sum
// and the row max are block reductions over those registers.
// codes: tiled int4 [rows_pad x d_pad] (ld_codes = rows_pad)
template <typename TX, int G>
__global__ void __launch_bounds__(1024) k_norm_quant(const TX* __restrict__ x, int ld_x,
                                                     const float* __restrict__ gain, int M, int D, int d_pad,
                                                     int qmax, int mode, double static_scale,
                                                     uint8_t* __restrict__ codes, int ld_codes,
                                                     double* __restrict__ scales, float* __restrict__ normed,
                                                     int8_t* __restrict__ codes8, int ld8) {
    __shared__ double red[32];
    pdl_launch_dependents();
    pdl_wait();  // x is produced by the previous kernel
    const int row = blockIdx.x;
    if (row >= M) return;
    const TX* xr = x + (size_t)row * ld_x;
    const int n_words = d_pad / 8;
    double v[G][8];
#pragma unroll
    for (int j = 0; j < G; ++j) {
        const int base = (threadIdx.x + j * blockDim.x) * 8;
        if (base < D) {
            load8<TX>(xr + base, v[j]);
        } else {
#pragma unroll
            for (int e = 0; e < 8; ++e) v[j][e] = 0.0;
        }
    }
    if (gain) {
        double ss = 0.0;
#pragma unroll
        for (int j = 0; j < G; ++j)
#pragma unroll
            for (int e = 0; e < 8; ++e) ss += v[j][e] * v[j][e];
        ss = block_sum(ss, red);
        const double inv = 1.0 / sqrt(ss / (double)D + kNormEps);
#pragma unroll
        for (int j = 0; j < G; ++j) {
            const int base = (threadIdx.x + j * blockDim.x) * 8;
            if (base < D) {
                float4 g0 = *reinterpret_cast<const float4*>(gain + base);
                float4 g1 = *reinterpret_cast<const float4*>(gain + base + 4);
                const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
#pragma unroll
                for (int e = 0; e < 8; ++e) v[j][e] = __dmul_rn(__dmul_rn(v[j][e], inv), (double)gg[e]);
            }
        }
    }
    double s;
    if (mode == 0) {
        s = static_scale;
    } else {
        double mx = 0.0;
#pragma unroll
        for (int j = 0; j < G; ++j)
#pragma unroll
            for (int e = 0; e < 8; ++e) mx = fmax(mx, fabs(v[j][e]));
        mx = block_max(mx, red);
        s = q_scale(mx, qmax);
    }
    const double inv_s = 1.0 / s;
#pragma unroll
    for (int j = 0; j < G; ++j) {
        const int w = threadIdx.x + j * blockDim.x;
        if (w >= n_words) continue;
        int c[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) c[e] = w * 8 + e < D ? q_code_r(v[j][e], s, inv_s, qmax) : 0;
        *reinterpret_cast<uint32_t*>(codes + w4t_offset(row, w * 4, ld_codes)) = pack8(c);  // tiled layout
        if (codes8) *reinterpret_cast<uint2*>(codes8 + (size_t)row * ld8 + w * 8) = pack8_i8x16(c);
        if (normed && w * 8 < D) {
#pragma unroll
            for (int e = 0; e < 8; ++e) normed[(size_t)row * D + w * 8 + e] = (float)v[j][e];
        }
    }
    if (threadIdx.x == 0) scales[row] = s;
}

// K1 for decode-sized batches: the k_norm_quant arithmetic with 4 elements per
// thread (up to 1024 threads per row): half the serial instructions per warp and
// twice the warps per SM, for a kernel whose time is its own latency chain.
template <typename TX>
__global__ void __launch_bounds__(1024) k_norm_quant4(const TX* __restrict__ x, int ld_x,
                                                      const float* __restrict__ gain, int M, int D, int d_pad,
                                                      int qmax, int mode, double static_scale,
                                                      uint8_t* __restrict__ codes, int ld_codes,
                                                      double* __restrict__ scales, int8_t* __restrict__ codes8,
                                                      int ld8) {
    __shared__ double red[32], red2[32];
    pdl_launch_dependents();
    const int row = blockIdx.x;
    const int base = threadIdx.x * 4;
    const bool in = base < D;
    // the gain is a weight: read before the dependency wait, off the critical path
    const float4 g4 = gain && in ? *reinterpret_cast<const float4*>(gain + base) : make_float4(1.f, 1.f, 1.f, 1.f);
    pdl_wait();  // x is produced by the previous kernel
    if (row >= M) return;
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    if (in) {
        const TX* xr = x + (size_t)row * ld_x + base;
        if constexpr (sizeof(TX) == 8) {
            const double2 a = reinterpret_cast<const double2*>(xr)[0], b = reinterpret_cast<const double2*>(xr)[1];
            v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
        } else {
            const float4 a = *reinterpret_cast<const float4*>(xr);
            v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
        }
    }
    if (gain) {
        double ss = 0.0;
#pragma unroll
        for (int e = 0; e < 4; ++e) ss += v[e] * v[e];
        ss = block_sum1(ss, red);
        const double inv = 1.0 / sqrt(ss / (double)D + kNormEps);
        if (in) {
            const float gg[4] = {g4.x, g4.y, g4.z, g4.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) v[e] = __dmul_rn(__dmul_rn(v[e], inv), (double)gg[e]);
        }
    }
    double s;
    if (mode == 0) {
        s = static_scale;
    } else {
        double mx = 0.0;
#pragma unroll
        for (int e = 0; e < 4; ++e) mx = fmax(mx, fabs(v[e]));
        mx = block_max1(mx, red2);
        s = q_scale(mx, qmax);
    }
    if (base < d_pad) {
        const double inv_s = 1.0 / s;
        uint32_t w = 0, w8 = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int c = in ? q_code_r(v[e], s, inv_s, qmax) : 0;
            w |= (uint32_t)(c & 0xF) << (4 * e);
            w8 |= (uint32_t)((c << 4) & 0xFF) << (8 * e);
        }
        *reinterpret_cast<uint16_t*>(codes + w4t_offset(row, base / 2, ld_codes)) = (uint16_t)w;
        if (codes8) *reinterpret_cast<uint32_t*>(codes8 + (size_t)row * ld8 + base) = w8;
    }
    if (threadIdx.x == 0) scales[row] = s;
}

// K1 without a row reduction: the row max |x| of an fp32 site input (mlp_mid,
// attn_out) arrives as the producing kernel's partial maxima (pmax[m][p], p <
// n_part; max is exact, so the scale is the one a full reduction gives).  Each
// thread quantizes WPT 8-element words (w = tid + j * 256 within the CTA's
// chunk), all loads issued first; every warp folds the row's partials itself, so
// no block barrier sits between the loads and the stores.  Grid (chunks, M).
template <int WPT>
__global__ void __launch_bounds__(256) k_quant_pmax(const float* __restrict__ x, int ld_x,
                                                    const float* __restrict__ pmax, int n_part, int pmax_ld, int M,
                                                    int D, int d_pad, int qmax, int mode, double static_scale,
                                                    uint8_t* __restrict__ codes, int ld_codes,
                                                    double* __restrict__ scales, int8_t* __restrict__ codes8,
                                                    int ld8) {
    pdl_launch_dependents();
    pdl_wait();  // x and the partials come from the previous kernel
    const int row = blockIdx.y, lane = threadIdx.x & 31;
    if (row >= M) return;
    const int w0 = blockIdx.x * (256 * WPT) + threadIdx.x;
    float4 v[WPT][2];  // fp32 site input as loaded (widened to fp64 at the quantizer)
#pragma unroll
    for (int j = 0; j < WPT; ++j)
        if ((w0 + j * 256) * 8 < D) {
            const float4* p = reinterpret_cast<const float4*>(x + (size_t)row * ld_x + (w0 + j * 256) * 8);
            v[j][0] = p[0];
            v[j][1] = p[1];
        }
    double s = static_scale;
    if (mode != 0 && n_part <= 32) {  // few partials (decode: one reduced slot): every warp folds
        const float mx = warp_max(lane < n_part ? pmax[(size_t)row * pmax_ld + lane] : 0.f);
        s = q_scale((double)mx, qmax);
    } else if (mode != 0) {  // warp 0 folds the row's partials (loads above already in flight); smem broadcast
        __shared__ float s_mx;
        if (threadIdx.x < 32) {
            float mx = 0.f;
            for (int p = lane; p < n_part; p += 32) mx = fmaxf(mx, pmax[(size_t)row * pmax_ld + p]);
            mx = warp_max(mx);
            if (lane == 0) s_mx = mx;
        }
        __syncthreads();
        s = q_scale((double)s_mx, qmax);
    }
    const double inv_s = 1.0 / s;
#pragma unroll
    for (int j = 0; j < WPT; ++j) {
        const int w = w0 + j * 256;
        if (w * 8 >= d_pad) break;
        const bool in = w * 8 < D;
        int c[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const float4 q4 = v[j][e >> 2];
            const float f = (e & 3) == 0 ? q4.x : (e & 3) == 1 ? q4.y : (e & 3) == 2 ? q4.z : q4.w;
            c[e] = in ? q_code_r((double)f, s, inv_s, qmax) : 0;
        }
        *reinterpret_cast<uint32_t*>(codes + w4t_offset(row, w * 4, ld_codes)) = pack8(c);
        if (codes8) *reinterpret_cast<uint2*>(codes8 + (size_t)row * ld8 + w * 8) = pack8_i8x16(c);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) scales[row] = s;
}

// ============================================================== K5
// One CTA per token.  qkv row layout: [q (H*dh) | k (Hkv*dh) | v (Hkv*dh)],
// fp32, ld = ld_qkv.  RoPE (interleaved pairs, model.cpp:156-168) is applied to
// q in place and to k, with the cos/sin table computed on the host with the
// reference's own libm calls.  k and v rows of each kv head are then
// quantized per (token, head) (kv_quantize, quant.cpp:117-119) and appended
// into the paged cache at (page_table[seq][row / kPage], row % kPage).
__global__ void __launch_bounds__(256) k_rope_kv_append(
    float* __restrict__ qkv, int ld_qkv, int M, int H, int Hkv, int dh, const int* __restrict__ pos,
    const int* __restrict__ tok_seq, const int* __restrict__ tok_row, const double2* __restrict__ rope,
    const int* __restrict__ page_table, int max_pages, uint8_t* __restrict__ pool, long long page_bytes,
    int qmax, float* __restrict__ k_dbg) {
    pdl_launch_dependents();
    const int m = blockIdx.x;
    if (m >= M) {
        pdl_wait();
        return;
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int t = blockIdx.y * nw + wid;  // head slot: q heads, k heads, v heads
    if (t >= H + 2 * Hkv) {
        pdl_wait();
        return;
    }
    const int E = dh / 32;  // elements per lane (2 or 4)
    // positions, rows, page table and the cos/sin table are final before the upstream kernels
    // run: host uploads (each followed by a full, non-programmatic dependency -- this also
    // orders the prefill's compaction gather of the positions), or the decode step's bump at
    // the end of the previous step.  Read them before the dependency wait, qkv after it.
    const int p = pos[m];
    const double2* rt = rope + (size_t)p * (dh / 2);
    float* row = qkv + (size_t)m * ld_qkv;
    const int b = tok_seq[m], r = tok_row[m];
    uint8_t* page = pool + (long long)page_table[b * max_pages + r / kPage] * page_bytes;
    const int slot = r % kPage;
    const size_t codes_bytes = (size_t)Hkv * kPage * (dh / 2);
    double2 csv[2] = {make_double2(1.0, 0.0), make_double2(1.0, 0.0)};
    if (t < H + Hkv) {
#pragma unroll
        for (int j = 0; j < 4; j += 2)
            if (j < E) csv[j / 2] = rt[(lane * E + j) / 2];
    }
    pdl_wait();
    {
        float* v = row + t * dh;  // q heads, then k heads, then v heads: contiguous
        double val[4];
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (j < E) val[j] = (double)v[lane * E + j];
        if (t < H + Hkv) {  // rope q and k
#pragma unroll
            for (int j = 0; j < 4; j += 2) {
                if (j < E) {
                    const double2 cs = csv[j / 2];
                    double a = val[j], bb = val[j + 1];
                    val[j] = __dsub_rn(__dmul_rn(a, cs.x), __dmul_rn(bb, cs.y));
                    val[j + 1] = __dadd_rn(__dmul_rn(a, cs.y), __dmul_rn(bb, cs.x));
                }
            }
        }
        if (t < H) {
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (j < E) v[lane * E + j] = (float)val[j];
            return;
        }
        // k or v head: quantize per (token, head)
        double mx = 0.0;
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (j < E) mx = fmax(mx, fabs(val[j]));
        mx = warp_max(mx);
        const double s = q_scale(mx, qmax), inv_s = 1.0 / s;
        const bool is_k = t < H + Hkv;
        const int kh = is_k ? t - H : t - H - Hkv;
        if (is_k && k_dbg) {
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (j < E) k_dbg[(size_t)m * Hkv * dh + kh * dh + lane * E + j] = (float)val[j];
        }
        int c[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) c[j] = j < E ? q_code_r(val[j], s, inv_s, qmax) : 0;
        uint8_t* dst = page + (is_k ? 0 : codes_bytes) + ((size_t)kh * kPage + slot) * (dh / 2) + lane * E / 2;
        if (E == 4) {
            uint16_t pk = (uint16_t)((c[0] & 0xF) | ((c[1] & 0xF) << 4) | ((c[2] & 0xF) << 8) | ((c[3] & 0xF) << 12));
            *reinterpret_cast<uint16_t*>(dst) = pk;
        } else {
            *dst = (uint8_t)((c[0] & 0xF) | ((c[1] & 0xF) << 4));
        }
        if (lane == 0) {
            float* sc = reinterpret_cast<float*>(page + 2 * codes_bytes) + (is_k ? 0 : Hkv * kPage);
            sc[kh * kPage + slot] = (float)s;
        }
    }
}

// K5 for token-rich launches (prefill), d_head = 128: one CTA per token, its 8
// warps loop over the token's head slots, 4 at a time with every load of the
// group issued first (float4 per lane); the RoPE cos/sin of the token's position
// are read once per lane and reused by every q and k head.  Same arithmetic as
// k_rope_kv_append.
#ifndef QT_KVTOK_G
#define QT_KVTOK_G 4
#endif
__global__ void __launch_bounds__(256) k_rope_kv_append_tok(
    float* __restrict__ qkv, int ld_qkv, int M, int H, int Hkv, const int* __restrict__ pos,
    const int* __restrict__ tok_seq, const int* __restrict__ tok_row, const double2* __restrict__ rope,
    const int* __restrict__ page_table, int max_pages, uint8_t* __restrict__ pool, long long page_bytes, int qmax) {
    constexpr int DH = 128, E = 4, G = QT_KVTOK_G;
    pdl_launch_dependents();
    pdl_wait();
    const int m = blockIdx.x;
    if (m >= M) return;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const double2* rt = rope + (size_t)pos[m] * (DH / 2);
    const double2 cs0 = rt[lane * 2], cs1 = rt[lane * 2 + 1];
    float* row = qkv + (size_t)m * ld_qkv;
    const int b = tok_seq[m], r = tok_row[m];
    uint8_t* page = pool + (long long)page_table[b * max_pages + r / kPage] * page_bytes;
    const int slot = r % kPage;
    const size_t codes_bytes = (size_t)Hkv * kPage * (DH / 2);
    const int nt = H + 2 * Hkv;
    for (int t0 = wid; t0 < nt; t0 += 8 * G) {
        float4 x4[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const int t = t0 + 8 * g;
            x4[g] = t < nt ? *reinterpret_cast<const float4*>(row + t * DH + lane * E) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const int t = t0 + 8 * g;
            if (t >= nt) break;
            double val[4] = {(double)x4[g].x, (double)x4[g].y, (double)x4[g].z, (double)x4[g].w};
            if (t < H + Hkv) {  // rope q and k
                double a = val[0], bb = val[1];
                val[0] = __dsub_rn(__dmul_rn(a, cs0.x), __dmul_rn(bb, cs0.y));
                val[1] = __dadd_rn(__dmul_rn(a, cs0.y), __dmul_rn(bb, cs0.x));
                a = val[2];
                bb = val[3];
                val[2] = __dsub_rn(__dmul_rn(a, cs1.x), __dmul_rn(bb, cs1.y));
                val[3] = __dadd_rn(__dmul_rn(a, cs1.y), __dmul_rn(bb, cs1.x));
            }
            if (t < H) {
                *reinterpret_cast<float4*>(row + t * DH + lane * E) =
                    make_float4((float)val[0], (float)val[1], (float)val[2], (float)val[3]);
                continue;
            }
            double mx = fmax(fmax(fabs(val[0]), fabs(val[1])), fmax(fabs(val[2]), fabs(val[3])));
            mx = warp_max(mx);
            const double sc = q_scale(mx, qmax), inv_s = 1.0 / sc;
            const bool is_k = t < H + Hkv;
            const int kh = is_k ? t - H : t - H - Hkv;
            int c[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) c[j] = q_code_r(val[j], sc, inv_s, qmax);
            uint8_t* dst = page + (is_k ? 0 : codes_bytes) + ((size_t)kh * kPage + slot) * (DH / 2) + lane * E / 2;
            *reinterpret_cast<uint16_t*>(dst) =
                (uint16_t)((c[0] & 0xF) | ((c[1] & 0xF) << 4) | ((c[2] & 0xF) << 8) | ((c[3] & 0xF) << 12));
            if (lane == 0) {
                float* scp = reinterpret_cast<float*>(page + 2 * codes_bytes) + (is_k ? 0 : Hkv * kPage);
                scp[kh * kPage + slot] = (float)sc;
            }
        }
    }
}

// ============================================================== K3b
// QUOTA per-visual-token metrics on the post-attention residual x
// (selector.cpp:19-68): mag = ||x_i||_2, res = ||fq_row(x_i) - x_i||_2 with
// the per-row quantizer fake_quant_per_row (quant.cpp:108-110).  grid (Vmax, B).
__global__ void __launch_bounds__(256) k_token_metrics(const double* __restrict__ x, int D,
                                                       const int* __restrict__ seq_off,
                                                       const int* __restrict__ vis, int vstride, int qmax,
                                                       int with_res, double* __restrict__ mag,
                                                       double* __restrict__ res) {
    __shared__ double red[32];
    const int b = blockIdx.y, i = blockIdx.x;
    if (i >= vis[b]) return;
    const double* xr = x + (size_t)(seq_off[b] + i) * D;
    double ss = 0.0, mx = 0.0;
    for (int j = threadIdx.x; j < D; j += blockDim.x) {
        double v = xr[j];
        ss += v * v;
        mx = fmax(mx, fabs(v));
    }
    ss = block_sum(ss, red);
    double rr = 0.0;
    if (with_res) {
        mx = block_max(mx, red);
        const double s = q_scale(mx, qmax);
        for (int j = threadIdx.x; j < D; j += blockDim.x) {
            double v = xr[j];
            double d = __dsub_rn(__dmul_rn((double)q_code(v, s, qmax), s), v);
            rr += d * d;
        }
        rr = block_sum(rr, red);
    }
    if (threadIdx.x == 0) {
        mag[(size_t)b * vstride + i] = sqrt(ss);
        res[(size_t)b * vstride + i] = with_res ? sqrt(rr) : 0.0;
    }
}

// ============================================================== weights
// prepare_quant_env for one weight W[K x N] given in the reference orientation
// (row-major d_in x d_out, y = x W).  One scale per output column n
// (GroupAxis::PerColumn, quant.cpp:15-31): s_n = max_k |W[k][n]| / qmax.
// Output: packed codes [N_pad x ldc] (row n = column n of W, K contiguous,
// zero-padded), fp32 scales.  dst_row maps column n to its storage row
// (identity, or the gate/up interleave for SwiGLU).
__global__ void k_weight_colmax(const float* __restrict__ w, int K, int N, double* __restrict__ colmax) {
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= N) return;
    double m = 0.0;
    for (int k = 0; k < K; ++k) m = fmax(m, fabs((double)w[(size_t)k * N + n]));
    colmax[n] = m;
}

__global__ void k_weight_pack(const float* __restrict__ w, int K, int N, const double* __restrict__ colmax,
                              int qmax, int row_mul, int row_add, uint8_t* __restrict__ codes, int ldc,
                              double* __restrict__ scales) {
    // thread per (n, word of 8 k)
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    const int wd = blockIdx.y;
    if (n >= N) return;
    const double s = q_scale(colmax[n], qmax);
    int c[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        int k = wd * 8 + j;
        c[j] = k < K ? q_code((double)w[(size_t)k * N + n], s, qmax) : 0;
    }
    const int dst = n * row_mul + row_add;
    *reinterpret_cast<uint32_t*>(codes + w4t_offset(dst, wd * 4, ldc)) = pack8(c);  // tiled layout
    if (wd == 0) scales[dst] = s;
}

// Pre-quantized weights (a QuantEnv's int8 codes, GroupAxis::PerColumn, reference
// orientation K x N row-major) into the tiled int4 layout, scales copied per row.
__global__ void k_codes_pack(const int8_t* __restrict__ src, int K, int N, const double* __restrict__ s_in,
                             int row_mul, int row_add, uint8_t* __restrict__ codes, int ldc,
                             double* __restrict__ scales) {
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    const int wd = blockIdx.y;
    if (n >= N) return;
    int c[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        int k = wd * 8 + j;
        c[j] = k < K ? (int)src[(size_t)k * N + n] : 0;
    }
    const int dst = n * row_mul + row_add;
    *reinterpret_cast<uint32_t*>(codes + w4t_offset(dst, wd * 4, ldc)) = pack8(c);
    if (wd == 0) scales[dst] = s_in[n];
}

// tiled int4 codes (w4t layout) -> row-major int8 [rows x K] (parity readback, qt_unpack_codes)
__global__ void k_unpack_codes(const uint8_t* __restrict__ tiled, int rows_pad, int rows, int K,
                               int8_t* __restrict__ out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;  // one packed byte
    if (i >= (long long)rows * (K / 2)) return;
    const int row = (int)(i / (K / 2)), kb = (int)(i % (K / 2));
    const uint8_t b = tiled[w4t_offset(row, kb, rows_pad)];
    char2 v;
    v.x = (char)(((int)(b << 28)) >> 28);
    v.y = (char)(((int)(b << 24)) >> 28);
    reinterpret_cast<char2*>(out)[i] = v;
}

__global__ void k_f32_to_f64(const float* __restrict__ a, double* __restrict__ b, long long n) {
    pdl_launch_dependents();
    pdl_wait();
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) b[i] = (double)a[i];
}

}  // namespace qt

// ---------------------------------------------------------------- launchers
using namespace qt;

extern "C" {

int qt_launch_f32_to_f64(const float* a, double* b, long long n, cudaStream_t st) {
    if (n <= 0) return 0;
    return launch_pdl(k_f32_to_f64, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, st, a, b, n);
}

int qt_launch_norm_quant(const void* x, int x_is_f64, int ld_x, const float* gain, int M, int D, int d_pad,
                         int bits, int mode, double static_scale, uint8_t* codes, int ld_codes, double* scales,
                         float* normed, int8_t* codes8, int ld8, cudaStream_t st) {
    if (M <= 0) return 0;
    if (D % 8 || d_pad % 8 || ld_x % 4) return -1;
    const int qmax = (1 << (bits - 1)) - 1;
    // decode-sized batches: 4 elements per thread (prefill sizes measured slower with it)
    if (M <= 64 && !normed && d_pad / 4 <= 1024 && d_pad / 4 >= 128) {
        const int th = (d_pad / 4 + 31) / 32 * 32;
        if (x_is_f64)
            return launch_pdl(k_norm_quant4<double>, dim3(M), dim3(th), 0, st, static_cast<const double*>(x), ld_x,
                              gain, M, D, d_pad, qmax, mode, static_scale, codes, ld_codes, scales, codes8, ld8);
        return launch_pdl(k_norm_quant4<float>, dim3(M), dim3(th), 0, st, static_cast<const float*>(x), ld_x, gain,
                          M, D, d_pad, qmax, mode, static_scale, codes, ld_codes, scales, codes8, ld8);
    }
    const int words = d_pad / 8;
    int threads = words <= 256 ? 256 : (words <= 512 ? 512 : 1024);
    // token-rich launches: narrower CTAs holding more of the row per thread, so more rows
    // (and their loads) are in flight per SM (128 threads with G = 4 spills)
    if (M >= 256 && (words + 255) / 256 <= 4) threads = 256;
    const int G = (words + threads - 1) / threads;
    if (G > 4) return -1;
#define QT_NQ(TX, GG)                                                                                        \
    return launch_pdl(k_norm_quant<TX, GG>, dim3(M), dim3(threads), 0, st, static_cast<const TX*>(x), ld_x, \
                      gain, M, D, d_pad, qmax, mode, static_scale, codes, ld_codes, scales, normed, codes8, ld8)
    if (x_is_f64) {
        if (G == 1) QT_NQ(double, 1);
        if (G == 2) QT_NQ(double, 2);
        if (G == 3) QT_NQ(double, 3);
        QT_NQ(double, 4);
    } else {
        if (G == 1) QT_NQ(float, 1);
        if (G == 2) QT_NQ(float, 2);
        if (G == 3) QT_NQ(float, 3);
        QT_NQ(float, 4);
    }
#undef QT_NQ
}

int qt_launch_quant_pmax(const float* x, int ld_x, const float* pmax, int n_part, int pmax_ld, int M, int D,
                         int d_pad, int qmax, int mode, double static_scale, uint8_t* codes, int ld_codes,
                         double* scales, int8_t* codes8, int ld8, cudaStream_t st) {
    if (M <= 0) return 0;
    if (D % 8 || d_pad % 8 || (mode != 0 && n_part < 1)) return -1;
    const int words = d_pad / 8;
    // one word per thread: measured faster than whole-row CTAs with 2-8 words per thread
    // (prefill 36.5 vs 36.8 ms) -- more CTAs in flight beat the amortised partial fold
    return launch_pdl(k_quant_pmax<1>, dim3((words + 255) / 256, M), dim3(256), 0, st, x, ld_x, pmax, n_part, pmax_ld,
                      M, D, d_pad, qmax, mode, static_scale, codes, ld_codes, scales, codes8, ld8);
}

int qt_launch_rope_kv_append(float* qkv, int ld_qkv, int M, int H, int Hkv, int dh, const int* pos,
                             const int* tok_seq, const int* tok_row, const double* rope, const int* page_table,
                             int max_pages, uint8_t* pool, long long page_bytes, int bits, float* k_dbg,
                             cudaStream_t st) {
    if (M <= 0) return 0;
    if (dh != 64 && dh != 128) return -1;
    const int qmax = (1 << (bits - 1)) - 1;
    if (dh == 128 && M >= 64 && !k_dbg)
        return launch_pdl(k_rope_kv_append_tok, dim3(M), dim3(256), 0, st, qkv, ld_qkv, M, H, Hkv, pos, tok_seq,
                          tok_row, reinterpret_cast<const double2*>(rope), page_table, max_pages, pool, page_bytes,
                          qmax);
    return launch_pdl(k_rope_kv_append, dim3(M, (H + 2 * Hkv + 7) / 8), dim3(256), 0, st, qkv, ld_qkv, M, H, Hkv,
                      dh, pos, tok_seq, tok_row, reinterpret_cast<const double2*>(rope), page_table, max_pages, pool,
                      page_bytes, qmax, k_dbg);
}

int qt_launch_unpack_codes(const uint8_t* tiled, int rows_pad, int rows, int K, int8_t* out, cudaStream_t st) {
    const long long n = (long long)rows * (K / 2);
    if (n <= 0) return 0;
    k_unpack_codes<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(tiled, rows_pad, rows, K, out);
    return (int)cudaGetLastError();
}

int qt_launch_token_metrics(const double* x, int D, const int* seq_off, const int* vis, int vmax, int B,
                            int vstride, int res_bits, double* mag, double* res, cudaStream_t st) {
    if (vmax <= 0 || B <= 0) return 0;
    const int qmax = res_bits > 0 ? (1 << (res_bits - 1)) - 1 : 7;
    k_token_metrics<<<dim3(vmax, B), 256, 0, st>>>(x, D, seq_off, vis, vstride, qmax, res_bits > 0, mag, res);
    return (int)cudaGetLastError();
}

int qt_launch_codes_pack(const int8_t* src, int K, int N, const double* s_in, int row_mul, int row_add,
                         uint8_t* codes, int ldc, double* scales, cudaStream_t st) {
    const int words = (K + 7) / 8;
    k_codes_pack<<<dim3((N + 127) / 128, words), 128, 0, st>>>(src, K, N, s_in, row_mul, row_add, codes, ldc,
                                                                scales);
    return (int)cudaGetLastError();
}

int qt_launch_weight_quant(const float* w, int K, int N, int bits, int row_mul, int row_add, uint8_t* codes,
                           int ldc, double* scales, double* colmax_scratch, cudaStream_t st) {
    const int qmax = (1 << (bits - 1)) - 1;
    k_weight_colmax<<<(N + 127) / 128, 128, 0, st>>>(w, K, N, colmax_scratch);
    const int words = (K + 7) / 8;
    k_weight_pack<<<dim3((N + 127) / 128, words), 128, 0, st>>>(w, K, N, colmax_scratch, qmax, row_mul, row_add,
                                                                 codes, ldc, scales);
    return (int)cudaGetLastError();
}

}  // extern "C"
