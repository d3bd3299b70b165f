// k_select.cu -- QUOTA budgeted selection and compaction.
//
//   K3c robust normalisation + fusion (selector.cpp:70-115; percentile
//       numeric.cpp:84-96): each metric clipped to [P5, P95] and rescaled to
//       [0, 1] (flat -> 0.5), fused with the recipe weights.  fp64, no FMA
//       contraction, so the fused score equals the reference's for the same
//       metrics.
//   K4  deterministic top-k (selector.cpp:117-136): the K largest fused scores,
//       ties to the smaller index, emitted ascending.  Radix select over
//       order-preserving 64-bit keys (8 passes of 8 bits) + block prefix sums,
//       no sort; then the keep list of apply_pruning (selector.cpp:138-160):
//       retained visual slots followed by every text row.
//       Gathers that rewrite the hidden states / position ids, and the in-place
//       filter of the pruning layer's KV rows (selector.cpp:168-206).
#include "qt_common.cuh"
#include "qt_kernels.h"

namespace qt {

constexpr int SEL_THREADS = 1024;

QT_DEV unsigned long long dkey(double v) {
    if (v == 0.0) v = 0.0;  // canonical +0: the reference compares with != and >
    unsigned long long b = (unsigned long long)__double_as_longlong(v);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// exclusive scan of one int per thread over the block (1024 threads)
QT_DEV int block_excl_scan(int v, int* sh, int* total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    __syncthreads();
    if (lane == 31) sh[wid] = x;
    __syncthreads();
    if (wid == 0) {
        int w = sh[lane];
        int s = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        sh[lane] = s - w;  // exclusive warp offsets
        if (lane == 31) sh[32] = s;
    }
    __syncthreads();
    *total = sh[32];
    return sh[wid] + x - v;
}

// bitonic sort (ascending) of n2 (power of two) doubles in smem
QT_DEV void bitonic_sort(double* a, int n2) {
    for (int k = 2; k <= n2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < n2; i += blockDim.x) {
                int ixj = i ^ j;
                if (ixj > i) {
                    double x = a[i], y = a[ixj];
                    bool up = (i & k) == 0;
                    if ((x > y) == up) {
                        a[i] = y;
                        a[ixj] = x;
                    }
                }
            }
            __syncthreads();
        }
    }
}

// percentile (numeric.cpp:84-96) of a sorted array of n values
QT_DEV double pct_sorted(const double* s, int n, double p) {
    if (n == 1) return s[0];
    double h = __dmul_rn(p / 100.0, (double)(n - 1));
    int lo = (int)floor(h);
    int hi = min(lo + 1, n - 1);
    double f = __dsub_rn(h, (double)lo);
    return __dadd_rn(s[lo], __dmul_rn(f, __dsub_rn(s[hi], s[lo])));
}

// One CTA per sequence.  Dynamic smem: 5 * n2 doubles (n2 = pow2 >= V).
__global__ void __launch_bounds__(SEL_THREADS) k_select_topk(
    const double* __restrict__ mag, const double* __restrict__ res, const float* __restrict__ inter_p,
    const float* __restrict__ intra_p, int H, int vstride, const int* __restrict__ vis, const int* __restrict__ txt,
    const int* __restrict__ budget, const int* __restrict__ old_off, const int* __restrict__ new_off,
    double w_mag, double w_inter, double w_intra, double w_quant, int* __restrict__ keep_src,
    int* __restrict__ keep_local, int kl_stride, const int* __restrict__ pos, int* __restrict__ kept_pos,
    double* __restrict__ fused_out, double* __restrict__ norm_out, const double* __restrict__ met_in, int raw) {
    extern __shared__ __align__(16) double sm[];
    __shared__ int hist[256];
    __shared__ int scan_sh[33];
    __shared__ unsigned long long s_prefix;
    __shared__ int s_krem, s_digit;
    const int b = blockIdx.x;
    // met_in (kernel-level ABI): metrics [B][4][vstride] given directly; raw: met_in[0] IS the
    // fused score (select_top_k alone).  txt / offsets / keep_src / pos may then be null.
    const int V = vis[b], T = txt ? txt[b] : 0, K = budget[b];
    const int ob = old_off ? old_off[b] : 0, nb = new_off ? new_off[b] : 0;
    int n2 = 1;
    while (n2 < V) n2 <<= 1;
    double* met = sm;            // [4][n2]
    double* srt = sm + 4 * n2;   // [n2]
    const double invH = 1.0 / (double)H;
    for (int i = threadIdx.x; i < V && met_in; i += blockDim.x) {
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) met[mi * n2 + i] = met_in[((size_t)b * 4 + mi) * vstride + i];
    }
    for (int i = threadIdx.x; i < V && !met_in; i += blockDim.x) {
        double si = 0.0, sa = 0.0;
        for (int h = 0; h < H; ++h) {
            si += (double)inter_p[((size_t)b * H + h) * vstride + i];
            sa += (double)intra_p[((size_t)b * H + h) * vstride + i];
        }
        met[0 * n2 + i] = mag[(size_t)b * vstride + i];
        met[1 * n2 + i] = __dmul_rn(si, invH);
        met[2 * n2 + i] = __dmul_rn(sa, invH);
        met[3 * n2 + i] = res[(size_t)b * vstride + i];
    }
    __syncthreads();
    // robust_normalize each metric in place (selector.cpp:70-84)
    for (int mi = 0; mi < 4 && !raw; ++mi) {
        double* m = met + mi * n2;
        for (int i = threadIdx.x; i < n2; i += blockDim.x) srt[i] = i < V ? m[i] : __longlong_as_double(0x7ff0000000000000ll);
        __syncthreads();
        bitonic_sort(srt, n2);
        const double p5 = pct_sorted(srt, V, 5.0), p95 = pct_sorted(srt, V, 95.0);
        const double spread = __dsub_rn(p95, p5);
        const double inv = 1.0 / spread;
        for (int i = threadIdx.x; i < V; i += blockDim.x) {
            double v = spread < 1e-12 ? 0.5 : fmin(fmax(__dmul_rn(__dsub_rn(m[i], p5), inv), 0.0), 1.0);
            m[i] = v;
            if (norm_out) norm_out[((size_t)b * 4 + mi) * vstride + i] = v;
        }
        __syncthreads();
    }
    // fuse (selector.cpp:86-104), evaluated left to right without contraction
    double* fused = srt;
    for (int i = threadIdx.x; i < V; i += blockDim.x) {
        double f = raw ? met[i] : __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(w_mag, met[i]), __dmul_rn(w_inter, met[n2 + i])),
                                       __dmul_rn(w_intra, met[2 * n2 + i])),
                             __dmul_rn(w_quant, met[3 * n2 + i]));
        fused[i] = f;
        if (fused_out) fused_out[(size_t)b * vstride + i] = f;
    }
    __syncthreads();
    const int kk = min(K, V);
    // radix select of the kk-th largest key
    if (threadIdx.x == 0) {
        s_prefix = 0ull;
        s_krem = kk;
    }
    __syncthreads();
    for (int pass = 0; pass < 8; ++pass) {
        const int shift = 56 - 8 * pass;
        for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
        __syncthreads();
        const unsigned long long pre = s_prefix;
        const unsigned long long hmask = pass == 0 ? 0ull : (~0ull << (shift + 8));
        for (int i = threadIdx.x; i < V; i += blockDim.x) {
            unsigned long long k = dkey(fused[i]);
            if ((k & hmask) == pre) atomicAdd(&hist[(k >> shift) & 0xFF], 1);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int rem = s_krem, d = 255;
            for (; d > 0; --d) {
                if (hist[d] >= rem) break;
                rem -= hist[d];
            }
            s_digit = d;
            s_krem = rem;
            s_prefix = pre | ((unsigned long long)d << shift);
        }
        __syncthreads();
    }
    const unsigned long long kth = s_prefix;
    const int need_eq = s_krem;  // how many keys == kth to take, smallest index first
    // per-thread contiguous ranges keep index order for the scans
    const int per = (V + blockDim.x - 1) / blockDim.x;
    const int i0 = threadIdx.x * per, i1 = min(V, i0 + per);
    int eq_cnt = 0;
    for (int i = i0; i < i1; ++i) eq_cnt += dkey(fused[i]) == kth;
    int tot;
    int eq_before = block_excl_scan(eq_cnt, scan_sh, &tot);
    int sel_cnt = 0;
    {
        int e = eq_before;
        for (int i = i0; i < i1; ++i) {
            unsigned long long k = dkey(fused[i]);
            bool s = k > kth || (k == kth && e < need_eq);
            if (k == kth) ++e;
            sel_cnt += s;
        }
    }
    int sel_before = block_excl_scan(sel_cnt, scan_sh, &tot);
    {
        int e = eq_before, j = sel_before;
        for (int i = i0; i < i1; ++i) {
            unsigned long long k = dkey(fused[i]);
            bool s = k > kth || (k == kth && e < need_eq);
            if (k == kth) ++e;
            if (s) {
                if (keep_src) keep_src[nb + j] = ob + i;
                keep_local[(size_t)b * kl_stride + j] = i;
                if (kept_pos) kept_pos[(size_t)b * vstride + j] = pos[ob + i];
                ++j;
            }
        }
    }
    for (int t = threadIdx.x; t < T; t += blockDim.x) {
        if (keep_src) keep_src[nb + kk + t] = ob + V + t;
        keep_local[(size_t)b * kl_stride + kk + t] = V + t;
    }
}

// compute_metrics output (selector.cpp:19-68) as [B][4][vstride] fp64: the per-head fp32
// column sums averaged over heads with the arithmetic of k_select_topk (the kernel-level
// qt_quota_score ABI).  grid B.
__global__ void k_metrics_pack(const double* __restrict__ mag, const double* __restrict__ res,
                               const float* __restrict__ inter_p, const float* __restrict__ intra_p, int H,
                               int vstride, const int* __restrict__ vis, double* __restrict__ met) {
    const int b = blockIdx.x, V = vis[b];
    const double invH = 1.0 / (double)H;
    for (int i = threadIdx.x; i < V; i += blockDim.x) {
        double si = 0.0, sa = 0.0;
        for (int h = 0; h < H; ++h) {
            si += (double)inter_p[((size_t)b * H + h) * vstride + i];
            sa += (double)intra_p[((size_t)b * H + h) * vstride + i];
        }
        met[((size_t)b * 4 + 0) * vstride + i] = mag[(size_t)b * vstride + i];
        met[((size_t)b * 4 + 1) * vstride + i] = __dmul_rn(si, invH);
        met[((size_t)b * 4 + 2) * vstride + i] = __dmul_rn(sa, invH);
        met[((size_t)b * 4 + 3) * vstride + i] = res[(size_t)b * vstride + i];
    }
}

// Greedy decoding input (an extension: the reference's decode_step takes the next token's
// embedding, model.hpp:177-180): per sequence, token = argmax of its previous logits over the
// first `vocab` entries (ties to the smaller id, as std::max_element / numpy argmax), then that
// row of the token-embedding table, widened to the fp64 residual, is the step's input.  grid B.
__global__ void __launch_bounds__(256) k_greedy_next(const float* __restrict__ logits, int ld, int vocab,
                                                     const float* __restrict__ table, int d, double* __restrict__ x,
                                                     int* __restrict__ tokens) {
    __shared__ float sv[8];
    __shared__ int si[8];
    __shared__ int s_tok;
    pdl_launch_dependents();
    pdl_wait();  // the logits come from the previous step's head GEMV
    logits = pdl_fresh(logits);
    const int b = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const float* lg = logits + (size_t)b * ld;
    float bv = -INFINITY;
    int bi = 0x7fffffff;
    if ((vocab & 3) == 0 && (ld & 3) == 0) {
        // 4 consecutive logits per load, 4 loads in flight per thread before the compares (the
        // scalar loop waited one L2 round trip per element); ascending indices per thread, so
        // the strict > keeps the first maximum
#pragma unroll 4
        for (int i = threadIdx.x * 4; i < vocab; i += blockDim.x * 4) {
            const float4 v = *reinterpret_cast<const float4*>(lg + i);
            if (v.x > bv) { bv = v.x; bi = i; }
            if (v.y > bv) { bv = v.y; bi = i + 1; }
            if (v.z > bv) { bv = v.z; bi = i + 2; }
            if (v.w > bv) { bv = v.w; bi = i + 3; }
        }
    } else {
        for (int i = threadIdx.x; i < vocab; i += blockDim.x) {
            const float v = lg[i];
            if (v > bv) {  // strided ascending scan: the first maximum of this thread's indices
                bv = v;
                bi = i;
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) {
            bv = ov;
            bi = oi;
        }
    }
    if (lane == 0) {
        sv[warp] = bv;
        si[warp] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        float v = sv[0];
        int id = si[0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
            if (sv[w] > v || (sv[w] == v && si[w] < id)) {
                v = sv[w];
                id = si[w];
            }
        s_tok = id < vocab ? id : 0;
        tokens[b] = s_tok;
    }
    __syncthreads();
    const float* row = table + (size_t)s_tok * d;
    for (int j = threadIdx.x; j < d; j += blockDim.x) x[(size_t)b * d + j] = (double)row[j];
}

// dst[b] = src[rows[b]] (fp32 rows of width d): the last prefill logits row of each sequence
__global__ void k_copy_rows_f32(const float* __restrict__ src, const int* __restrict__ rows, int d,
                                float* __restrict__ dst) {
    const int b = blockIdx.x;
    for (int j = threadIdx.x; j < d; j += blockDim.x) dst[(size_t)b * d + j] = src[(size_t)rows[b] * d + j];
}

// x_new[j] = x_old[src[j]], pos_new[j] = pos_old[src[j]]
__global__ void k_gather_rows(const double* __restrict__ x, double* __restrict__ xn, int D,
                              const int* __restrict__ pos, int* __restrict__ posn, const int* __restrict__ src, int M) {
    const int j = blockIdx.x;
    if (j >= M) return;
    const int s = src[j];
    const double2* a = reinterpret_cast<const double2*>(x + (size_t)s * D);
    double2* o = reinterpret_cast<double2*>(xn + (size_t)j * D);
    for (int i = threadIdx.x; i < D / 2; i += blockDim.x) o[i] = a[i];
    if (threadIdx.x == 0) posn[j] = pos[s];
}

// In-place filter of one layer's paged KV rows for (seq b, kv head, K|V):
// row j <- row keep_local[j] (ascending, keep_local[j] >= j), chunks of 64
// destination rows read fully before any write.  grid (Hkv, 2, B).
template <int DH>
__global__ void __launch_bounds__(256) k_kv_compact(uint8_t* __restrict__ pool, long long page_bytes,
                                                    const int* __restrict__ pt, int max_pages, int Hkv,
                                                    const int* __restrict__ keep_local, int kl_stride,
                                                    const int* __restrict__ new_len) {
    constexpr int RB = DH / 2;       // bytes per row
    constexpr int CPR = RB / 16;     // 16-byte chunks per row
    constexpr int ROWS = 256 / CPR;  // rows per chunk step
    const int kh = blockIdx.x, which = blockIdx.y, b = blockIdx.z;
    const int n = new_len[b];
    const size_t cb = (size_t)Hkv * kPage * RB;
    const int* kl = keep_local + (size_t)b * kl_stride;
    for (int j0 = 0; j0 < n; j0 += ROWS) {
        const int j = j0 + threadIdx.x / CPR, q = threadIdx.x % CPR;
        uint4 v = make_uint4(0, 0, 0, 0);
        float sc = 0.f;
        if (j < n) {
            const int s = kl[j];
            const uint8_t* page = pool + (long long)pt[b * max_pages + s / kPage] * page_bytes;
            v = *reinterpret_cast<const uint4*>(page + which * cb + ((size_t)kh * kPage + s % kPage) * RB + q * 16);
            sc = reinterpret_cast<const float*>(page + 2 * cb)[which * Hkv * kPage + kh * kPage + s % kPage];
        }
        __syncthreads();
        if (j < n) {
            uint8_t* page = pool + (long long)pt[b * max_pages + j / kPage] * page_bytes;
            *reinterpret_cast<uint4*>(page + which * cb + ((size_t)kh * kPage + j % kPage) * RB + q * 16) = v;
            if (q == 0) reinterpret_cast<float*>(page + 2 * cb)[which * Hkv * kPage + kh * kPage + j % kPage] = sc;
        }
        __syncthreads();
    }
}

}  // namespace qt

using namespace qt;

extern "C" {

int qt_launch_select_topk(const double* mag, const double* res, const float* inter, const float* intra, int H,
                          int vstride, const int* vis, const int* txt, const int* budget, const int* old_off,
                          const int* new_off, int B, int vmax, const double* w4, int* keep_src, int* keep_local,
                          int kl_stride, const int* pos, int* kept_pos, double* fused_out, double* norm_out,
                          const double* met_in, int raw, cudaStream_t st) {
    if (B <= 0) return 0;
    int n2 = 1;
    while (n2 < vmax) n2 <<= 1;
    const size_t smem = (size_t)5 * n2 * sizeof(double);
    if (smem > 220 * 1024) return -1;
    cudaFuncSetAttribute(k_select_topk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const double w0 = w4 ? w4[0] : 0.0, w1 = w4 ? w4[1] : 0.0, w2 = w4 ? w4[2] : 0.0, w3 = w4 ? w4[3] : 0.0;
    k_select_topk<<<B, SEL_THREADS, smem, st>>>(mag, res, inter, intra, H, vstride, vis, txt, budget, old_off,
                                                new_off, w0, w1, w2, w3, keep_src, keep_local,
                                                kl_stride, pos, kept_pos, fused_out, norm_out, met_in, raw);
    return (int)cudaGetLastError();
}

int qt_launch_metrics_pack(const double* mag, const double* res, const float* inter, const float* intra, int H,
                           int vstride, const int* vis, int B, double* metrics, cudaStream_t st) {
    if (B <= 0) return 0;
    k_metrics_pack<<<B, 256, 0, st>>>(mag, res, inter, intra, H, vstride, vis, metrics);
    return (int)cudaGetLastError();
}

int qt_launch_greedy_next(const float* logits, int ld, int vocab, const float* table, int d, double* x, int* tokens,
                          int B, cudaStream_t st) {
    if (B <= 0) return 0;
    return launch_pdl(k_greedy_next, dim3(B), dim3(256), 0, st, logits, ld, vocab, table, d, x, tokens);
}

int qt_launch_copy_rows_f32(const float* src, const int* rows, int d, float* dst, int B, cudaStream_t st) {
    if (B <= 0) return 0;
    k_copy_rows_f32<<<B, 256, 0, st>>>(src, rows, d, dst);
    return (int)cudaGetLastError();
}

int qt_launch_gather_rows(const double* x, double* xn, int D, const int* pos, int* posn, const int* src, int M,
                          cudaStream_t st) {
    if (M <= 0) return 0;
    k_gather_rows<<<M, 256, 0, st>>>(x, xn, D, pos, posn, src, M);
    return (int)cudaGetLastError();
}

int qt_launch_kv_compact(uint8_t* pool, long long page_bytes, const int* pt, int max_pages, int Hkv, int dh,
                         const int* keep_local, int kl_stride, const int* new_len, int B, cudaStream_t st) {
    if (B <= 0) return 0;
    const dim3 grid(Hkv, 2, B);
    if (dh == 128) k_kv_compact<128><<<grid, 256, 0, st>>>(pool, page_bytes, pt, max_pages, Hkv, keep_local, kl_stride, new_len);
    else if (dh == 64) k_kv_compact<64><<<grid, 256, 0, st>>>(pool, page_bytes, pt, max_pages, Hkv, keep_local, kl_stride, new_len);
    else return -1;
    return (int)cudaGetLastError();
}

}  // extern "C"
