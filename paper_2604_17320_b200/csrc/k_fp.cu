// k_fp.cu -- the full-precision forward used for calibration:
// fit_act_scales (calibrator.cpp:237-249) runs forward_prefill in ExecMode::Fp
// with an ActStats collector (model.cpp:174-210, observed at model.cpp:348,
// 393, 430, 434, 443).  Here the same forward runs on the B200 in fp64 -- the
// reference's arithmetic type -- with cuBLAS DGEMM for the projections (a plain
// library GEMM, not the hot path) and these kernels for everything else; the
// per-site max |x| is reduced with order-independent atomics, so the fitted
// static scales match the reference's up to DGEMM summation order.
#include "qt_common.cuh"
#include "qt_kernels.h"

namespace qt {

// max |v| over non-negative doubles: the IEEE bit pattern is order-preserving
QT_DEV void atomic_max_abs(unsigned long long* slot, double v) {
    atomicMax(slot, (unsigned long long)__double_as_longlong(fabs(v)));
}

// RMSNorm (model.cpp:147-154) of fp64 rows, optionally observed
__global__ void __launch_bounds__(256) k_fp_rmsnorm(const double* __restrict__ x, const float* __restrict__ gain,
                                                    int D, double* __restrict__ out,
                                                    unsigned long long* __restrict__ obs) {
    __shared__ double red[32];
    const int row = blockIdx.x;
    const double* xr = x + (size_t)row * D;
    double ss = 0.0;
    for (int i = threadIdx.x; i < D; i += blockDim.x) ss += xr[i] * xr[i];
    ss = block_sum(ss, red);
    const double inv = 1.0 / sqrt(ss / (double)D + kNormEps);
    double mx = 0.0;
    for (int i = threadIdx.x; i < D; i += blockDim.x) {
        const double y = __dmul_rn(__dmul_rn(xr[i], inv), (double)gain[i]);
        out[(size_t)row * D + i] = y;
        mx = fmax(mx, fabs(y));
    }
    if (obs) {
        mx = block_max(mx, red);
        if (threadIdx.x == 0) atomic_max_abs(obs, mx);
    }
}

// interleaved-pair RoPE of the q and k heads (model.cpp:156-168) at original positions
__global__ void k_fp_rope(double* __restrict__ qkv, int ldq, int nheads_qk, int dh, const int* __restrict__ pos,
                          const double2* __restrict__ rope) {
    const int row = blockIdx.x;
    const double2* rt = rope + (size_t)pos[row] * (dh / 2);
    double* r = qkv + (size_t)row * ldq;
    for (int i = threadIdx.x; i < nheads_qk * dh / 2; i += blockDim.x) {
        const int hd = i / (dh / 2), p = i % (dh / 2);
        double* v = r + hd * dh + 2 * p;
        const double2 cs = rt[p];
        const double a = v[0], b = v[1];
        v[0] = __dsub_rn(__dmul_rn(a, cs.x), __dmul_rn(b, cs.y));
        v[1] = __dadd_rn(__dmul_rn(a, cs.y), __dmul_rn(b, cs.x));
    }
}

// masked softmax attention (model.cpp:35-44, 272-292, 385) for one (query row,
// head) per CTA, fp64: visual queries see visual keys; text queries see every
// visual key and causal text.  dh threads.  probs (optional, recipe hook): the
// normalised probabilities on the visual keys, [H][S][V] -- the blocks the
// reference slices into attn_inter / attn_intra (model.cpp:386-389).
__global__ void k_fp_attention(const double* __restrict__ qkv, int ldq, int H, int Hkv, int dh, int S, int V,
                               double* __restrict__ out, int ldo, unsigned long long* __restrict__ obs,
                               double* __restrict__ probs) {
    extern __shared__ double sm[];
    double* qs = sm;           // [dh]
    double* p = sm + dh;       // [S] probabilities
    __shared__ double red[32];
    const int i = blockIdx.x, h = blockIdx.y;
    const int kh = h / (H / Hkv);
    const double inv_sqrt = 1.0 / sqrt((double)dh);
    for (int c = threadIdx.x; c < dh; c += blockDim.x) qs[c] = qkv[(size_t)i * ldq + h * dh + c];
    __syncthreads();
    const int nkeys = i < V ? V : i + 1;  // allowed keys are the prefix [0, nkeys)
    double mx = -1e300;
    for (int j = threadIdx.x; j < nkeys; j += blockDim.x) {
        const double* kr = qkv + (size_t)j * ldq + (H + kh) * dh;
        double s = 0.0;
        for (int c = 0; c < dh; ++c) s += qs[c] * kr[c];
        s *= inv_sqrt;
        p[j] = s;
        mx = fmax(mx, s);
    }
    mx = block_max(mx, red);
    double sum = 0.0;
    for (int j = threadIdx.x; j < nkeys; j += blockDim.x) {
        const double e = exp(p[j] - mx);
        p[j] = e;
        sum += e;
    }
    sum = block_sum(sum, red);
    __syncthreads();
    double omax = 0.0;
    for (int c = threadIdx.x; c < dh; c += blockDim.x) {
        double o = 0.0;
        for (int j = 0; j < nkeys; ++j) o += (p[j] / sum) * qkv[(size_t)j * ldq + (H + Hkv + kh) * dh + c];
        out[(size_t)i * ldo + h * dh + c] = o;
        omax = fmax(omax, fabs(o));
    }
    if (probs)
        for (int j = threadIdx.x; j < V; j += blockDim.x) probs[((size_t)h * S + i) * V + j] = p[j] / sum;
    if (obs) {
        omax = block_max(omax, red);
        if (threadIdx.x == 0) atomic_max_abs(obs, omax);
    }
}

// compute_metrics' attention cues (selector.cpp:40-53) from the [H][S][V] probabilities:
// inter[j] = sum over heads, then text query rows, of p(row, j); intra over visual query
// rows; both * (1/H).  One thread per visual key, summed in the reference's order.
__global__ void k_fp_colsum(const double* __restrict__ probs, int H, int S, int V, double* __restrict__ inter,
                            double* __restrict__ intra) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= V) return;
    double si = 0.0, sa = 0.0;
    for (int h = 0; h < H; ++h)
        for (int r = V; r < S; ++r) si = __dadd_rn(si, probs[((size_t)h * S + r) * V + j]);
    for (int h = 0; h < H; ++h)
        for (int r = 0; r < V; ++r) sa = __dadd_rn(sa, probs[((size_t)h * S + r) * V + j]);
    const double inv = 1.0 / (double)H;
    inter[j] = __dmul_rn(si, inv);
    intra[j] = __dmul_rn(sa, inv);
}

// mid = silu(g) (SiLU MLP, model.cpp:432-434) or silu(g) * u (SwiGLU), observed
__global__ void k_fp_mlp_act(const double* __restrict__ g, const double* __restrict__ u, long long n,
                             double* __restrict__ mid, unsigned long long* __restrict__ obs) {
    __shared__ double red[32];
    double mx = 0.0;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
        const double x = g[e];
        double y = x / (1.0 + exp(-x));
        if (u) y *= u[e];
        mid[e] = y;
        mx = fmax(mx, fabs(y));
    }
    mx = block_max(mx, red);
    if (threadIdx.x == 0) atomic_max_abs(obs, mx);
}

// QUOTA diagnostics (profile_diagnostics, calibrator.cpp:147-195): for text query i
// and head h of the quantized forward, the attention probabilities over the
// allowed keys (every visual key + causal text, model.cpp:35-44) from q and the
// dequantised int4 keys of the cache (model.cpp:371-381); out = the summed top-10
// mass on the visual keys (concentration_for_record, calibrator.cpp:151-167).
// One warp per (text query, head); scores staged in shared memory.
__global__ void k_diag_top10(const float* __restrict__ qkv, int ldq, int H, int Hkv, int dh, int V, int S,
                             const uint8_t* __restrict__ pool, long long page_bytes, const int* __restrict__ pt,
                             double* __restrict__ out) {
    extern __shared__ float sc[];  // [warps][S]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int item = blockIdx.x * nw + warp;  // (text query t, head h)
    const int T = S - V;
    if (item >= T * H) return;
    const int t = item / H, h = item % H, i = V + t;
    const int kh = h / (H / Hkv);
    float* s = sc + (size_t)warp * S;
    const float* q = qkv + (size_t)i * ldq + h * dh;
    const float inv_sqrt = (float)(1.0 / sqrt((double)dh));
    const size_t cb = (size_t)Hkv * kPage * (dh / 2);
    float mx = -1e30f;
    const int nkeys = i + 1;  // visual prefix + causal text up to i
    for (int j = lane; j < nkeys; j += 32) {
        const uint8_t* page = pool + (long long)pt[j / kPage] * page_bytes;
        const uint8_t* kr = page + ((size_t)kh * kPage + j % kPage) * (dh / 2);
        const float ks = reinterpret_cast<const float*>(page + 2 * cb)[kh * kPage + j % kPage];
        float dsum = 0.f;
        for (int c = 0; c < dh / 2; ++c) {
            const int b = kr[c];
            dsum = fmaf(q[2 * c], (float)(((int)(b << 28)) >> 28), dsum);
            dsum = fmaf(q[2 * c + 1], (float)(((int)(b << 24)) >> 28), dsum);
        }
        const float v = dsum * ks * inv_sqrt;
        s[j] = v;
        mx = fmaxf(mx, v);
    }
    mx = warp_max(mx);
    float sum = 0.f;
    for (int j = lane; j < nkeys; j += 32) {
        const float e = expf(s[j] - mx);
        s[j] = e;
        sum += e;
    }
    sum = warp_sum(sum);
    __syncwarp();
    // top-10 of the visual probabilities: 10 rounds of a warp argmax, each removing the winner
    double mass = 0.0;
    const int k = min(10, V);
    for (int r = 0; r < k; ++r) {
        float best = -1.f;
        int bj = -1;
        for (int j = lane; j < V; j += 32)
            if (s[j] > best) {
                best = s[j];
                bj = j;
            }
        for (int o = 16; o > 0; o >>= 1) {
            const float ob = __shfl_xor_sync(0xffffffffu, best, o);
            const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
            if (ob > best || (ob == best && oj < bj)) {
                best = ob;
                bj = oj;
            }
        }
        mass += (double)best / (double)sum;
        __syncwarp();
        if (lane == 0 && bj >= 0) s[bj] = -2.f;
        __syncwarp();
    }
    if (lane == 0) out[(size_t)h * T + t] = mass;
}

}  // namespace qt

using namespace qt;

extern "C" {

int qt_launch_fp_rmsnorm(const double* x, const float* gain, int M, int D, double* out, unsigned long long* obs,
                         cudaStream_t st) {
    if (M <= 0) return 0;
    k_fp_rmsnorm<<<M, 256, 0, st>>>(x, gain, D, out, obs);
    return (int)cudaGetLastError();
}

int qt_launch_fp_rope(double* qkv, int ldq, int M, int nheads_qk, int dh, const int* pos, const double* rope,
                      cudaStream_t st) {
    if (M <= 0) return 0;
    k_fp_rope<<<M, 128, 0, st>>>(qkv, ldq, nheads_qk, dh, pos, reinterpret_cast<const double2*>(rope));
    return (int)cudaGetLastError();
}

int qt_launch_fp_attention(const double* qkv, int ldq, int H, int Hkv, int dh, int S, int V, double* out, int ldo,
                           unsigned long long* obs, double* probs, cudaStream_t st) {
    if (S <= 0) return 0;
    const size_t smem = (size_t)(dh + S) * sizeof(double);
    if (smem > 200 * 1024) return -1;
    cudaFuncSetAttribute(k_fp_attention, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_fp_attention<<<dim3(S, H), dh, smem, st>>>(qkv, ldq, H, Hkv, dh, S, V, out, ldo, obs, probs);
    return (int)cudaGetLastError();
}

int qt_launch_fp_colsum(const double* probs, int H, int S, int V, double* inter, double* intra, cudaStream_t st) {
    if (V <= 0) return 0;
    k_fp_colsum<<<(V + 127) / 128, 128, 0, st>>>(probs, H, S, V, inter, intra);
    return (int)cudaGetLastError();
}

int qt_launch_fp_mlp_act(const double* g, const double* u, long long n, double* mid, unsigned long long* obs,
                         cudaStream_t st) {
    if (n <= 0) return 0;
    k_fp_mlp_act<<<296, 256, 0, st>>>(g, u, n, mid, obs);
    return (int)cudaGetLastError();
}

int qt_launch_diag_top10(const float* qkv, int ldq, int H, int Hkv, int dh, int V, int S, const uint8_t* pool,
                         long long page_bytes, const int* pt, double* out, cudaStream_t st) {
    const int T = S - V;
    if (T <= 0 || V <= 0) return 0;
    const int nw = 4;
    const size_t smem = (size_t)nw * S * sizeof(float);
    if (smem > 200 * 1024) return -1;
    cudaFuncSetAttribute(k_diag_top10, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_diag_top10<<<(T * H + nw - 1) / nw, nw * 32, smem, st>>>(qkv, ldq, H, Hkv, dh, V, S, pool, page_bytes, pt, out);
    return (int)cudaGetLastError();
}

}  // extern "C"
