// qt_common.cuh -- shared device helpers for the QUOTA B200 kernels (sm_100a).
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#define QT_DEV __device__ __forceinline__
#define QT_HD __host__ __device__ __forceinline__

namespace qt {

// ---------------------------------------------------------------- constants
constexpr double kNormEps = 1e-6;   // model.cpp:15
constexpr int kWarp = 32;
constexpr int kPage = 64;           // KV page: 64 token rows per (layer, sequence)

// ---------------------------------------------------------------- reductions
template <typename T>
QT_DEV T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
template <typename T>
QT_DEV T warp_max(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Block-wide sum/max through shared scratch (>= 32 entries); result broadcast.
template <typename T>
QT_DEV T block_sum(T v, T* scratch) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) scratch[wid] = v;
    __syncthreads();
    T r = lane < nw ? scratch[lane] : T(0);
    r = warp_sum(r);
    return r;
}
// One-barrier block reductions: `scratch` must not be in use by another reduction of the
// same block (give each reduction of a kernel its own scratch array).
template <typename T>
QT_DEV T block_sum1(T v, T* scratch) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    v = warp_sum(v);
    if (lane == 0) scratch[wid] = v;
    __syncthreads();
    return warp_sum(lane < nw ? scratch[lane] : T(0));
}
template <typename T>
QT_DEV T block_max1(T v, T* scratch) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    v = warp_max(v);
    if (lane == 0) scratch[wid] = v;
    __syncthreads();
    return warp_max(lane < nw ? scratch[lane] : T(0));
}
template <typename T>
QT_DEV T block_max(T v, T* scratch) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    v = warp_max(v);
    __syncthreads();
    if (lane == 0) scratch[wid] = v;
    __syncthreads();
    T r = lane < nw ? scratch[lane] : T(0);
    r = warp_max(r);
    return r;
}

// ---------------------------------------------------------------- quantizer
// Reference quantizer (quant.cpp:39-45, 64-66, 85-87): symmetric, codes
// clamp(rne(x/s), -qmax, qmax), scale max|x|/qmax (1 for an all-zero group).
// Evaluated in fp64 so a code equals the reference code for the same input.
QT_DEV double q_scale(double max_abs, int qmax) { return max_abs == 0.0 ? 1.0 : max_abs / (double)qmax; }

QT_DEV int q_code(double x, double s, int qmax) {
    double q = rint(x / s);  // cvt.rni: round half to even == round_half_even
    q = fmin(fmax(q, -(double)qmax), (double)qmax);
    return (int)q;
}

// Same code as q_code(x, s) (the reference's fp64 rint(x / s)), computed in
// fp32 whenever that is provably the same decision: the fp32 quotient is
// within ~3 ulp (< 1e-5 absolute for |q| < 16) of the exact one, so unless it
// lies within 1e-4 of a .5 tie, rint() of both agrees; |q| >= 8 clamps either
// way.  Near-ties take the fp64 path: x * (1/s), and the correctly rounded
// x / s when even that sits within 1e-9 of the tie.
// The fp32 rounding is the 1.5 * 2^23 magic add (round half to even, exact for |q| < 2^22 --
// the quotient is first clamped to [-(qmax + 1), qmax + 1]); the integer is read from the
// sum's mantissa and the distance to the rounded value (exact) is the tie test: no F2I or
// FRND in the fast path.
QT_DEV int q_code_r(double x, double s, double inv_s, int qmax) {
    const float qf = (float)x * (float)inv_s;
    const float lim = (float)qmax + 1.0f;
    const float qc = fminf(fmaxf(qf, -lim), lim);
    const float t = qc + 12582912.0f;
    if (fabsf(qc - (t - 12582912.0f)) < 0.4999f) {
        const int c = __float_as_int(t) - 0x4B400000;
        return c > qmax ? qmax : (c < -qmax ? -qmax : c);
    }
    double q = x * inv_s;
    const double f = q - floor(q);
    if (fabs(f - 0.5) < 1e-9) q = x / s;
    q = rint(q);
    q = fmin(fmax(q, -(double)qmax), (double)qmax);
    return (int)q;
}

// int4 two's-complement nibble packing: low nibble = even k.
QT_DEV uint32_t pack8(const int* c) {
    uint32_t w = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) w |= (uint32_t)(c[i] & 0xF) << (4 * i);
    return w;
}

// 8 codes -> 8 int8 bytes holding 16 x code (the int8-operand GEMM's activation layout)
QT_DEV uint2 pack8_i8x16(const int* c) {
    uint32_t lo = 0, hi = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        lo |= (uint32_t)((c[i] << 4) & 0xFF) << (8 * i);
        hi |= (uint32_t)((c[i + 4] << 4) & 0xFF) << (8 * i);
    }
    return make_uint2(lo, hi);
}

// Unpack 8 int4 nibbles into two int8x4 registers holding 16*code: the
// nibble lands in the high half of each byte so the byte's sign bit is the
// nibble's.  lo = even k (nibbles 0,2,4,6), hi = odd k (1,3,5,7).  Products of
// two such operands carry a factor 256, removed exactly after accumulation.
QT_DEV void unpack_x16(uint32_t w, uint32_t& lo, uint32_t& hi) {
    lo = (w << 4) & 0xF0F0F0F0u;
    hi = w & 0xF0F0F0F0u;
}

QT_DEV int nib(uint32_t w, int i) { return ((int)(w << (28 - 4 * i))) >> 28; }

// ---------------------------------------------------------------- W4 tiled layout
// Packed int4 code matrices (weights [N_pad x K_pad] and activations
// [rows_pad x K_pad]) are stored as 1 KB tiles of 16 rows x 128 k (16 rows x 64
// bytes, row-major inside the tile), k-block-major: tile (rt, kt) sits at
// (kt * rows_pad/16 + rt) * 1024.  All row blocks of one k-block are therefore
// contiguous -- a whole 128/256-row GEMM stage is ONE TMA bulk copy -- and a
// lane (g, tig) of an mma.sync fragment reads 16 contiguous bytes at
// tile + g*64 + tig*16 (+512 for rows 8-15).
QT_HD size_t w4t_offset(int row, int kbyte, int rows_pad) {
    return ((size_t)(kbyte >> 6) * (rows_pad >> 4) + (row >> 4)) * 1024 + (size_t)(row & 15) * 64 + (kbyte & 63);
}

// ---------------------------------------------------------------- mbarrier / TMA bulk
QT_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
QT_DEV void mbar_init(uint64_t* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
QT_DEV void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
QT_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
QT_DEV void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// arrive on the mbarrier at this offset in CTA `rank` of the cluster (release, cluster scope)
QT_DEV void mbar_arrive_cluster(uint64_t* bar, uint32_t rank) {
    asm volatile(
        "{\n"
        ".reg .b32 ra;\n"
        "mapa.shared::cluster.u32 ra, %0, %1;\n"
        "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(rank)
        : "memory");
}
QT_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// 1D TMA bulk copy global -> shared, completion counted on an mbarrier
QT_DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// ---------------------------------------------------------------- mma.sync
// D(16x8 s32) += A(16x32 s8, row) * B(32x8 s8, col)
QT_DEV void mma_s8_16832(int* d, const uint32_t* a, const uint32_t* b) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 "
        "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

// D(16x8 f32) += A(16x16 f16, row) * B(16x8 f16, col)
QT_DEV void mma_f16_16816(float* d, const uint32_t* a, const uint32_t* b) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 "
        "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

QT_DEV uint32_t h2_as_u32(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }

// split an fp32 pair into hi/lo fp16 pairs: x ~= hi + lo to ~2^-22 relative
QT_DEV void split_h2(float x0, float x1, uint32_t& hi, uint32_t& lo) {
    __half2 h = __floats2half2_rn(x0, x1);
    float2 hf = __half22float2(h);
    __half2 l = __floats2half2_rn(x0 - hf.x, x1 - hf.y);
    hi = h2_as_u32(h);
    lo = h2_as_u32(l);
}

// 8 nibbles of one word (channel e at bits 4e) -> 4 exact half2 of consecutive channel pairs
// (2j, 2j + 1): byte j of w and of w >> 4 go to the two halves (PRMT), their low nibbles
// offset by 8 into the mantissas of fp16 1024 (LOP3 0x6A: b ? a ^ c : c), and the magic
// 1032 is subtracted (HSUB2) -- 3 instructions per pair, no I2F
QT_DEV void word_to_h2_pairs(uint32_t w, uint32_t* h) {  // h: 16-byte aligned (one uint4 store)
    const uint32_t w4 = w >> 4;
    uint32_t o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const uint32_t z = __byte_perm(w, w4, (uint32_t)(j | ((4 + j) << 8)));
        uint32_t m;
        asm("lop3.b32 %0, %1, %2, %3, 0x6A;\n" : "=r"(m) : "r"(z), "r"(0x000F000Fu), "r"(0x64086408u));
        const __half2 r = __hsub2(*reinterpret_cast<const __half2*>(&m), __half2half2(__ushort_as_half(0x6408)));
        o[j] = *reinterpret_cast<const uint32_t*>(&r);
    }
    *reinterpret_cast<uint4*>(h) = make_uint4(o[0], o[1], o[2], o[3]);
}

// int4 nibble pair (one byte: even k low, odd k high) -> half2(code_even, code_odd)
QT_DEV uint32_t nib2_to_h2(uint32_t byte) {
    int lo = ((int)(byte << 28)) >> 28;
    int hi = ((int)(byte << 24)) >> 28;
    return h2_as_u32(__halves2half2(__int2half_rn(lo), __int2half_rn(hi)));
}

// ---------------------------------------------------------------- cp.async
QT_DEV void cp_async16(void* smem, const void* gmem, bool pred) {
    uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    int n = pred ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
QT_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
QT_DEV void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

QT_DEV uint4 ldg_nc_v4(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// 256-bit global accesses (sm_100: LDG/STG.E.ENL2.256): one full 32-byte sector per thread
// and instruction -- the row-per-thread GEMM epilogues touch 32 rows per warp instruction
QT_DEV double4 ld_v4f64(const double* p) {
    double4 r;
    asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];\n" : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w) : "l"(p));
    return r;
}
QT_DEV void st_v4f64(double* p, double4 v) {
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};\n" ::"l"(p), "d"(v.x), "d"(v.y), "d"(v.z), "d"(v.w)
                 : "memory");
}
QT_DEV void st_v8f32(float* p, const float* v) {
    asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"l"(p), "f"(v[0]), "f"(v[1]), "f"(v[2]),
                 "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
                 : "memory");
}

QT_DEV float silu_f(float x) { return x / (1.0f + expf(-x)); }

// ---------------------------------------------------------------- PDL
// Programmatic dependent launch: a kernel launched with
// cudaLaunchAttributeProgrammaticStreamSerialization may start while its
// predecessor drains; pdl_wait() blocks until the predecessor grid completed
// and its writes are visible.  Every kernel calls pdl_wait() before touching
// data produced upstream (and before exiting), so completion stays transitive.
QT_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
// A pointer to upstream-produced data, opaque to the compiler from this point on.  Loads
// through `const T* __restrict__` are invariant to the compiler, which may hoist them above
// the (memory-clobbering) griddepcontrol.wait -- measured in k_attn_dec_w: the q loads moved
// before the wait and read the upstream GEMV's output before it was written.  Passing the
// pointer through an empty volatile asm after pdl_wait() pins those loads below the wait.
template <typename T>
QT_DEV T* pdl_fresh(T* p) {
    asm volatile("" : "+l"(p));
    return p;
}
QT_DEV void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

}  // namespace qt

#ifndef __CUDACC_RTC__
#include <cstdlib>
namespace qt {
// Set by the host engine after it enqueues a copy / memset on the stream: the
// next launch then takes a full stream dependency instead of a programmatic
// (PDL) one, so it cannot start before the copy has landed.
inline thread_local bool g_pdl_block = false;
// Weights of the NEXT weight-streaming GEMV on the stream: the decode GEMV launched next
// pulls them toward L2 (cp.async.bulk.prefetch) while it streams its own, so HBM keeps
// streaming through the latency-bound attention / quantizer kernels in between.  Set by
// the engine right before the launch; consumed (cleared) by the GEMV launcher.
inline thread_local const void* g_l2_next = nullptr;
inline thread_local long long g_l2_next_bytes = 0;

template <typename... KArgs, typename... Args>
inline int launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                      Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = g_pdl_block ? 0 : 1;
    g_pdl_block = false;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
    return (int)e;
}
}  // namespace qt
#endif

namespace qt {

}  // namespace qt
