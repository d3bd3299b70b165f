// k_decode_mk.cu -- the whole decode step (model.cpp:455-562) as ONE persistent
// kernel for small batches (B <= 8 sequences), sm_100a.
//
// Why: at decode the step is HBM-bound on the int4 weights (3.24 GB at the 7B
// shape, >= 0.5 ms at 6.5 TB/s), but as ~300 separate launches every GEMV
// pays its fill/drain and every small op (norm, RoPE+KV append, attention,
// quantizers) a dependent-launch gap.  Here one CTA per SM runs all layers:
//
//   warp 8 (producer): one elected lane streams THIS CTA's share of every
//     weight matrix of the step -- a static sequence (layers x {qkv, o,
//     gate|up, down}, then head) -- into a ring of 8 KB slots with 1 KB TMA
//     bulk copies (cp.async.bulk + mbarrier complete_tx).  It never waits for
//     activations, so weights keep streaming through every phase barrier.
//   warps 0-7 (workers): consume the ring (mma.sync s8 m16n8k32, swap-AB:
//     16 weight rows x 8 tokens, int4 -> int8 x16 in registers, int32 exact)
//     and run the phases between the GEMVs.
//
// GEMV partition: the (row block x k block) tiles of a matrix are split into
// G equal contiguous ranges (row-block-major), one per CTA -- balanced to one
// tile.  A CTA reduces its partial sums in shared memory and writes them to a
// global int32 accumulator (plain stores for row blocks it owns entirely,
// red.add for the <= 2 it shares).  Integer sums are order independent, so the
// result is deterministic and equal to the unfused GEMV's.  The epilogue
// (scales, residual add, SwiGLU, RoPE) runs in the consumer phase.
//
// Phases per layer (owner = CTA t for token t):
//   S0 owners : x += down-proj (prev layer); RMSNorm + quantize   -> codes
//   S1 all    : QKV GEMV                                           -> acc_qkv
//   S2 units  : per (seq, kv head): q/k/v epilogue, RoPE, int4 K/V quantize +
//               append, attention over the cache; the LAST unit of a sequence
//               quantizes its attention row (attn_out site)        -> codes
//   S4 all    : O GEMV                                             -> acc_o
//   S5 owners : x += O; RMSNorm + quantize                          -> codes
//   S6 all    : gate|up GEMV                                       -> acc_gu
//   S7 owners : SiLU / SwiGLU + quantize (mlp_mid)                 -> codes
//   S8 all    : down GEMV                                          -> acc_dn
// then final norm + head GEMV + logits.  GEMV -> consumer transitions are grid
// barriers; owner -> GEMV transitions wait on a completion counter.  Every
// spin is bounded (trap instead of a hang).  Cross-CTA data is read with
// ld.global.cg (L2), never through a possibly stale L1 line.
//
// Arithmetic mirrors the unfused kernels (k_gemv_reg epilogues, k_rope_kv_append,
// k_attn_decode, k_norm_quant), so results stay within the same parity bounds.
#include "qt_common.cuh"
#include "qt_kernels.h"
#include "qt_decode_mk.h"

namespace qt {

constexpr int MK_WORKERS = 256;             // warps 0-7
constexpr int MK_THREADS = MK_WORKERS + 32;  // + producer warp
constexpr int MK_TILE = 1024;                // 16 rows x 128 k int4
constexpr int MK_SLOT_TILES = 8;
constexpr int MK_SLOT = MK_SLOT_TILES * MK_TILE;
constexpr int MK_TOK = 8;

// ------------------------------------------------------------------ sync helpers
QT_DEV unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

QT_DEV void wk_sync() { asm volatile("bar.sync 1, 256;\n" ::: "memory"); }

QT_DEV unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}

QT_DEV void spin_until(const unsigned* p, unsigned target) {
    long long n = 0;
    while (ld_acquire(p) < target) {
        __nanosleep(20);
        if (++n > (1ll << 24)) __trap();  // a lost arrival: fail loudly, never hang the GPU
    }
}

// all workers' writes done -> arrive (release) -> the last arriver publishes the
// epoch on a separate flag line -> everyone polls only the flag (acquire).
QT_DEV void grid_barrier(unsigned* ctr, unsigned target) {
    wk_sync();
    if (threadIdx.x == 0) {
        unsigned old;
        asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;\n" : "=r"(old) : "l"(ctr) : "memory");
        unsigned* flag = ctr + 32;  // 128 B away from the counter
        if (old + 1 == target) {
            asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(flag), "r"(target) : "memory");
        } else {
            spin_until(flag, target);
        }
    }
    wk_sync();
}

QT_DEV void signal(unsigned* ctr) {
    wk_sync();
    if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(ctr) : "memory");
}

QT_DEV void wait_count(const unsigned* ctr, unsigned target) {
    if (threadIdx.x == 0) spin_until(ctr, target);
    wk_sync();
}

template <typename T>
QT_DEV T wk_sum(T v, T* red) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    v = warp_sum(v);
    wk_sync();
    if (lane == 0) red[w] = v;
    wk_sync();
    T r = lane < 8 ? red[lane] : T(0);
    return warp_sum(r);
}
template <typename T>
QT_DEV T wk_max(T v, T* red) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    v = warp_max(v);
    wk_sync();
    if (lane == 0) red[w] = v;
    wk_sync();
    T r = lane < 8 ? red[lane] : T(0);
    return warp_max(r);
}

// ------------------------------------------------------------------ GEMV plan
struct Gemv {
    const uint8_t* w;
    int rt;   // rows_pad / 16 (tile stride of one k block)
    int rb;   // row blocks with real rows
    int kt;   // k blocks
    int t0, t1;  // this CTA's tile range
};

QT_DEV Gemv gemv_of(const MkParams& p, int g) {
    // g = 4 * layer + kind, or 4 * L = head
    Gemv v;
    int N, K;
    if (g < 4 * p.L) {
        const MkLayer& ly = p.layers[g >> 2];
        const int k = g & 3;
        v.w = ly.w[k];
        v.rt = ly.rows_pad[k] >> 4;
        N = p.N[k];
        K = p.Kp[k];
    } else {
        v.w = p.head;
        v.rt = p.head_rows_pad >> 4;
        N = p.d;
        K = p.Kp[0];
    }
    v.rb = (N + 15) >> 4;
    v.kt = K >> 7;
    const long long T = (long long)v.rb * v.kt;
    v.t0 = (int)(T * blockIdx.x / gridDim.x);
    v.t1 = (int)(T * (blockIdx.x + 1) / gridDim.x);
    return v;
}

// ------------------------------------------------------------------ producer
QT_DEV void producer(const MkParams& p, uint8_t* ring, uint64_t* full, uint64_t* empty) {
    int slot = 0;
    uint32_t phase = 0;
    const int ng = 4 * p.L + 1;
    for (int g = 0; g < ng; ++g) {
        const Gemv v = gemv_of(p, g);
        if (v.t1 <= v.t0) continue;
        int rb = v.t0 / v.kt, kt = v.t0 % v.kt;  // walk (rb, kt) incrementally: no divisions per tile
        const size_t kstride = (size_t)v.rt * MK_TILE;
        for (int i = v.t0; i < v.t1; i += MK_SLOT_TILES) {
            const int n = min(MK_SLOT_TILES, v.t1 - i);
            mbar_wait(&empty[slot], phase ^ 1);
            mbar_arrive_expect_tx(&full[slot], (uint32_t)n * MK_TILE);
            uint8_t* dst = ring + (size_t)slot * MK_SLOT;
            const uint8_t* src = v.w + (size_t)kt * kstride + (size_t)rb * MK_TILE;
            for (int j = 0; j < n; ++j) {
                bulk_g2s(dst + j * MK_TILE, src, MK_TILE, &full[slot]);
                src += kstride;
                if (++kt == v.kt) {
                    kt = 0;
                    ++rb;
                    src = v.w + (size_t)rb * MK_TILE;
                }
            }
            if (++slot == p.nslot) {
                slot = 0;
                phase ^= 1;
            }
        }
    }
}

// ------------------------------------------------------------------ GEMV consumer
// Activation codes of the 8 token rows (tiled, rows_pad 16) -> smem rows.
QT_DEV void load_act(const MkParams& p, int K, uint8_t* As) {
    const int kb = K / 2, chunks = kb / 16;
    for (int c = threadIdx.x; c < MK_TOK * chunks; c += MK_WORKERS) {
        const int t = c / chunks, q = c % chunks;
        cp_async16(As + (size_t)t * p.a_ld + q * 16, p.codes + w4t_offset(t, q * 16, 16), t < p.B);
    }
    cp_async_commit();
    cp_async_wait<0>();
    wk_sync();
}

// One GEMV: ring tiles of this CTA -> smem int32 partial sums -> global acc.
QT_DEV void gemv_consume(const MkParams& p, const Gemv& v, int* accg, int acc_ld, const uint8_t* ring,
                         uint64_t* full, uint64_t* empty, int& slot, uint32_t& phase, const uint8_t* As,
                         int* sacc) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, tig = lane & 3;
    const int rb0 = v.t0 / v.kt;
    const int nrows = v.t1 > v.t0 ? (v.t1 - 1) / v.kt - rb0 + 1 : 0;
    for (int i = threadIdx.x; i < nrows * 16 * MK_TOK; i += MK_WORKERS) sacc[i] = 0;
    wk_sync();
    int acc[4] = {0, 0, 0, 0};
    int cur = -1;
    auto flush = [&]() {
        if (cur < 0) return;
        int* r = sacc + (cur - rb0) * 16 * MK_TOK;
        atomicAdd(&r[g * MK_TOK + 2 * tig], acc[0]);
        atomicAdd(&r[g * MK_TOK + 2 * tig + 1], acc[1]);
        atomicAdd(&r[(g + 8) * MK_TOK + 2 * tig], acc[2]);
        atomicAdd(&r[(g + 8) * MK_TOK + 2 * tig + 1], acc[3]);
        acc[0] = acc[1] = acc[2] = acc[3] = 0;
    };
    // this warp's first tile t0 + warp as (rb, kt), then advance by 8 tiles per slot
    int wrb = v.t0 / v.kt, wkt = v.t0 % v.kt + warp;
    while (wkt >= v.kt) {
        wkt -= v.kt;
        ++wrb;
    }
    for (int i = v.t0; i < v.t1; i += MK_SLOT_TILES) {
        mbar_wait(&full[slot], phase);
        if (i + warp < v.t1) {
            const uint8_t* tile = ring + (size_t)slot * MK_SLOT + warp * MK_TILE;
            const uint4 wa = *reinterpret_cast<const uint4*>(tile + g * 64 + tig * 16);
            const uint4 wb = *reinterpret_cast<const uint4*>(tile + 512 + g * 64 + tig * 16);
            const uint4 bv = *reinterpret_cast<const uint4*>(As + (size_t)g * p.a_ld + wkt * 64 + tig * 16);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
            if (wrb != cur) {
                flush();
                cur = wrb;
            }
#pragma unroll
            for (int s2 = 0; s2 < 4; ++s2) {
                uint32_t a[4], b[2];
                unpack_x16((&wa.x)[s2], a[0], a[2]);
                unpack_x16((&wb.x)[s2], a[1], a[3]);
                unpack_x16((&bv.x)[s2], b[0], b[1]);
                mma_s8_16832(acc, a, b);
            }
        } else {
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
        }
        wkt += MK_SLOT_TILES;
        while (wkt >= v.kt) {
            wkt -= v.kt;
            ++wrb;
        }
        if (++slot == p.nslot) {
            slot = 0;
            phase ^= 1;
        }
    }
    flush();
    wk_sync();
    // smem partials -> global: plain stores for fully owned row blocks, red.add for shared ones
    for (int i = threadIdx.x; i < nrows * 16 * MK_TOK; i += MK_WORKERS) {
        const int rl = i / (16 * MK_TOK), rr = (i / MK_TOK) % 16, tok = i % MK_TOK;
        if (tok >= p.B) continue;
        const int rb = rb0 + rl;
        const int n = rb * 16 + rr;
        const bool owned = rb * v.kt >= v.t0 && (rb + 1) * v.kt <= v.t1;
        const int val = sacc[i] >> 8;  // exact: every product carries 16 x 16
        int* dst = accg + (size_t)tok * acc_ld + n;
        if (owned) *dst = val;
        else atomicAdd(dst, val);
    }
}

// ------------------------------------------------------------------ owner phases
// Compact rolled loops over a shared-memory staging row: straight-line fp64
// code executed once per phase would be instruction-fetch bound (the kernel is
// large and the i-cache cold for it), so each phase is a few short loops.

// codes of one token row (tiled row t, rows_pad 16) from staged values v[0..D)
// (zero beyond D up to Kp) with scale s
template <typename TV>
QT_DEV void quant_row_smem(const MkParams& p, int t, double s, const TV* v, int D, int Kp) {
    const double inv_s = 1.0 / s;
#pragma unroll 1
    for (int w = threadIdx.x; w * 8 < Kp; w += MK_WORKERS) {
        int c[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) c[e] = w * 8 + e < D ? q_code_r((double)v[w * 8 + e], s, inv_s, 7) : 0;
        *reinterpret_cast<uint32_t*>(p.codes + w4t_offset(t, w * 4, 16)) = pack8(c);
    }
}

// Every global-memory loop below issues MK_UNR independent loads before using
// any of them (one latency per batch, not per element): under a full-HBM weight
// stream a DRAM miss costs microseconds.
constexpr int MK_UNR = 8;

// x[t] (+)= residual GEMV result; RMSNorm(gain); quantize -> codes row t (K = d)
QT_DEV void owner_norm_quant(const MkParams& p, int t, const int* accr, const double* sw, const float* gain,
                             double site_scale, double* red, double* v, unsigned long long* tr = nullptr) {
    const int D = p.d;
    double* xr = p.x + (size_t)t * D;
    const double a_s = accr ? __ldcg(p.sa + t) : 0.0;
    double ss = 0.0;
#pragma unroll 1
    for (int n0 = threadIdx.x; n0 < D; n0 += MK_UNR * MK_WORKERS) {
        double xv[MK_UNR], sv[MK_UNR];
        int av[MK_UNR];
#pragma unroll
        for (int u = 0; u < MK_UNR; ++u) {
            const int n = n0 + u * MK_WORKERS;
            xv[u] = n < D ? __ldcg(xr + n) : 0.0;
            av[u] = accr && n < D ? __ldcg(accr + n) : 0;
            sv[u] = accr && n < D ? __ldg(sw + n) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < MK_UNR; ++u) {
            const int n = n0 + u * MK_WORKERS;
            if (n < D) {
                double y = xv[u];
                if (accr) {
                    y += (double)av[u] * (a_s * sv[u]);
                    xr[n] = y;
                }
                v[n] = y;
                ss += y * y;
            }
        }
    }
    if (tr && threadIdx.x == 0) tr[16] = gtimer();
    ss = wk_sum(ss, red);
    if (tr && threadIdx.x == 0) tr[17] = gtimer();
    const double inv = 1.0 / sqrt(ss / (double)D + kNormEps);
    double mx = 0.0;
#pragma unroll 1
    for (int n0 = threadIdx.x; n0 < D; n0 += MK_UNR * MK_WORKERS) {
        float gv[MK_UNR];
#pragma unroll
        for (int u = 0; u < MK_UNR; ++u) {
            const int n = n0 + u * MK_WORKERS;
            gv[u] = n < D ? __ldg(gain + n) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < MK_UNR; ++u) {
            const int n = n0 + u * MK_WORKERS;
            if (n < D) {
                const double y = __dmul_rn(__dmul_rn(v[n], inv), (double)gv[u]);
                v[n] = y;
                mx = fmax(mx, fabs(y));
            }
        }
    }
    if (tr && threadIdx.x == 0) tr[18] = gtimer();
    double s = site_scale;
    if (p.act_mode == 1) s = q_scale(wk_max(mx, red), 7);
    wk_sync();
    if (tr && threadIdx.x == 0) tr[19] = gtimer();
    quant_row_smem(p, t, s, v, D, p.Kp[0]);
    if (threadIdx.x == 0) p.sa[t] = s;
    if (tr && threadIdx.x == 0) tr[20] = gtimer();
}

// attn_out site for token b once all its heads are written (the last unit does it)
QT_DEV void attn_row_quant(const MkParams& p, int l, int b, double* red, float* v) {
    const int D = p.d;
    double mx = 0.0;
#pragma unroll 1
    for (int n0 = threadIdx.x; n0 < D; n0 += MK_UNR * MK_WORKERS) {
        float y[MK_UNR];
#pragma unroll
        for (int u = 0; u < MK_UNR; ++u) {
            const int n = n0 + u * MK_WORKERS;
            y[u] = n < D ? __ldcg(p.attn + (size_t)b * D + n) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < MK_UNR; ++u) {
            const int n = n0 + u * MK_WORKERS;
            if (n < D) {
                v[n] = y[u];
                mx = fmax(mx, fabs((double)y[u]));
            }
        }
    }
    double s = p.act[4 * l + 1];
    if (p.act_mode == 1) s = q_scale(wk_max(mx, red), 7);
    wk_sync();
    quant_row_smem(p, b, s, v, D, p.Kp[1]);
    if (threadIdx.x == 0) p.sa[b] = s;
}

// mlp_mid site: SiLU / SwiGLU from acc_gu (values rounded to fp32 like the
// unfused epilogue), then quantize (K = d_ff)
QT_DEV void owner_mid_quant(const MkParams& p, int l, int t, double* red, float* v) {
    const MkLayer& ly = p.layers[l];
    const int F = p.dff;
    const int* ar = p.acc[2] + (size_t)t * p.acc_ld[2];
    const double* sw = ly.s[2];
    const double a_s = __ldcg(p.sa + t);
    const int glu = p.mlp == 1 ? 2 : 1;
    double mx = 0.0;
#pragma unroll 1
    for (int n0 = threadIdx.x; n0 < F; n0 += MK_UNR * MK_WORKERS) {
        int ag[MK_UNR], au[MK_UNR];
        double sg[MK_UNR], su[MK_UNR];
#pragma unroll
        for (int u = 0; u < MK_UNR; ++u) {
            const int n = n0 + u * MK_WORKERS;
            const bool ok = n < F;
            ag[u] = ok ? __ldcg(ar + glu * n) : 0;
            sg[u] = ok ? __ldg(sw + glu * n) : 0.0;
            au[u] = ok && glu == 2 ? __ldcg(ar + 2 * n + 1) : 0;
            su[u] = ok && glu == 2 ? __ldg(sw + 2 * n + 1) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < MK_UNR; ++u) {
            const int n = n0 + u * MK_WORKERS;
            if (n < F) {
                // the mid activation is an fp32 tensor: SiLU / SwiGLU in fp32
                const float g = (float)((double)ag[u] * (a_s * sg[u]));
                float y = g / (1.0f + expf(-g));
                if (glu == 2) y *= (float)((double)au[u] * (a_s * su[u]));
                v[n] = y;
                mx = fmax(mx, fabs((double)y));
            }
        }
    }
    double s = p.act[4 * l + 3];
    if (p.act_mode == 1) s = q_scale(wk_max(mx, red), 7);
    wk_sync();
    quant_row_smem(p, t, s, v, F, p.Kp[3]);
    if (threadIdx.x == 0) p.sa[t] = s;
}

// ------------------------------------------------------------------ attention unit
// (seq b, kv head g): q/k/v epilogue + RoPE + int4 K/V append + attention for the
// group's query heads over the cache (rows 0..len).
template <int DH>
QT_DEV void attn_unit(const MkParams& p, int l, int b, int kh, float* scratch) {
    constexpr int CPL = DH / 4;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int q4 = lane & 3, quad = lane >> 2;
    const MkLayer& ly = p.layers[l];
    const int* accq = p.acc[0] + (size_t)b * p.acc_ld[0];
    const double* sq = ly.s[0];
    const double a_s = __ldcg(p.sa + b);
    const int pos = __ldcg(p.next_pos + b);
    const int r = __ldcg(ly.kv_len + b);  // the new row's index
    const int len = r + 1;
    const int H = p.H, Hkv = p.Hkv, hpg = H / Hkv;
    const double2* rt = p.rope + (size_t)pos * (DH / 2);
    uint8_t* page = p.pool + (long long)ly.pt[b * p.max_pages + r / kPage] * p.page_bytes;
    const size_t cb = (size_t)Hkv * kPage * (DH / 2);
    // --- K and V rows of this head: warp 0 -> K, warp 1 -> V (E = DH/32 elements per lane)
    if (warp < 2) {
        constexpr int E = DH / 32;
        const bool is_k = warp == 0;
        const int n0 = (is_k ? H * DH : (H + Hkv) * DH) + kh * DH;
        double val[E];
#pragma unroll
        for (int j = 0; j < E; ++j) {
            const int n = n0 + lane * E + j;
            val[j] = (double)(float)((double)__ldcg(accq + n) * (a_s * sq[n]));
        }
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
    float* sm_ml = scratch;               // [8 warps][2]
    float* sm_o = scratch + 16;           // [8 warps][DH]
    int* spt = reinterpret_cast<int*>(scratch + 16 + 8 * DH);  // this sequence's page table
    for (int j = threadIdx.x; j < (len + kPage - 1) / kPage; j += MK_WORKERS) spt[j] = __ldg(ly.pt + b * p.max_pages + j);
    __threadfence_block();
    wk_sync();
    const float inv_sqrt = (float)(1.0 / sqrt((double)DH));
    for (int hh = 0; hh < hpg; ++hh) {
        const int h = kh * hpg + hh;
        // q (RoPE'd, rounded to fp32 like the unfused path): lane holds channels q4*CPL..
        float q[CPL];
#pragma unroll
        for (int c = 0; c < CPL; c += 2) {
            const int ch = q4 * CPL + c;
            const int n = h * DH + ch;
            const double a = (double)(float)((double)__ldcg(accq + n) * (a_s * sq[n]));
            const double bb = (double)(float)((double)__ldcg(accq + n + 1) * (a_s * sq[n + 1]));
            const double2 cs = rt[ch / 2];
            q[c] = (float)__dsub_rn(__dmul_rn(a, cs.x), __dmul_rn(bb, cs.y));
            q[c + 1] = (float)__dadd_rn(__dmul_rn(a, cs.y), __dmul_rn(bb, cs.x));
        }
        float m = -1e30f, lsum = 0.f;
        float o[CPL];
#pragma unroll
        for (int c = 0; c < CPL; ++c) o[c] = 0.f;
        // rows: warp w takes 32-row blocks w, w+8, ...; quad q of the warp rows q, q+8, q+16, q+24
        // of the block (4 lanes per row, each 16 bytes of int4 codes); all loads of a block are
        // issued before any math
        constexpr int R = 4;
        for (int r0 = warp * 32; r0 < len; r0 += 256) {
            uint32_t kw[R][CPL / 8], vw[R][CPL / 8];
            float sk[R], sv[R];
#pragma unroll
            for (int i = 0; i < R; ++i) {
                const int row = r0 + quad + 8 * i;
                const bool valid = row < len;
                const uint8_t* pg = p.pool + (long long)spt[valid ? row / kPage : 0] * p.page_bytes;
                const int slot = valid ? row % kPage : 0;
                const uint8_t* krow = pg + ((size_t)kh * kPage + slot) * (DH / 2) + q4 * (CPL / 2);
                if (CPL == 32) {
                    const uint4 ka = valid ? __ldcg(reinterpret_cast<const uint4*>(krow)) : make_uint4(0, 0, 0, 0);
                    const uint4 va = valid ? __ldcg(reinterpret_cast<const uint4*>(krow + cb)) : make_uint4(0, 0, 0, 0);
                    kw[i][0] = ka.x; kw[i][1] = ka.y; kw[i][2] = ka.z; kw[i][3] = ka.w;
                    vw[i][0] = va.x; vw[i][1] = va.y; vw[i][2] = va.z; vw[i][3] = va.w;
                } else {
                    const uint2 ka = valid ? __ldcg(reinterpret_cast<const uint2*>(krow)) : make_uint2(0, 0);
                    const uint2 va = valid ? __ldcg(reinterpret_cast<const uint2*>(krow + cb)) : make_uint2(0, 0);
                    kw[i][0] = ka.x; kw[i][1] = ka.y;
                    vw[i][0] = va.x; vw[i][1] = va.y;
                }
                const float* scp = reinterpret_cast<const float*>(pg + 2 * cb);
                sk[i] = valid ? __ldcg(scp + kh * kPage + slot) : 0.f;
                sv[i] = valid ? __ldcg(scp + Hkv * kPage + kh * kPage + slot) : 0.f;
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
        // merge the 8 quads of the warp
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
        wk_sync();
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
            p.attn[(size_t)b * p.d + h * DH + threadIdx.x] = oo / ll;
        }
        wk_sync();
    }
}

QT_DEV void zero_row(int* a, int n) {
    for (int i = threadIdx.x; i < n; i += MK_WORKERS) a[i] = 0;
}

// ------------------------------------------------------------------ the kernel
template <int DH>
__global__ void __launch_bounds__(MK_THREADS, 1) k_decode_mk(const MkParams p) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* ring = smem;
    uint8_t* As = ring + (size_t)p.nslot * MK_SLOT;
    const int kmax = max(p.Kp[0], p.Kp[3]);
    int* sacc = reinterpret_cast<int*>(As + (size_t)MK_TOK * p.a_ld);
    uint64_t* full = reinterpret_cast<uint64_t*>(sacc + p.acc_rows * 16 * MK_TOK);
    uint64_t* empty = full + p.nslot;
    __shared__ double red[32];
    __shared__ int s_last;
    (void)kmax;
    if (threadIdx.x == MK_WORKERS) {
        for (int i = 0; i < p.nslot; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 8);
        }
        mbar_fence_init();
    }
    __syncthreads();
    if (threadIdx.x >= MK_WORKERS) {  // producer warp
        if (threadIdx.x == MK_WORKERS) producer(p, ring, full, empty);
        return;
    }
    unsigned* bar = p.sync;              // + flag at p.sync + 32
    unsigned* owner_done = p.sync + 64;
    unsigned* attn_done = p.sync + 96;
    unsigned* unit_cnt = p.sync + 128;   // [8]
    const unsigned G = gridDim.x;
    unsigned nbar = 0, nown = 0;
    int slot = 0;
    uint32_t phase = 0;
    const int t_own = blockIdx.x < (unsigned)p.B ? (int)blockIdx.x : -1;
    double* stage = reinterpret_cast<double*>(As);  // owner-phase staging row (As is idle then)
#define TR(ev) \
    if (p.trace && threadIdx.x == 0) p.trace[((size_t)blockIdx.x * (p.L + 1) + l) * 32 + (ev)] = gtimer();
    for (int l = 0; l <= p.L; ++l) {
        TR(0);
        const bool head = l == p.L;
        const MkLayer* ly = head ? nullptr : &p.layers[l];
        // ---- S0: residual (previous down-proj) + norm1 (or final norm) + quantize
        if (t_own >= 0) {
            const int* accr = l > 0 ? p.acc[3] + (size_t)t_own * p.acc_ld[3] : nullptr;
            const double* sw = l > 0 ? p.layers[l - 1].s[3] : nullptr;
            const float* gain = head ? p.gf : ly->g1;
            const double site = head ? p.act[4 * p.L] : p.act[4 * l + 0];
            owner_norm_quant(p, t_own, accr, sw, gain, site, red, stage,
                             p.trace ? p.trace + ((size_t)blockIdx.x * (p.L + 1) + l) * 32 : nullptr);
            TR(14);
            wk_sync();
            if (l > 0) zero_row(p.acc[3] + (size_t)t_own * p.acc_ld[3], p.d);
            if (!head) zero_row(p.acc[1] + (size_t)t_own * p.acc_ld[1], p.d);
            signal(owner_done);
        }
        ++nown;
        wait_count(owner_done, nown * (unsigned)p.B);
        TR(1);
        // ---- S1: QKV GEMV (or head)
        {
            const int g = head ? 4 * p.L : 4 * l;
            const Gemv v = gemv_of(p, g);
            load_act(p, p.Kp[0], As);
            gemv_consume(p, v, head ? p.acc[4] : p.acc[0], head ? p.acc_ld[4] : p.acc_ld[0], ring, full, empty, slot,
                         phase, As, sacc);
            TR(2);
            grid_barrier(bar, ++nbar * G);
            TR(3);
        }
        if (head) {
            // logits = head epilogue; decode state bump (model.cpp:553-556)
            if (t_own >= 0) {
                int* ar = p.acc[4] + (size_t)t_own * p.acc_ld[4];
                const double a_s = __ldcg(p.sa + t_own);
                for (int n = threadIdx.x; n < p.d; n += MK_WORKERS) {
                    p.logits[(size_t)t_own * p.d + n] = (float)((double)__ldcg(ar + n) * (a_s * p.s_head[n]));
                }
                wk_sync();
                zero_row(ar, p.d);
                for (int ll = threadIdx.x; ll < p.L; ll += MK_WORKERS) p.layers[ll].kv_len[t_own] += 1;
                if (threadIdx.x == 0) p.next_pos[t_own] += 1;
            }
            break;
        }
        // ---- S2: attention units (seq, kv head); the last unit of a sequence quantizes its row
        {
            const int units = p.B * p.Hkv;
            float* scratch = reinterpret_cast<float*>(As);
            for (int u = blockIdx.x; u < units; u += G) {
                const int b = u / p.Hkv, kh = u % p.Hkv;
                attn_unit<DH>(p, l, b, kh, scratch);
                wk_sync();
                if (threadIdx.x == 0) {
                    __threadfence();
                    const unsigned old = atomicAdd(&unit_cnt[b], 1u);
                    s_last = old == (unsigned)(p.Hkv * (l + 1) - 1);
                    __threadfence();
                }
                wk_sync();
                if (s_last) {
                    attn_row_quant(p, l, b, red, reinterpret_cast<float*>(stage));
                    wk_sync();
                    zero_row(p.acc[0] + (size_t)b * p.acc_ld[0], p.N[0]);
                    signal(attn_done);
                }
            }
        }
        TR(4);
        wait_count(attn_done, (unsigned)((l + 1) * p.B));
        TR(5);
        // ---- S4: O GEMV
        {
            const Gemv v = gemv_of(p, 4 * l + 1);
            load_act(p, p.Kp[1], As);
            gemv_consume(p, v, p.acc[1], p.acc_ld[1], ring, full, empty, slot, phase, As, sacc);
            TR(6);
            grid_barrier(bar, ++nbar * G);
            TR(7);
        }
        // ---- S5: x += O ; norm2 + quantize
        if (t_own >= 0) {
            const int* accr = p.acc[1] + (size_t)t_own * p.acc_ld[1];
            owner_norm_quant(p, t_own, accr, ly->s[1], ly->g2, p.act[4 * l + 2], red, stage);
            wk_sync();
            zero_row(p.acc[2] + (size_t)t_own * p.acc_ld[2], p.N[2]);
            signal(owner_done);
        }
        ++nown;
        wait_count(owner_done, nown * (unsigned)p.B);
        TR(8);
        // ---- S6: gate|up GEMV
        {
            const Gemv v = gemv_of(p, 4 * l + 2);
            load_act(p, p.Kp[2], As);
            gemv_consume(p, v, p.acc[2], p.acc_ld[2], ring, full, empty, slot, phase, As, sacc);
            TR(9);
            grid_barrier(bar, ++nbar * G);
            TR(10);
        }
        // ---- S7: mlp_mid
        if (t_own >= 0) {
            owner_mid_quant(p, l, t_own, red, reinterpret_cast<float*>(stage));
            TR(15);
            signal(owner_done);
        }
        ++nown;
        wait_count(owner_done, nown * (unsigned)p.B);
        TR(11);
        // ---- S8: down GEMV
        {
            const Gemv v = gemv_of(p, 4 * l + 3);
            load_act(p, p.Kp[3], As);
            gemv_consume(p, v, p.acc[3], p.acc_ld[3], ring, full, empty, slot, phase, As, sacc);
            TR(12);
            grid_barrier(bar, ++nbar * G);
            TR(13);
        }
    }
#undef TR
}

}  // namespace qt

using namespace qt;

extern "C" {

// smem plan: ring slots fill what the activation rows and the accumulator leave
int qt_decode_mk_smem(int kmax_pad, int acc_rows, int nslot, int* a_ld) {
    *a_ld = kmax_pad / 2 + 64;
    return nslot * MK_SLOT + MK_TOK * (*a_ld) + acc_rows * 16 * MK_TOK * 4 + 2 * nslot * 8;
}

int qt_launch_decode_mk(const void* params, int dh, int grid, int smem, cudaStream_t st) {
    const MkParams& p = *static_cast<const MkParams*>(params);
    auto kfn = dh == 128 ? k_decode_mk<128> : k_decode_mk<64>;
    if (dh != 128 && dh != 64) return -1;
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e) return (int)e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(MK_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident: the grid barriers rely on it
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return (int)cudaLaunchKernelEx(&cfg, kfn, p);
}

int qt_decode_mk_params_size() { return (int)sizeof(MkParams); }
int qt_decode_mk_layer_size() { return (int)sizeof(MkLayer); }

}  // extern "C"
