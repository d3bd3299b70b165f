// qt_epilogue.cuh -- fused GEMM/GEMV epilogues shared by the mma.sync and tcgen05 paths.
#pragma once

#include "qt_common.cuh"
#include "qt_kernels.h"

namespace qt {

// SiLU / SwiGLU of the fp64 GEMM outputs, evaluated in fp32 in the tcgen05
// prefill epilogue (epi_row32): the result is an fp32 tensor (the mlp_mid site
// input), and fp64 exp/div there made the epilogue, not the tensor cores, the
// bottleneck of the gate|up GEMM.  The row-wise epi_store (decode GEMV) keeps fp64.
QT_DEV float silu_f32(double g) {
    const float gf = (float)g;
    // approximate divide (2 ulp; 0 once 1 + e^-g > 2^126, where silu underflows anyway): the
    // IEEE division's subroutine call dominated the gate|up epilogue (ncu source page);
    // expf stays the accurate one (the mlp_mid quantizer's tie budget, tests/replay.py)
    return __fdividef(gf, 1.0f + expf(-gf));
}

// int32 -> fp64 without the F64 conversion unit: (2^52 + 2^31 + a) as bits, minus the offset (exact)
QT_DEV double i2d_exact(int a) {
    return __hiloint2double(0x43300000, (unsigned)a ^ 0x80000000u) - 4503601774854144.0;
}

// y = (acc / 256) * s_a[m] * s_w[n] in fp64 (scales are the reference's fp64
// scales; the integer sum is exact), then the epilogue: store fp32, add into
// the fp64 residual, SiLU, or SwiGLU over interleaved (gate, up) columns.
// Returns max |v| over the fp32 values written (0 for the residual add): the
// producer-side partial row max the dynamic quantizer of the next site reads.
template <int EPI>
QT_DEV float epi_store(void* __restrict__ outv, int ldo, int m, int n, double y0, double y1, int N) {
    if (EPI == QT_EPI_RESADD) {
        double* p = static_cast<double*>(outv) + (size_t)m * ldo + n;
        if (n + 1 < N) {
            double2 v = *reinterpret_cast<double2*>(p);
            v.x += y0;
            v.y += y1;
            *reinterpret_cast<double2*>(p) = v;
        } else if (n < N) {
            p[0] += y0;
        }
        return 0.f;
    }
    float* out = static_cast<float*>(outv);
    if (EPI == QT_EPI_SWIGLU) {
        // silu(g) * u (model.cpp:170-172 silu; SwiGLU is the R1 extension)
        // fp64 here (decode GEMV / small GEMMs: a handful of rows), so the fp32 result is the
        // correctly rounded value of the reference's fp64 expression
        if (n >= N) return 0.f;
        const float v = (float)(y0 / (1.0 + exp(-y0)) * y1);
        out[(size_t)m * ldo + n / 2] = v;
        return fabsf(v);
    }
    float* p = out + (size_t)m * ldo + n;
    float v0, v1;
    if (EPI == QT_EPI_SILU) {
        v0 = (float)(y0 / (1.0 + exp(-y0)));
        v1 = (float)(y1 / (1.0 + exp(-y1)));
    } else {
        v0 = (float)y0;
        v1 = (float)y1;
    }
    if (n + 1 < N) {
        *reinterpret_cast<float2*>(p) = make_float2(v0, v1);
        return fmaxf(fabsf(v0), fabsf(v1));
    }
    if (n < N) {
        p[0] = v0;
        return fabsf(v0);
    }
    return 0.f;
}

// 32 consecutive columns of one row (tcgen05.ld 32x32b: one row per thread).
// mx: running max |v| of the fp32 values written (untouched by the residual add).
template <int EPI>
QT_DEV void epi_row32(void* __restrict__ outv, int ldo, int m, int n, const uint32_t* r, double a_s,
                      const double* swt, float& mx) {
    if (EPI == QT_EPI_RESADD) {
        double* p = static_cast<double*>(outv) + (size_t)m * ldo + n;
        if ((reinterpret_cast<uintptr_t>(p) & 31) == 0) {  // 256-bit row accesses: full sectors
#pragma unroll
            for (int e = 0; e < 32; e += 8) {
                double4 v0 = ld_v4f64(p + e), v1 = ld_v4f64(p + e + 4);
                double* w0 = &v0.x;
                double* w1 = &v1.x;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    w0[u] += i2d_exact((int)r[e + u] >> 8) * (a_s * swt[e + u]);
                    w1[u] += i2d_exact((int)r[e + 4 + u] >> 8) * (a_s * swt[e + 4 + u]);
                }
                st_v4f64(p + e, v0);
                st_v4f64(p + e + 4, v1);
            }
            return;
        }
        double2* p2 = reinterpret_cast<double2*>(p);
#pragma unroll
        for (int e = 0; e < 32; e += 8) {
            double2 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = p2[e / 2 + u];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                v[u].x += i2d_exact((int)r[e + 2 * u] >> 8) * (a_s * swt[e + 2 * u]);
                v[u].y += i2d_exact((int)r[e + 2 * u + 1] >> 8) * (a_s * swt[e + 2 * u + 1]);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) p2[e / 2 + u] = v[u];
        }
        return;
    }
    float* out = static_cast<float*>(outv);
    if (EPI == QT_EPI_SWIGLU) {
        float* pf = out + (size_t)m * ldo + n / 2;
        const bool wide = (reinterpret_cast<uintptr_t>(pf) & 31) == 0;
#pragma unroll
        for (int e = 0; e < 32; e += 16) {
            float v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const double g = i2d_exact((int)r[e + 2 * u] >> 8) * (a_s * swt[e + 2 * u]);
                const double up = i2d_exact((int)r[e + 2 * u + 1] >> 8) * (a_s * swt[e + 2 * u + 1]);
                v[u] = silu_f32(g) * (float)up;
                mx = fmaxf(mx, fabsf(v[u]));
            }
            if (wide) {
                st_v8f32(pf + e / 2, v);
            } else {
                reinterpret_cast<float4*>(pf + e / 2)[0] = make_float4(v[0], v[1], v[2], v[3]);
                reinterpret_cast<float4*>(pf + e / 2)[1] = make_float4(v[4], v[5], v[6], v[7]);
            }
        }
        return;
    }
    float* pf = out + (size_t)m * ldo + n;
    const bool wide = (reinterpret_cast<uintptr_t>(pf) & 31) == 0;
#pragma unroll
    for (int e = 0; e < 32; e += 8) {
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const double y = i2d_exact((int)r[e + u] >> 8) * (a_s * swt[e + u]);
            v[u] = EPI == QT_EPI_SILU ? silu_f32(y) : (float)y;
            mx = fmaxf(mx, fabsf(v[u]));
        }
        if (wide) {
            st_v8f32(pf + e, v);
        } else {
            reinterpret_cast<float4*>(pf + e)[0] = make_float4(v[0], v[1], v[2], v[3]);
            reinterpret_cast<float4*>(pf + e)[1] = make_float4(v[4], v[5], v[6], v[7]);
        }
    }
}

}  // namespace qt
