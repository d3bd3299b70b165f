// qt_epilogue.cuh -- fused GEMM/GEMV epilogues shared by the mma.sync and tcgen05 paths.
#pragma once

#include "qt_common.cuh"
#include "qt_kernels.h"

namespace qt {

// y = (acc / 256) * s_a[m] * s_w[n] in fp64 (scales are the reference's fp64
// scales; the integer sum is exact), then the epilogue: store fp32, add into
// the fp64 residual, SiLU, or SwiGLU over interleaved (gate, up) columns.
template <int EPI>
QT_DEV void epi_store(void* __restrict__ outv, int ldo, int m, int n, double y0, double y1, int N) {
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
        return;
    }
    float* out = static_cast<float*>(outv);
    if (EPI == QT_EPI_SWIGLU) {
        // silu(g) * u (model.cpp:170-172 silu; SwiGLU is the R1 extension)
        if (n < N) out[(size_t)m * ldo + n / 2] = (float)(y0 / (1.0 + exp(-y0)) * y1);
        return;
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
    if (n + 1 < N) *reinterpret_cast<float2*>(p) = make_float2(v0, v1);
    else if (n < N) p[0] = v0;
}

}  // namespace qt
