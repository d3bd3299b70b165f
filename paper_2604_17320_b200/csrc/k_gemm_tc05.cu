// k_gemm_tc05.cu -- tcgen05 (kind::i8, TMEM accumulators) W4A4 GEMM.  (in progress)
#include "qt_common.cuh"
#include "qt_kernels.h"

extern "C" int qt_launch_w4a4_tc05(int, const uint8_t*, int, const double*, const uint8_t*, int, const double*, int,
                                   int, int, void*, int, int*, cudaStream_t) {
    return -1;
}
