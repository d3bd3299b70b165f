// Dependent-launch floor on this GPU: a CUDA graph of N chained kernels (PDL or plain),
// grids of 8 / 148 / 296 CTAs; prints microseconds per kernel.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* p, int pdl) {
    if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 0) atomicAdd(p + blockIdx.x % 8, 1);
    if (pdl) asm volatile("griddepcontrol.launch_dependents;");
}
int main() {
    int* d; cudaMalloc(&d, 4096); cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    for (int pdl = 0; pdl < 2; ++pdl)
        for (int grid : {8, 148, 296}) {
            const int N = 320;
            cudaGraph_t g; cudaGraphExec_t ge;
            cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
            for (int i = 0; i < N; ++i) {
                cudaLaunchConfig_t cfg = {}; cudaLaunchAttribute at[1];
                cfg.gridDim = grid; cfg.blockDim = 256; cfg.stream = s;
                at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization; at[0].val.programmaticStreamSerializationAllowed = 1;
                cfg.attrs = at; cfg.numAttrs = pdl;
                cudaLaunchKernelEx(&cfg, k, d, pdl);
            }
            cudaStreamEndCapture(s, &g); cudaGraphInstantiate(&ge, g, 0);
            cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
            cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
            cudaEventRecord(a, s); for (int r = 0; r < 5; ++r) cudaGraphLaunch(ge, s); cudaEventRecord(b, s);
            cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b);
            printf("pdl=%d grid=%3d: %.2f us per kernel\n", pdl, grid, ms * 1e3 / (5 * N));
        }
    return 0;
}
