// qt_decode_mk.h -- parameter block of the persistent decode kernel (k_decode_mk.cu),
// shared with the host engine (engine.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace qt {

struct MkLayer {
    const uint8_t* w[4];  // qkv, o, gate|up, down: tiled int4 codes
    const double* s[4];   // per-output-channel scales
    int rows_pad[4];
    const float* g1;
    const float* g2;
    const int* pt;  // page table [max_batch][max_pages]
    int* kv_len;    // [max_batch]
};

struct MkParams {
    const MkLayer* layers;
    int L, d, H, Hkv, dh, dff, mlp, act_mode, B;
    int N[4];     // rows of qkv, o, gate|up, down
    int Kp[4];    // padded K of qkv, o, gate|up, down
    const uint8_t* head;
    const double* s_head;
    int head_rows_pad;
    const float* gf;
    const double* act;  // 4L + 1 static scales (act_mode 0)
    double* x;          // [B][d] fp64 residual (the step's input)
    int* acc[5];        // int32 [8][N] accumulators: qkv, o, gu, down, head
    int acc_ld[5];
    uint8_t* codes;  // tiled [16 rows x Kmax/2]
    double* sa;      // [16]
    float* attn;     // [8][d]
    uint8_t* pool;
    long long page_bytes;
    int max_pages;
    const double2* rope;  // [max_pos][dh/2] (cos, sin)
    int* next_pos;
    float* logits;  // [B][d]
    unsigned* sync;  // [256]: 0 barrier arrivals, 32 barrier flag, 64 owner done, 96 attention rows done, 128.. per-seq unit counts
    int nslot;
    int a_ld;     // smem bytes per token row of the activation codes
    int acc_rows; // smem accumulator rows
    unsigned long long* trace;  // optional [G][L+1][16] globaltimer stamps (phase timing)
};

}  // namespace qt

extern "C" {
// smem bytes for a ring of nslot 8 KB slots + activation rows + accumulator rows; a_ld out
int qt_decode_mk_smem(int kmax_pad, int acc_rows, int nslot, int* a_ld);
int qt_launch_decode_mk(const void* params, int dh, int grid, int smem, cudaStream_t st);
}
