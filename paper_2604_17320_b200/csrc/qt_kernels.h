// qt_kernels.h -- internal launcher prototypes (host side, C linkage).
// Every launcher takes caller-owned device buffers and an explicit stream and
// returns 0 or a CUDA/argument error code; no hidden allocation.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define QT_EPI_STORE 0   // out = y
#define QT_EPI_RESADD 1  // out += y           (residual add, model.cpp:396,437)
#define QT_EPI_SILU 2    // out = silu(y)      (model.cpp:433)
#define QT_EPI_SWIGLU 3  // out[n/2] = silu(y[n]) * y[n+1], gate/up interleaved columns

#ifdef __cplusplus
extern "C" {
#endif

int qt_launch_f32_to_f64(const float* a, double* b, long long n, cudaStream_t st);
int qt_launch_norm_quant(const void* x, int x_is_f64, int ld_x, const float* gain, int M, int D, int d_pad,
                         int bits, int mode, double static_scale, uint8_t* codes, int ld_codes, double* scales,
                         float* normed, int8_t* codes8, int ld8, cudaStream_t st);
int qt_launch_rope_kv_append(float* qkv, int ld_qkv, int M, int H, int Hkv, int dh, const int* pos,
                             const int* tok_seq, const int* tok_row, const double* rope, const int* page_table,
                             int max_pages, uint8_t* pool, long long page_bytes, int bits, float* k_dbg,
                             cudaStream_t st);
int qt_launch_token_metrics(const double* x, int D, const int* seq_off, const int* vis, int vmax, int B,
                            int vstride, int res_bits, double* mag, double* res, cudaStream_t st);
int qt_launch_weight_quant(const float* w, int K, int N, int bits, int row_mul, int row_add, uint8_t* codes,
                           int ldc, double* scales, double* colmax_scratch, cudaStream_t st);
// full-precision (fp64) calibration forward pieces (k_fp.cu)
int qt_launch_fp_rmsnorm(const double* x, const float* gain, int M, int D, double* out, unsigned long long* obs,
                         cudaStream_t st);
int qt_launch_fp_rope(double* qkv, int ldq, int M, int nheads_qk, int dh, const int* pos, const double* rope,
                      cudaStream_t st);
int qt_launch_fp_attention(const double* qkv, int ldq, int H, int Hkv, int dh, int S, int V, double* out, int ldo,
                           unsigned long long* obs, double* probs, cudaStream_t st);
int qt_launch_fp_colsum(const double* probs, int H, int S, int V, double* inter, double* intra, cudaStream_t st);
int qt_launch_fp_mlp_act(const double* g, const double* u, long long n, double* mid, unsigned long long* obs,
                         cudaStream_t st);
int qt_launch_diag_top10(const float* qkv, int ldq, int H, int Hkv, int dh, int V, int S, const uint8_t* pool,
                         long long page_bytes, const int* pt, double* out, cudaStream_t st);
int qt_launch_codes_pack(const int8_t* src, int K, int N, const double* s_in, int row_mul, int row_add,
                         uint8_t* codes, int ldc, double* scales, cudaStream_t st);
// out: double* for QT_EPI_RESADD (the fp64 residual stream), float* otherwise
// int8-operand tcgen05 GEMM (operands 16 x code, k natural order, row-major; TMA SW128)
int qt_launch_w4a4_tc05_i8(int epi, const int8_t* A8, int lda8, const double* sa, const int8_t* W8, int w_rows,
                           int ldw8, const double* sw, int M, int N, int K, void* out, int ldo, int* acc_dbg,
                           float* pmax, int pmax_ld, int* n_part, int* ws, cudaStream_t st);
// ws (nullable): int32 split-K workspace of qt_tc05_i8_splitk(M, N, K) * M * N entries (the 2-SM kernel
// splits K when its 256 x 256 tiles would leave CTA pairs idle: decode batches of 129..256 tokens)
int qt_tc05_i8_splitk(int M, int N, int K);
int qt_launch_w4a4_tc05_i8_ex(int epi, const int8_t* A8, int lda8, const double* sa, const int8_t* W8, int w_rows,
                              int ldw8, const double* sw, int M, int N, int K, void* out, int ldo, int* acc_dbg,
                              float* pmax, int pmax_ld, int* n_part, int* ws, int flags, cudaStream_t st);
int qt_launch_w4t_to_i8(const uint8_t* tiled, int rows_pad, int K, int8_t* out, cudaStream_t st);
int qt_launch_w4a4_mma_ex(int epi, const uint8_t* A, int lda, const double* sa, const uint8_t* W, int ldw,
                          const double* sw, int M, int N, int K, void* out, int ldo, int* acc_dbg, float* pmax,
                          int pmax_ld, int* n_part, cudaStream_t st);
int qt_launch_w4a4_tc05_ex(int epi, const uint8_t* A, int lda, const double* sa, const uint8_t* W, int ldw,
                           const double* sw, int M, int N, int K, void* out, int ldo, int* acc_dbg, int* ws,
                           float* pmax, int pmax_ld, int* n_part, cudaStream_t st);
// dynamic int4 quantizer of fp32 rows whose max |x| is given as producer partials
// (pmax[m * pmax_ld + p], p < n_part): no row reduction; mode 0 = static scale
int qt_launch_quant_pmax(const float* x, int ld_x, const float* pmax, int n_part, int pmax_ld, int M, int D,
                         int d_pad, int qmax, int mode, double static_scale, uint8_t* codes, int ld_codes,
                         double* scales, int8_t* codes8, int ld8, cudaStream_t st);
int qt_launch_w4a4_mma(int epi, const uint8_t* A, int lda, const double* sa, const uint8_t* W, int ldw,
                       const double* sw, int M, int N, int K, void* out, int ldo, int* acc_dbg, cudaStream_t st);
// ws (nullable): int32 split-K workspace of qt_tc05_splitk(M, N, K) * M * N entries; with ws the
// GEMM splits K across CTAs when its tiles would underfill the SMs (decode batches 17..256)
int qt_tc05_splitk(int M, int N, int K);
int qt_launch_w4a4_tc05(int epi, const uint8_t* A, int lda, const double* sa, const uint8_t* W, int ldw,
                        const double* sw, int M, int N, int K, void* out, int ldo, int* acc_dbg, int* ws,
                        cudaStream_t st);
// pmax (may be null): max |out| per (token row, head), pmax[row * pmax_ld + h]
int qt_launch_attn_prefill(const float* qkv, int ldq, int H, int Hkv, int dh, const int* seq_off, const int* vis,
                           const int* seq_len, int B, int smax, const uint8_t* pool, long long page_bytes,
                           const int* pt, int max_pages, float* out, int ldo, float* ml, float* pmax, int pmax_ld,
                           cudaStream_t st);
int qt_launch_attn_colsum(const float* qkv, int ldq, int H, int Hkv, int dh, const int* seq_off, const int* vis,
                          const int* seq_len, int B, int vmax, const uint8_t* pool, long long page_bytes,
                          const int* pt, int max_pages, const float* ml, int vstride, float* inter, float* intra,
                          float* probs, int p_rows, int p_ld, cudaStream_t st);
// probs (nullable): the softmax probabilities p[b][h][query < p_rows][visual key < p_ld]
// K6 decode attention (k_attn_decode.cu): grid (nsplit, Hkv, B), pps pages of 64 rows per
// split (qt_attn_decode_plan); rope/pos non-null: the decode step -- q/k RoPE and the new
// token's K/V quantize + append at row kv_len[b] fused in, attention over kv_len[b] + 1
// rows; null: q post-RoPE, kv_len[b] rows.  Then the split merge (fixed order) writing the
// fp32 rows to out (nullable) and/or the attn_out site codes (codes non-null).
int qt_attn_decode_plan(int B, int H, int Hkv, int pages, int sms, int* pps, int* nsplit);
int qt_launch_attn_decode(const float* qkv, int ldq, int H, int Hkv, int dh, const int* kv_len, int B,
                          uint8_t* pool, long long page_bytes, const int* pt, int max_pages, int pps, int nsplit,
                          const double* rope, const int* pos, float* part_ml, float* part_o, float* out, int ldo,
                          uint8_t* codes, int ld_codes, double* scales, int qmode, double static_scale, int d_pad,
                          int bits, int8_t* codes8, int ld8, cudaStream_t st);
int qt_launch_select_topk(const double* mag, const double* res, const float* inter, const float* intra, int H,
                          int vstride, const int* vis, const int* txt, const int* budget, const int* old_off,
                          const int* new_off, int B, int vmax, const double* w4, int* keep_src, int* keep_local,
                          int kl_stride, const int* pos, int* kept_pos, double* fused_out, double* norm_out,
                          const double* met_in, int raw, cudaStream_t st);
int qt_launch_gather_rows(const double* x, double* xn, int D, const int* pos, int* posn, const int* src, int M,
                          cudaStream_t st);
int qt_launch_kv_compact(uint8_t* pool, long long page_bytes, const int* pt, int max_pages, int Hkv, int dh,
                         const int* keep_local, int kl_stride, const int* new_len, int B, cudaStream_t st);
int qt_launch_kv_len_bump(int* kv_len, int n, int* next_pos, int B, cudaStream_t st);
// greedy decoding: token = argmax(logits[b][0..vocab)), x[b] = (double) table[token]
int qt_launch_greedy_next(const float* logits, int ld, int vocab, const float* table, int d, double* x, int* tokens,
                          int B, cudaStream_t st);
int qt_launch_copy_rows_f32(const float* src, const int* rows, int d, float* dst, int B, cudaStream_t st);
// tiled int4 codes -> row-major int8 [rows x K]
int qt_launch_unpack_codes(const uint8_t* tiled, int rows_pad, int rows, int K, int8_t* out, cudaStream_t st);
// per-head fp32 column sums + fp64 token metrics -> metrics [B][4][vstride] (mag, inter, intra, res),
// the head average evaluated exactly as k_select_topk does
int qt_launch_metrics_pack(const double* mag, const double* res, const float* inter, const float* intra, int H,
                           int vstride, const int* vis, int B, double* metrics, cudaStream_t st);

#ifdef __cplusplus
}
#endif
