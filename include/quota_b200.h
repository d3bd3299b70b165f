/* quota_b200.h -- C ABI of the B200-native QUOTA hot path.
 *
 * Drop-in boundary for the reference's deployed low-bit pruned forward pass
 * (/root/reference/proj/include/quota/model.hpp:158-186, selector.hpp:55-57,
 * recipe.hpp:25-54).  Plain pointers and sizes, no C++ or torch types:
 * the reference C++ API (forward_prefill / decode_step / make_recipe_hook /
 * load_recipe) is re-implemented on top of these calls by the C++ host layer
 * (include/quota_b200.hpp), and INTEGRATION.md shows the ctypes binding.
 *
 * Status: every call returns 0 on success or a negative code; the message is
 * available from qt_last_error() (thread-local).  The codes mirror the
 * reference exception types:
 *   QT_EINVAL   std::invalid_argument   (shape / config / recipe violations)
 *   QT_ERUNTIME std::runtime_error      (prune / mode violations)
 *   QT_ERANGE   std::out_of_range
 *   QT_ECUDA    CUDA error (no CPU fallback exists: the path fails loudly)
 *
 * Orientation: weights are given as the reference stores them,
 * W[d_in x d_out] row-major with y = x W (model.hpp:52-57).  Activations are
 * row-major [tokens x d_model], sequences packed back to back, each sequence
 * a visual prefix followed by text (model.hpp:40-50).
 */
#ifndef QUOTA_B200_H
#define QUOTA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QT_OK 0
#define QT_EINVAL (-1)
#define QT_ERUNTIME (-2)
#define QT_ERANGE (-3)
#define QT_ECUDA (-4)

/* Model shape + semantic switches.  Reference semantics (model.hpp:29-37,
 * model.cpp:31-33,212-237): mlp = 0, act_mode = 0, n_kv_heads = n_heads,
 * d_ff = 4 * d_model.  Weight scales are always per output channel
 * (GroupAxis::PerColumn, quant.hpp:22) -- the axis an int32-accumulator GEMM
 * can apply in its epilogue. */
typedef struct qt_config {
    int n_layers;
    int d_model;
    int n_heads;
    int n_kv_heads;  /* GQA when < n_heads */
    int d_head;      /* 64 or 128 */
    int d_ff;
    int mlp;         /* 0 = SiLU MLP (reference), 1 = SwiGLU */
    int act_mode;    /* 0 = static per-tensor site scales (reference), 1 = dynamic per-token */
    int weight_bits; /* 4 */
    int act_bits;    /* 4 */
    int kv_bits;     /* 4 */
} qt_config;

typedef struct qt_engine qt_engine;

const char* qt_last_error(void);

/* Capacity: max_batch sequences per call, max_tokens packed prefill tokens,
 * max_seq tokens per sequence, max_decode decode steps after a prefill. */
int qt_engine_create(const qt_config* cfg, int max_batch, int max_tokens, int max_seq, int max_decode,
                     qt_engine** out);
void qt_engine_destroy(qt_engine* e);
/* cudaStream_t to run on (0 = the engine's own stream).  Device-pointer inputs
 * of qt_engine_prefill / qt_engine_decode must be ready in stream order on this
 * stream (the engine stream is non-blocking: it does not wait for the legacy
 * default stream). */
int qt_engine_set_stream(qt_engine* e, void* stream);
int qt_engine_synchronize(qt_engine* e);
/* make the engine stream wait for a pending asynchronous logits readback */
int qt_engine_join_copies(qt_engine* e);

/* init_model / prepare_quant_env (model.cpp:113-135, 212-237): fp32 weights
 * in reference orientation, quantized on the device to int4 codes with one
 * fp64-derived scale per output channel.  w3 (SwiGLU up) may be null for
 * mlp = 0; gains may be null (= 1.0, model.cpp:129-132).  on_device != 0:
 * the pointers are device pointers. */
int qt_engine_load_layer(qt_engine* e, int layer, const float* wq, const float* wk, const float* wv,
                         const float* wo, const float* w1, const float* w2, const float* w3, const float* g1,
                         const float* g2, int on_device);
int qt_engine_load_head(qt_engine* e, const float* w_head, const float* final_gain, int on_device);
/* Packed-weight loader: a QuantEnv's pre-quantized weights as they are
 * (QuantizedLayerWeights, model.hpp:141-151): int8 codes in [-7, 7], host,
 * reference orientation [d_in x d_out] row-major, with one fp64 scale per
 * OUTPUT channel (GroupAxis::PerColumn).  codes/scales: arrays of 7 pointers in
 * the order wq, wk, wv, wo, w1, w2, w3 (w3 = SwiGLU up; null for mlp = 0).
 * Gains fp64 (null = 1.0).  Bit-identical weights to the caller's QuantEnv. */
int qt_engine_load_layer_codes(qt_engine* e, int layer, const int8_t* const* codes, const double* const* scales,
                               const double* g1, const double* g2);
int qt_engine_load_head_codes(qt_engine* e, const int8_t* codes, const double* scales, const double* final_gain);
/* Calibration.  keep_fp_weights(1) before loading keeps fp64
 * copies of the full-precision weights on the device; fit_act_scales then runs
 * fit_act_scales (calibrator.cpp:237-249): full-precision forward_prefill of
 * each sample (fp64, model.cpp:315-453 with ExecMode::Fp) collecting max|x|
 * at the five quantizer sites (model.cpp:348,393,430,434,443), returning the
 * 4 * n_layers + 1 static per-tensor scales (max/7, all-zero -> 1.0); apply != 0
 * also installs them (qt_engine_set_act_scales).  embs: host fp64
 * [visual+text x d_model] per sample. */
int qt_engine_keep_fp_weights(qt_engine* e, int on);
int qt_engine_fit_act_scales(qt_engine* e, int n_samples, const double* const* embs, const int* visual,
                             const int* text, double* scales_out, int apply);
/* fit_act_scales with a prune hook (calibrator.cpp:237-249 given calib_hook):
 * the fp64 forwards run under the engine's recipe (qt_engine_set_recipe: layers,
 * keeps, v0, metric weights, res_bits -- -1 for nullopt), the scale fit of the
 * prune_then_quant harness mode (harness.cpp:103-106). */
int qt_engine_fit_act_scales_hooked(qt_engine* e, int n_samples, const double* const* embs, const int* visual,
                                    const int* text, double* scales_out, int apply);
/* forward_prefill in ExecMode::Fp (model.cpp:315-453) of n_seq independent
 * samples, fp64 on the device, hook != 0 under the engine's recipe
 * (make_recipe_hook, selector.cpp:211-228, on the fp64 LayerActivationRecord).
 * The fp_baseline / prune_only forwards of the harness (harness.cpp:134-137).
 * logits_out (host fp64, may be NULL): each sample's [final rows x d_model]
 * logits, concatenated, at most cap_rows rows; the trace and final layouts are
 * read with qt_engine_n_prunes / qt_engine_prune / qt_engine_layout.  No device
 * KV cache is kept: qt_engine_decode after this call fails. */
int qt_engine_prefill_fp(qt_engine* e, int n_seq, const double* const* embs, const int* visual, const int* text,
                         int hook, double* logits_out, long long cap_rows);
/* profile_sensitivity (calibrator.cpp:42-82), QUOTA Eq. 1: per listed layer the
 * median over samples of ||x_q - x||_F / (||x||_F + eta) between this engine's
 * quantized block outputs and the fp64 forward's, plus normalize_sensitivities
 * (calibrator.cpp:84-98: P10/P90 clip to [0.1, 0.9], flat -> 0.5). */
int qt_engine_profile_sensitivity(qt_engine* e, int n_samples, const double* const* embs, const int* visual,
                                  const int* text, int n_layers, const int* layers, double eta, double* raw,
                                  double* normalized);
/* profile_diagnostics (calibrator.cpp:147-195) with the quantized forward:
 * per layer, over samples, the median and IQR of the text queries' summed
 * top-10 visual attention mass (averaged over heads and text rows) and the
 * median of the visual rows' median pairwise cosine (numeric.cpp:117-127). */
int qt_engine_profile_diagnostics(qt_engine* e, int n_samples, const double* const* embs, const int* visual,
                                  const int* text, double* conc_median, double* conc_iqr, double* red_median);
/* run_quota_calibration (calibrator.cpp:251-268) on explicit
 * samples: fit_act_scales (installed), profile_diagnostics, select_candidate_
 * layers (window, first 2 and last n_layers/4 excluded, calibrator.cpp:197-223),
 * profile_sensitivity, make_budget_schedule (Eqs. 3-4, calibrator.cpp:100-141).
 * Outputs the recipe's candidate_layers / keep_ratios (window entries each) and
 * optionally the sensitivities [window] and diagnostics [n_layers]. */
int qt_engine_run_quota_calibration(qt_engine* e, int n_samples, const double* const* embs, const int* visual,
                                    const int* text, int window, double p_min, double tau, double eta,
                                    double* act_scales, int* layers, double* keep_ratios, double* raw,
                                    double* normalized, double* conc_median, double* red_median);
/* Packed-int4 weight file (the reference has no checkpoint
 * format -- it regenerates weights from the seed, model.cpp:113-135): the
 * engine's device layout byte for byte (tiled int4 codes, fp64 per-channel
 * scales, gains, static act scales if set) behind a header that must match the
 * engine's qt_config.  Loading is a straight copy, no quantization. */
int qt_engine_save(qt_engine* e, const char* path);
int qt_engine_load(qt_engine* e, const char* path);
/* ActScales (model.hpp:114-133): 4 * n_layers + 1 static per-tensor scales,
 * order (attn_in, attn_out, mlp_in, mlp_mid) per layer, then head_in. */
int qt_engine_set_act_scales(qt_engine* e, const double* scales);

/* make_recipe_hook (selector.cpp:211-228) over a PruningRecipe
 * (recipe.hpp:25-34): validated like PruningRecipe::validate (recipe.cpp:21-46).
 * res_bits < 0 = nullopt (no quantization-residual metric). n_layers = 0 clears. */
int qt_engine_set_recipe(qt_engine* e, int n_layers, const int* layers, const double* keep_ratios,
                         const double* weights4, int v0, int res_bits);
/* parse_recipe (recipe.cpp:91-116) semantics: strict keys, schema_version 1. */
int qt_recipe_parse(const char* json, int max_layers, int* n_layers, int* layers, double* keep_ratios,
                    double* weights4, int* v0, char* quant_digest, int digest_cap);

/* forward_prefill (model.cpp:315-453), quantized mode, recipe hook, for a
 * batch of independent sequences.  emb: packed [sum(visual+text) x d_model].
 * v0: per-sequence reference visual length (null = recipe v0).  positions:
 * packed original position ids (null = 0..S-1 per sequence).  logits_out
 * (nullable): packed [sum(final rows) x d_model]; out_on_device 0 = host,
 * 1 = device, 2 = host read back asynchronously on a copy stream (overlapping
 * the decode steps that follow; valid after qt_engine_synchronize, and
 * qt_engine_join_copies orders the engine stream after it). */
int qt_engine_prefill(qt_engine* e, int n_seq, const float* emb, int emb_on_device, const int* visual,
                      const int* text, const int* v0, const int* positions, float* logits_out, int out_on_device);
/* Same with fp64 embeddings (the reference's Matrix element type). */
int qt_engine_prefill_f64(qt_engine* e, int n_seq, const double* emb, int emb_on_device, const int* visual,
                          const int* text, const int* v0, const int* positions, float* logits_out, int out_on_device);
/* rows of the packed prefill logits (sum over sequences of the final layout) */
int qt_engine_prefill_rows(qt_engine* e);
/* decode_step (model.cpp:455-562) for every sequence of the last prefill:
 * emb [n_seq x d_model], logits_out [n_seq x d_model]. */
int qt_engine_decode(qt_engine* e, const float* emb, int emb_on_device, float* logits_out, int out_on_device);
int qt_engine_decode_f64(qt_engine* e, const double* emb, int emb_on_device, float* logits_out, int out_on_device);
/* Greedy decoding (BASELINE.json configs: "128 greedy steps").  An extension: the reference's
 * decode_step takes the next token's embedding (model.hpp:177-180) and its head is d_model wide
 * (model.hpp:63), so a token is an index into the logits and the caller supplies a
 * token-embedding table [vocab x d_model] fp32, vocab <= d_model.
 * qt_engine_decode_greedy runs one decode_step for every sequence of the last prefill with
 * input table[argmax(previous logits[0..vocab))] (the prefill's last row for the first step;
 * ties to the smaller token id); the argmax + embedding kernel is part of the step's CUDA
 * graph.  tokens_out: int [n_seq], host or device (nullable); logits_out as qt_engine_decode. */
int qt_engine_set_token_table(qt_engine* e, const float* table, int vocab, int on_device);
/* Decode steps replay a captured CUDA graph (on, the default) or launch their kernels eagerly
 * (off; the same kernels and programmatic-dependent launches -- for per-kernel tools such as
 * an ncu launch list, whose graph-node replay of the page-streaming attention kernel fails). */
int qt_engine_set_graphs(qt_engine* e, int on);
int qt_engine_decode_greedy(qt_engine* e, int* tokens_out, float* logits_out, int out_on_device);

/* Introspection (parity tests, reports). */
int qt_engine_layout(qt_engine* e, int seq, int* visual, int* text, int* positions, int cap);
int qt_engine_n_prunes(qt_engine* e, int seq);
int qt_engine_prune(qt_engine* e, int seq, int i, int* layer, int* budget, int* positions, int cap, int* count);
/* QUOTA scores of the last prefill at candidate layer `layer` for sequence
 * `seq` (fuse_scores output, selector.cpp:86-104, and the four
 * robust-normalised metrics mag/inter/intra/res, [4][n]); *n = visual tokens
 * scored.  Null buffers: only *n. */
int qt_engine_scores(qt_engine* e, int layer, int seq, double* fused, double* norm4, int cap, int* n);
int qt_engine_kv(qt_engine* e, int layer, int seq, int kv_head, int which, int8_t* codes, float* scales,
                 int* rows, int cap_rows);
/* device pointers for in-place timing / inspection */
int qt_engine_info(qt_engine* e, int64_t* out16);
/* Profile the next prefill or decode call (decode runs eagerly, not from the
 * graph): per kernel class {gemm, attention, quant, kv, select, other} the
 * CUDA-event time (ms), launches, algorithmic bytes and flops -> out[6*4]. */
int qt_engine_profile_next(qt_engine* e);
int qt_engine_profile_read(qt_engine* e, double* out24);
/* Device time (ms) of one decode step of the current cache restricted to some
 * kernel classes -- skip_mask bits 1 GEMM, 2 attention, 4 quantizers, 8 KV
 * append -- captured as a CUDA graph and replayed reps times back to back
 * (launch overheads and PDL overlap as in the real step).  Cache lengths and
 * positions are restored, so decoding continues unaffected. */
int qt_engine_profile_chain(qt_engine* e, int skip_mask, int reps, double* ms_per_step);
/* ForwardResult::records / block_outputs and arbitrary prune hooks for reference-API
 * callers (model.hpp:74-80,155-156,164-171; model.cpp:380-406,439), one sequence per
 * prefill (B = 1).  qt_engine_set_records(mode): bit 1 keeps every layer's post-block
 * hidden states (qt_engine_block_output), bit 2 every layer's LayerActivationRecord
 * (qt_engine_record_get): the post-attention-residual states of the visual and text rows
 * (fp64) and the softmax probabilities of every query over the visual keys per head
 * (fp32 on the device) -- attn_inter / attn_intra are its text / visual query rows.
 * qt_engine_set_prune_hook: the engine calls hook(user, record, slots, n, budget) at every
 * layer after the attention residual, as forward_prefill calls a PruneHook; return 1 with
 * the retained visual slots (ascending, unique: apply_pruning's rules, violations fail with
 * its messages) to prune on the device, 0 for no retained set (std::nullopt), < 0 to fail.
 * Exclusive with a device recipe (qt_engine_set_recipe).  Both modes synchronise per layer. */
typedef struct qt_layer_record {
    int layer, visual, text, d_model, n_heads;
    const int* positions;         /* [visual + text] original position ids */
    const double* visual_states;  /* [visual x d_model] */
    const double* text_states;    /* [text x d_model] */
    const float* probs;           /* [n_heads x (visual + text) x visual] */
} qt_layer_record;
typedef int (*qt_prune_hook_fn)(void* user, const qt_layer_record* rec, int* slots, int* n_slots, int* budget);
int qt_engine_set_records(qt_engine* e, int mode);
int qt_engine_set_prune_hook(qt_engine* e, qt_prune_hook_fn hook, void* user);
/* records of the last prefill: meta4 = {layer, visual, text, n_heads}; any output may be
 * null (positions [v + t], states [(v + t) x d_model], probs [n_heads x (v + t) x v]) */
int qt_engine_record_count(qt_engine* e);
int qt_engine_record_get(qt_engine* e, int i, int* meta4, int* positions, double* states, float* probs);
int qt_engine_block_output(qt_engine* e, int layer, double* out, long long cap, int* rows);
/* Decision capture (parity / debugging only; never on the product path): with on != 0
 * the following prefill / decode calls read back, after every quantizer site, the int4
 * codes and scales it produced (synchronously; decode steps then run eagerly instead of
 * from the CUDA graph).  Records: meta = {phase (0 prefill, 1 + t decode step t), layer
 * (n_layers for head_in), site (0 attn_in, 1 attn_out, 2 mlp_in, 3 mlp_mid, 4 head_in,
 * 5 K cache rows, 6 V cache rows), rows, cols, groups}; codes int8 [rows x cols] (rows
 * packed by sequence), scales fp64 [rows x groups] (groups = n_kv_heads for K / V, else 1).
 * The quantizer sites are model.cpp:349,394,431,435,444 (static) / quant.cpp:108-110
 * (per token) and the cache rows kv_quantize (quant.cpp:117-119, model.cpp:368-374,499-501).
 * Calling it clears earlier records. */
int qt_engine_capture(qt_engine* e, int on);
int qt_engine_capture_count(qt_engine* e);
int qt_engine_capture_get(qt_engine* e, int i, int* meta6, int8_t* codes, double* scales);

/* ---- per-kernel ABI (caller-owned device buffers, explicit stream) ----
 * int4 code matrices (weights and activations) use the tiled layout of
 * csrc/qt_common.cuh: 1 KB tiles of 16 rows x 128 k, k-block-major; a tiled
 * matrix is described by its padded row count (ld_codes / lda / ldw / ldc
 * below = rows_pad, a multiple of 16) and K. */
/* K1: RMSNorm (gain != null) + int4 activation quantizer; x fp32 or fp64
 * (x_is_f64); act_mode 0 = static_scale, 1 = per-row max|x|/7; fp64 scales. */
int qt_rmsnorm_quant_i4(const void* x, int x_is_f64, int ld_x, const float* gain, int M, int D, int d_pad,
                        int act_mode, double static_scale, uint8_t* codes, int ld_codes, double* scales,
                        float* normed, void* stream);
/* K2: y = s_a[m] s_w[n] sum_k a[m][k] w[n][k]; out is double* for epilogue
 * 1 (residual add), float* otherwise; acc_out (nullable) receives the int32
 * accumulators.  impl 0 = mma.sync GEMM / weight-streaming GEMV (<= 64 tokens);
 * 1 = tcgen05 on packed int4 (converter warps); 2 = the same with split-K across
 * CTAs when its tiles would underfill the SMs (65..128 tokens); 3 = tcgen05 on
 * int8 operands via TMA (2-SM cta_group::2 pairs for M >= 8192; the prefill GEMM);
 * 4 = impl 3 with split-K (decode batches up to 512 tokens: k slices across CTAs, int32
 * partials reduced in fixed order).  Impls 3 and 4
 * widen the operands to int8 in temporary buffers first (the engine keeps them). */
int qt_w4a4_gemm(int epilogue, const uint8_t* a_codes, int lda, const double* a_scales, const uint8_t* w_codes,
                 int ldw, const double* w_scales, int M, int N, int K, void* out, int ldo, int32_t* acc_out,
                 int impl, void* stream);
/* K2 on int8 operands (16 x code, k in natural order, row-major: the prefill layout, see
 * qt_unpack_codes): a8 [>= M x lda8], w8 [w_rows x ldw8]; M >= 8192 runs the 2-SM
 * (cta_group::2) kernel -- flags bit 0 forces the single-CTA one (A/B measurement) --
 * with split-K when workspace (qt_w4a4_gemm_i8_workspace bytes, nullable) is given;
 * flags bits 8..15 = a k-slice count for the single-CTA kernel (measurement; the
 * workspace then needs slices x M x N int32). */
int qt_w4a4_gemm_i8(int epi, const int8_t* a8, int lda8, const double* sa, const int8_t* w8, int w_rows, int ldw8,
                    const double* sw, int M, int N, int K, void* out, int ldo, int32_t* acc_out, int* workspace,
                    int flags, void* stream);
int64_t qt_w4a4_gemm_i8_workspace(int M, int N, int K);
int qt_quant_weight_i4(const float* w, int K, int N, int row_mul, int row_add, uint8_t* codes, int ldc,
                       double* scales, double* scratch, void* stream);
int qt_kv_quant_append_i4(float* qkv, int ld_qkv, int M, int H, int Hkv, int d_head, const int* positions,
                          const int* tok_seq, const int* tok_row, const double* rope_table, const int* page_table,
                          int max_pages, uint8_t* pool, int64_t page_bytes, float* k_out, void* stream);
int qt_rope_table(int max_pos, int d_head, double* host_out);
/* Tiled int4 code matrix (activations or weights, layout above) -> row-major int8
 * [rows x K], one code per byte (parity readback of QuantizedTensor::codes,
 * quant.hpp:32-39). */
int qt_unpack_codes(const uint8_t* tiled, int rows_pad, int rows, int K, int8_t* out, void* stream);
/* K7: masked prefill attention over the paged int4 cache -- masked_attention_probs +
 * matmul(probs, v^) (model.cpp:272-292,366-391) with the reference mask (model.cpp:35-44:
 * visual queries see visual keys only, text queries see every visual key + causal text),
 * keys/values dequantised from the int4 rows (model.cpp:371-372).  q: fp32 post-RoPE
 * queries [sum(S_b) x ldq], head h at column h * d_head; the cache as written by
 * qt_kv_quant_append_i4; seq_off [B + 1], visual [B], seq_len [B]: device ints; smax =
 * max S_b.  out: fp32 [sum(S_b) x ldo]; row_stats (nullable): fp32 [sum(S_b) x H x 2]
 * = (row max, row sum) of the unnormalised softmax (natural-log units), the input of
 * qt_quota_score. */
int qt_attn_prefill_i4kv(const float* q, int ldq, int B, int H, int Hkv, int d_head, const int* seq_off,
                         const int* visual, const int* seq_len, int smax, const uint8_t* pool, int64_t page_bytes,
                         const int* page_table, int max_pages, float* out, int ldo, float* row_stats, void* stream);
/* K6: decode attention (model.cpp:515-535): for each of B sequences one query row, an
 * unmasked softmax over its kv_len[b] (device int) cached rows, int4 K/V dequantised in
 * registers.  q: fp32 post-RoPE [B x ldq]; max_len >= every kv_len[b]; out fp32 [B x ldo];
 * workspace: qt_attn_decode_workspace(B, H, d_head, max_len) bytes of device memory. */
int64_t qt_attn_decode_workspace(int B, int H, int d_head, int max_len);
int qt_attn_decode_i4kv(const float* q, int ldq, int B, int H, int Hkv, int d_head, const int* kv_len, int max_len,
                        const uint8_t* pool, int64_t page_bytes, const int* page_table, int max_pages, float* out,
                        int ldo, void* workspace, void* stream);
/* K3a + K3b: QUOTA token metrics at a candidate layer -- compute_metrics
 * (selector.cpp:19-68): mag_i = ||x_i||, inter_i / intra_i = attention received from
 * text / visual queries summed over heads and divided by H (softmax rebuilt from
 * qt_attn_prefill_i4kv's row_stats), res_i = ||fake_quant_per_row(x_i, res_bits) - x_i||
 * (res_bits < 0: nullopt, 0).  x: fp64 residual [sum(S_b) x d_model]; metrics out: fp64
 * [B][4][vstride] (mag, inter, intra, res), vstride >= vmax = max visual_b; workspace:
 * qt_quota_score_workspace(B, H, vstride) bytes. */
int64_t qt_quota_score_workspace(int B, int H, int vstride);
int qt_quota_score(const double* x, int d_model, const float* q, int ldq, int B, int H, int Hkv, int d_head,
                   const int* seq_off, const int* visual, const int* seq_len, int vmax, const uint8_t* pool,
                   int64_t page_bytes, const int* page_table, int max_pages, const float* row_stats, int res_bits,
                   double* metrics, int vstride, void* workspace, void* stream);
/* K3c + K4 + compaction: score_tokens / select_top_k / apply_pruning (selector.cpp:70-209,
 * numeric.cpp:22-31) for B sequences: robust-normalised metrics fused with weights4
 * (host {mag, inter, intra, quant}), the budget[b] best visual slots (ties to the smaller
 * index, ascending), then x / positions gathered into the new packed layout (retained
 * visual rows, then every text row: new_off [B + 1], new_len [B], new_rows = new_off[B],
 * device) and -- pool != null -- the layer's K/V rows filtered in place.  keep_local
 * [B x vstride] and keep_src [new_rows]: device int scratch (keep_local holds the kept
 * slots); kept_pos (nullable) [B x vstride]: the kept visual positions (PruneEvent). */
int qt_topk_compact(const double* metrics, int B, int vstride, const int* visual, const int* text, const int* budget,
                    const double* weights4, const int* seq_off, const int* new_off, const int* new_len,
                    const double* x, int d_model, const int* pos, int new_rows, double* x_out, int* pos_out,
                    uint8_t* pool, int64_t page_bytes, const int* page_table, int max_pages, int Hkv, int d_head,
                    int* keep_local, int* keep_src, int* kept_pos, void* stream);
/* FNV-1a 64 over raw bytes (digest.hpp:12-20; seed 0xcbf29ce484222325 to
 * start): the harness report digests (sample_set_digest, calibrator.cpp:31-40;
 * recipe_digest, recipe.cpp:132-134; sample_logits_digests, harness.cpp:144). */
uint64_t qt_fnv1a64(const void* data, size_t len, uint64_t seed);
/* K3c + K4 on given metrics: score_tokens (robust_normalize x4 + fuse_scores,
 * selector.cpp:70-115) and select_top_k (selector.cpp:117-136) for B
 * sequences.  metrics: device fp64 [B][4][vstride] in (mag, inter, intra, res)
 * order; visual / budget: device int[B] (V_b <= vstride, budget >= 1);
 * weights4: HOST {mag, inter, intra, quant}, or null = metrics[b][0] already
 * is the fused score (select_top_k alone).  slots: device int[B][vstride],
 * the min(budget, V) retained slots ascending; fused_out [B][vstride] and
 * norm_out [B][4][vstride] nullable. */
int qt_quota_topk(const double* metrics, int B, int vstride, const int* visual, const int* budget,
                  const double* weights4, int* slots, double* fused_out, double* norm_out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* QUOTA_B200_H */
