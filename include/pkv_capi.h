/* pkv_capi.h — C ABI of the B200-native ProxyKV pruning hot path
 * (libpkv_b200.so). Plain pointers and sizes only; no C++ or torch types.
 *
 * Path: proxy scoring -> HybridAxialMapper forward -> per-head Top-K select
 *       -> KV compaction. Each entry point names the reference
 * interface it replaces (paths relative to /root/reference/).
 *
 * Conventions
 *  - Status codes mirror the reference exception taxonomy
 *    (proj/include/proxykv/common.hpp:13-52): PKV_ESHAPE <-> ShapeError,
 *    PKV_EVALUE <-> ValueError, PKV_ECONFIG <-> ConfigError. The message text
 *    (pkv_last_error, thread-local) mirrors the reference PKV_CHECK text.
 *  - "_dev" pointers are device pointers owned by the caller; "_host" pointers
 *    are host memory (pinned or pageable). Device work is stream-ordered on
 *    the given cudaStream_t (passed as void*; NULL = legacy default stream).
 *  - One pkv_ctx per host thread, or external synchronisation.
 *  - There is no CPU fallback: without a usable sm_100 device every compute
 *    entry point returns PKV_ENODEV.
 */
#ifndef PKV_CAPI_H
#define PKV_CAPI_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    PKV_OK = 0,
    PKV_ESHAPE = 1,  /* ShapeError  */
    PKV_EVALUE = 2,  /* ValueError  */
    PKV_ECUDA = 3,   /* CUDA runtime / launch failure */
    PKV_ENCCL = 4,   /* reserved: collective failure */
    PKV_ECONFIG = 5, /* ConfigError (incl. configurations the GPU path does not support) */
    PKV_ENODEV = 6,  /* no sm_100 device */
    PKV_EIO = 7,           /* IoError (common.hpp:33) */
    PKV_EIO_MAGIC = 8,     /* BadMagicError */
    PKV_EIO_VERSION = 9,   /* VersionMismatchError */
    PKV_EIO_TRUNCATED = 10, /* TruncatedFileError */
    PKV_EIO_LENGTH = 11    /* PayloadLengthError */
} pkv_status;

typedef struct pkv_ctx_s* pkv_ctx;
typedef struct pkv_mapper_s* pkv_mapper;
typedef struct pkv_pruner_s* pkv_pruner;

/* ---------------------------------------------------------------- runtime */
int pkv_abi_version(void);
const char* pkv_last_error(void);
/* Number of visible CUDA devices with compute capability 10.x (0 on a CPU box). */
int pkv_sm100_device_count(void);
pkv_status pkv_ctx_create(int device, pkv_ctx* out);
void pkv_ctx_destroy(pkv_ctx ctx);
/* Launches of this library's kernels since ctx creation (for bench accounting). */
int64_t pkv_ctx_launch_count(pkv_ctx ctx);

/* ------------------------------------------------------- select (a-3) ---- */
/* Replaces retention_count, proj/src/pruning.cpp:14-18 (pruning.hpp:14):
 * ceil(rho * n) in double. PKV_EVALUE if rho∉(0,1] or n<=0. */
pkv_status pkv_retention_count(double rho, int64_t n, int64_t* k_out);

/* Replaces topk_indices + topk_mask (proj/src/pruning.cpp:20-56;
 * pruning.hpp:18,32) and the index lists of apply_mask (pruning.cpp:197-215;
 * pruning.hpp:57): for each of `slices` rows of `n` fp32 scores, selects the k
 * best under v[a] > v[b] || (v[a] == v[b] && a < b) (-0.0 == +0.0), writing
 * a 0/1 mask [slices, n] and/or the ascending retained indices [slices, k].
 * Radix select on the GPU; bit-exact with the reference for fp32 scores.
 * PKV_EVALUE if k∉[1,n]. NaN scores: unspecified (as in the reference). */
pkv_status pkv_topk_select(pkv_ctx ctx, const float* scores_dev, int64_t slices, int64_t n, int64_t k,
                           uint8_t* mask_dev, int32_t* idx_asc_dev, void* stream);

/* fp64 device scores [slices, n] (the reference's ScoreTensor element type,
 * tensor.hpp:86): same contract as pkv_topk_select, ranked on 64-bit order keys
 * so distinct doubles never collide (replaces topk_indices / topk_mask,
 * pruning.cpp:20-56, on arbitrary double inputs, bit-exact). */
pkv_status pkv_topk_select_f64(pkv_ctx ctx, const double* scores_dev, int64_t slices, int64_t n, int64_t k,
                               uint8_t* mask_dev, int32_t* idx_asc_dev, void* stream);

/* Host-buffer form of topk_mask (pruning.cpp:37-56): fp64 scores -> mask bits,
 * k = retention_count(rho, n); the doubles are ranked as they are (64-bit
 * keys, bit-exact for any input without NaN); H2D/D2H inside. */
pkv_status pkv_topk_mask_host(pkv_ctx ctx, const double* scores_host, int64_t slices, int64_t n, double rho,
                              uint8_t* bits_host, int64_t* k_out);
/* Replaces topk_indices (pruning.cpp:20-35): the k best of values[0..n) by
 * the reference order (ties to the lower index), fp64 exact; returned in
 * ASCENDING index order (the reference leaves them in nth_element order; the
 * set is identical). PKV_EVALUE "top-k count k out of range for length n". */
pkv_status pkv_topk_indices_host(pkv_ctx ctx, const double* values_host, int64_t n, int64_t k, int64_t* idx_out);
/* Replaces topk_overlap_per_slice (pruning.cpp:91-108) on host masks u8
 * [slices, n] with per-slice count k: |a ∩ b| / k per slice, computed on the
 * device. */
pkv_status pkv_topk_overlap_host(pkv_ctx ctx, const uint8_t* mask_a_host, const uint8_t* mask_b_host, int64_t slices,
                                 int64_t n, int64_t k, double* per_slice_out);

/* Ranking metrics on the device, per slice, fp64:
 * replaces topk_overlap_per_slice (pruning.cpp:91-108: |a ∩ b| / k) and
 * captured_mass_per_slice (pruning.cpp:58-80: sum of y over the predicted mask
 * / sum of y over y's own Top-K, 1 when that is 0). Masks u8 [slices, n]. */
pkv_status pkv_topk_overlap(pkv_ctx ctx, const uint8_t* mask_a_dev, const uint8_t* mask_b_dev, int64_t slices,
                            int64_t n, int64_t k, double* per_slice_out_dev, void* stream);
pkv_status pkv_captured_mass(pkv_ctx ctx, const uint8_t* mask_pred_dev, const float* y_dev, int64_t slices,
                             int64_t n, int64_t k, double* per_slice_out_dev, void* stream);

/* Spearman rank correlation per slice (replaces spearman_per_slice,
 * pruning.cpp:173-186): Pearson correlation of the average ranks (ties share
 * the mean of their 1-based positions, pruning.cpp:122-140) of a and b,
 * fp32 rows [slices, n] (−0 ties with +0, as the reference's double compare);
 * 1 when both rows are constant, 0 when exactly one is. n >= 2 (PKV_EVALUE
 * otherwise, the reference's ValueError). The sums are exact integers; the one
 * rounding is the final division. */
pkv_status pkv_spearman(pkv_ctx ctx, const float* a_dev, const float* b_dev, int64_t slices, int64_t n,
                        double* per_slice_out_dev, void* stream);

/* One MetricAccumulator::add sample on the device (pruning.cpp:218-247):
 * both Top-K masks at k = retention_count(rho, n), then per slice the
 * captured mass of y_pred's mask in y_true, the Top-K overlap of the two
 * masks and the Spearman correlation of y_pred vs y_true. The running means
 * over samples (MetricAccumulator::report) are host arithmetic. */
pkv_status pkv_slice_metrics(pkv_ctx ctx, const float* y_pred_dev, const float* y_true_dev, int64_t slices, int64_t n,
                             int64_t k, double* mass_out_dev, double* overlap_out_dev, double* spearman_out_dev,
                             void* stream);

/* Training loss suite on the device (replaces
 * loss_total, loss.cpp:324-374, with loss_bin / loss_mse / loss_fine /
 * loss_global / loss_cos and their pair sampling, loss.cpp:53-322): logits and
 * ground-truth scores fp32 [shape] on the device (the reference's fp64 inputs
 * must be fp32-representable for parity), computed in fp64. The pair samples
 * are the reference's own (same xoshiro256** streams per slice, same partial
 * Fisher-Yates / Floyd sampling, same filter), so used / filtered counts match
 * exactly. grad_dev (nullable, fp64 [shape]) receives d total / d logits — what
 * the reference's tape computes for report.total_tensor.backward().
 * Errors: LossConfig::validate's messages (PKV_EVALUE), "degenerate oracle"
 * when max(y) <= 0. Synchronises the stream (the report is host memory). */
typedef struct {
    double lambda_mse, lambda_bin, lambda_fine, lambda_global, lambda_cos;
    const double* ratios; /* host array */
    int64_t n_ratios;
    double gamma, epsilon, mse_exponent, margin, clip_lo, clip_hi, pair_filter_frac, topk_ratio_for_rank;
    int64_t max_pairs;
} pkv_loss_config;

typedef struct {
    double bin, mse, fine, global, cos;
    double weighted_bin, weighted_mse, weighted_fine, weighted_global, weighted_cos;
    double total, s_max;
    int64_t fine_used, fine_filtered, global_used, global_filtered, cos_floor_hits;
} pkv_loss_report;

pkv_status pkv_loss_total(pkv_ctx ctx, const float* logits_dev, const float* y_dev, const int64_t* shape, int rank,
                          const pkv_loss_config* cfg, uint64_t seed, pkv_loss_report* report_out, double* grad_dev,
                          void* stream);

/* ------------------------------------------- mapper training (f-4) ---- */
/* GPU training of the HybridAxialMapper: the reference's training forward
 * (forward_pair(x, params, training = true), mapper.cpp:274-342: batchnorm1d
 * on batch statistics with the running-stat EMA, ops.cpp:806-850) and the
 * reverse sweep its tape performs (tensor.cpp:156-199 over the op closures of
 * ops.cpp / mapper.cpp) from d loss / d logits — e.g. pkv_loss_total's
 * grad_dev — to d loss / d every parameter. fp32 on the device (the
 * reference is fp64). A trainer owns an fp32 copy of the blob
 * (pkv_mapper_init_params layout: named_parameters then the BN buffers). */
typedef struct pkv_trainer_s* pkv_trainer;
pkv_status pkv_trainer_create(pkv_ctx ctx, const int64_t* geom5, const int64_t* cfg12, const double* blob,
                              int64_t count, pkv_trainer* out);
void pkv_trainer_destroy(pkv_trainer t);
/* params = parameter values (the gradient's length), total = params + BN buffers */
pkv_status pkv_trainer_param_count(pkv_trainer t, int64_t* params, int64_t* total);
/* training forward_pair: x fp32 [B, H_s, n] (n <= crop_len) -> logits fp32
 * [B, H_l, n]; keeps the activations for pkv_trainer_backward and updates the
 * BN running statistics (ValueError "exceeds crop_len", "needs B*N >= 2"). */
pkv_status pkv_trainer_forward(pkv_trainer t, const float* x_dev, int64_t B, int64_t n, float* logits_dev,
                               void* stream);
/* d loss / d logits (fp64 [B, H_l, n], e.g. pkv_loss_total's grad_dev) of the
 * last forward -> grad_dev[params] += d loss / d parameters (fp64,
 * named_parameters order). */
pkv_status pkv_trainer_backward(pkv_trainer t, const double* dlogits_dev, double* grad_dev, void* stream);
/* host fp64 forms of forward / backward (synchronous; grad_host += d loss / d params) */
pkv_status pkv_trainer_forward_host(pkv_trainer t, const double* x_host, int64_t B, int64_t n, double* logits_host);
pkv_status pkv_trainer_backward_host(pkv_trainer t, const double* dlogits_host, double* grad_host);
/* the current blob (parameters + BN running statistics), host fp64 [total] */
pkv_status pkv_trainer_blob(pkv_trainer t, double* blob_host);

/* --------------------------------------------------- compaction (a-4) ---- */
/* Packed KV gather in apply_mask order (no reference code; the reference only
 * reports indices, pruning.cpp:197-215): for s < slices, j < k,
 *   k_out[s, j, :] = k_in[s, idx_asc[s, j], :]   (same for V)
 * rows of d elements of elem_bytes (2 for bf16/fp16). 128-bit vectorised. */
pkv_status pkv_compact_kv(pkv_ctx ctx, const void* k_in_dev, const void* v_in_dev, const int32_t* idx_asc_dev,
                          int64_t slices, int64_t n, int64_t k, int64_t d, int64_t elem_bytes, void* k_out_dev,
                          void* v_out_dev, void* stream);

/* Select + compaction in one call (topk_indices / apply_mask,
 * pruning.cpp:20-56,197-215, followed by the packed gather above): writes the
 * ascending retained indices idx_asc [slices, k] and the packed K/V exactly as
 * pkv_topk_select then pkv_compact_kv (the two kernels, stream-ordered). */
pkv_status pkv_select_compact(pkv_ctx ctx, const float* scores_dev, int64_t slices, int64_t n, int64_t k,
                              const void* k_in_dev, const void* v_in_dev, int64_t d, int64_t elem_bytes,
                              int32_t* idx_asc_dev, void* k_out_dev, void* v_out_dev, void* stream);

/* The same gather into a paged cache: row j of slice
 * s goes to page block_table[s * max_blocks + j / page_size], row
 * j % page_size, of the pools k_pool / v_pool [pages, page_size, d]. */
pkv_status pkv_compact_kv_paged(pkv_ctx ctx, const void* k_in_dev, const void* v_in_dev, const int32_t* idx_asc_dev,
                                int64_t slices, int64_t n, int64_t k, int64_t d, int64_t elem_bytes,
                                const int32_t* block_table_dev, int64_t max_blocks, int64_t page_size,
                                void* k_pool_dev, void* v_pool_dev, void* stream);

/* ------------------------------------------------------ scoring (a-1) ---- */
#define PKV_SCORE_REDUCE_MAX 0u /* north star: max over queries (and GQA group) */
#define PKV_SCORE_REDUCE_SUM 1u /* SPEC.md:423-431 accumulate_attention / PAPER.md:46 */
#define PKV_SCORE_CAUSAL 2u     /* mask keys j > q + (Nk - Nq) */

/* Proxy reconstruction-importance scoring (SPEC.md:423-431 accumulate_attention,
 * without materialising attn[B,H,Nq,Nk]):
 *   P[l,h,q,:] = softmax(Q[l,h,q]·K[l,h/g,:]^T / sqrt(d)),  g = Hq / Hkv
 *   X[l,kh,j]  = max (or sum) over h in group kh and q of P[l,h,q,j]
 * q_dev bf16 [L, Hq, Nq, d], k_dev bf16 [L, Hkv, Nk, d], x_out fp32 [L, Hkv, Nk].
 * lse_dev (nullable) fp32 [L, Hq, Nq]: natural-log row LSE of the scaled
 * scores, e.g. from the proxy's own prefill; when NULL a first tensor-core
 * pass computes it. d must be 64 or 128. */
pkv_status pkv_score(pkv_ctx ctx, const void* q_dev, const void* k_dev, int64_t L, int64_t Hq, int64_t Hkv,
                     int64_t Nq, int64_t Nk, int64_t d, uint32_t flags, const float* lse_dev, float* x_out_dev,
                     void* stream);

/* Pass 1 alone: lse_out fp32 [L, Hq, Nq]. */
pkv_status pkv_score_lse(pkv_ctx ctx, const void* q_dev, const void* k_dev, int64_t L, int64_t Hq, int64_t Hkv,
                         int64_t Nq, int64_t Nk, int64_t d, uint32_t flags, float* lse_out_dev, void* stream);

/* Proxy prefill attention that also emits the row LSE (
 * the scores are a by-product of the proxy's own prefill):
 *   o_out[l,h,q,:] = softmax(Q·K^T/sqrt(d)) · V   (bf16, nullable)
 *   lse_out[l,h,q] = log sum_j exp(Q·K_j/sqrt(d))  (fp32, nullable)
 * q bf16 [L, Hq, Nq, d], k/v bf16 [L, Hkv, Nk, d]; flags: PKV_SCORE_CAUSAL.
 * Passing lse_out to pkv_score(..., lse_dev = lse_out, ...) makes scoring a
 * single tensor-core pass. d must be 64 or 128. */
pkv_status pkv_proxy_prefill_attention(pkv_ctx ctx, const void* q_dev, const void* k_dev, const void* v_dev,
                                       int64_t L, int64_t Hq, int64_t Hkv, int64_t Nq, int64_t Nk, int64_t d,
                                       uint32_t flags, void* o_out_dev, float* lse_out_dev, void* stream);

/* ------------------------------------------------------- mapper (a-2) ---- */
/* geom5 = {target_layers, target_heads, proxy_layers, proxy_heads, head_dim}
 *   (ModelGeometry, proj/include/proxykv/mapper.hpp:16-25)
 * cfg12 = {d_time, encoder_layers, encoder_heads, ffn_mult, d_head, crop_len,
 *          stride, synthetic_heads, stage_conv, stage_encoder, stage_cross,
 *          normalize_input}   stage_*: 0 active, 1 bypass
 *   (MapperConfig, mapper.hpp:35-55) */

/* Replaces layer_pair, proj/src/mapper.cpp:44-49 (mapper.hpp:58). */
pkv_status pkv_layer_pair(int64_t target_layer, const int64_t* geom5, int64_t* proxy_layer_out);
/* Replaces window_offsets, proj/src/mapper.cpp:66-79 (mapper.hpp:65). */
pkv_status pkv_window_offsets(int64_t n, int64_t crop, int64_t stride, int64_t* out, int64_t cap,
                              int64_t* count_out);
/* Replaces MapperParams::init, proj/src/mapper.cpp:97-164 (mapper.hpp:94):
 * the reference initialisation as a flat fp64 blob in named_parameters() then
 * named_buffers() order (mapper.cpp:166-225). blob_out may be NULL to query
 * the count. */
pkv_status pkv_mapper_init_params(const int64_t* geom5, const int64_t* cfg12, uint64_t seed, double* blob_out,
                                  int64_t* count_out);

#define PKV_MAPPER_FP16 1u   /* fp16 operands, fp32 accumulate (1 MMA per product) */
#define PKV_MAPPER_FP16X2 2u /* activations split hi+lo fp16 (2 MMAs per product) */
#define PKV_MAPPER_FP16X3 3u /* activations and weights split (3 MMAs per product) */
#define PKV_MAPPER_FP16W2 4u /* weights split hi+lo fp16, activations fp16 (2 MMAs per product) */
#define PKV_MAPPER_FP16X3F 5u /* FP16X3 except the FFN down-projection, whose GELU input is one fp16
                                 plane (2 MMAs there; its hidden activations are half the bytes) */
#define PKV_MAPPER_FP16F8 6u /* FP16X3's two correction products as e4m3 MMAs (kind::f8f6f4, half the tensor
                                time each) in the same accumulator, for the conv2 / QKV / FFN1 / FFN2 GEMMs
                                (Wo and stage 3 stay FP16X3): 2 MMA-equivalents per product */

/* Uploads a mapper (weights in the pkv_mapper_init_params layout, fp64) to the
 * device; prepares the B200 weight layouts (K-major fp16 planes, BN folded,
 * stage-3 query/out projections folded). */
pkv_status pkv_mapper_create(pkv_ctx ctx, const int64_t* geom5, const int64_t* cfg12, const double* blob,
                             int64_t count, uint32_t precision, pkv_mapper* out);
void pkv_mapper_destroy(pkv_mapper m);

/* Replaces forward_full, proj/src/mapper.cpp:379-398 (mapper.hpp:126), eval
 * mode: x_all fp32 [B, L_s, H_s, N] -> y_all fp32 [B, L_l, H_l, N] (raw
 * logits). Includes sliding_forward's window overlap average
 * (mapper.cpp:344-377); shared proxy layers are computed once. */
pkv_status pkv_mapper_forward_full(pkv_mapper m, const float* x_all_dev, int64_t B, int64_t N, float* y_all_dev,
                                   void* stream);
/* Replaces sliding_forward (mapper.cpp:344-377; forward_pair when N <= crop):
 * x fp32 [B, H_s, N] -> y fp32 [B, H_l, N]. */
pkv_status pkv_mapper_sliding_forward(pkv_mapper m, const float* x_dev, int64_t B, int64_t N, float* y_dev,
                                      void* stream);
/* Replaces forward_pair, proj/src/mapper.cpp:274-342 (mapper.hpp:118-119),
 * eval mode: x fp32 [B, H_s, n] -> y fp32 [B, H_l, n], n <= crop_len
 * (PKV_EVALUE "... long inputs go through sliding_forward" otherwise, as
 * mapper.cpp:281-282). attn_dev (nullable) receives the StageTrace capture,
 * the Stage-3 attention fp32 [B, n, H_l, H_syn] (mapper.hpp:111-114; left
 * untouched when stage_cross is bypassed, where the reference records none). */
pkv_status pkv_mapper_forward_pair(pkv_mapper m, const float* x_dev, int64_t B, int64_t n, float* y_dev,
                                   float* attn_dev, void* stream);

/* Host-tensor forms of the three (the reference's own calling convention:
 * fp64 row-major host buffers in and out; the device computes in the
 * precision mode the mapper was created with, from the fp32 rounding of x).
 * Synchronous. attn_host as above (nullable). */
pkv_status pkv_mapper_forward_pair_host(pkv_mapper m, const double* x_host, int64_t B, int64_t n, double* y_host,
                                        double* attn_host);
pkv_status pkv_mapper_sliding_forward_host(pkv_mapper m, const double* x_host, int64_t B, int64_t N,
                                           double* y_host);
pkv_status pkv_mapper_forward_full_host(pkv_mapper m, const double* x_all_host, int64_t B, int64_t N,
                                        double* y_all_host);

/* ------------------------------------------------- whole path (a-1..a-4) -- */
/* A pruner owns the workspaces for one context shape:
 *   proxy: L_s layers, Hq query heads, H_s KV heads, head dim dp
 *   target: L_l layers, H_l KV heads, head dim dt; context N; ratio rho. */
pkv_status pkv_pruner_create(pkv_ctx ctx, pkv_mapper m, int64_t Hq, int64_t dp, int64_t dt, int64_t N, double rho,
                             uint32_t score_flags, pkv_pruner* out);
void pkv_pruner_destroy(pkv_pruner p);
/* K = retention_count(rho, N) for this pruner. */
int64_t pkv_pruner_k(pkv_pruner p);
/* score -> map -> select -> compact, device buffers:
 *   q bf16 [L_s, Hq, N, dp], kp bf16 [L_s, H_s, N, dp] (proxy),
 *   kt, vt bf16/fp16 [L_l, H_l, N, dt] (target KV),
 *   k_out, v_out [L_l, H_l, K, dt], idx_out int32 [L_l, H_l, K] (nullable),
 *   scores_out fp32 [L_l, H_l, N] (nullable: mapped scores Ŷ). */
/* Stage profiling of the next `runs` device-resident single-stream runs (pkv_pruner_run):
 * CUDA events on the launching stream at the stage boundaries; pkv_pruner_profile_read
 * synchronises and returns, per profiled run, the ms of {LSE pass, pooled pass, map,
 * select, compaction} (ms_out [runs][5]). No reference counterpart (measurement). */
pkv_status pkv_pruner_profile(pkv_pruner p, int64_t runs);
pkv_status pkv_pruner_profile_read(pkv_pruner p, double* ms_out, int64_t cap_runs, int64_t* runs_out);
pkv_status pkv_pruner_run(pkv_pruner p, const void* q_dev, const void* kp_dev, const void* kt_dev,
                          const void* vt_dev, void* k_out_dev, void* v_out_dev, int32_t* idx_out_dev,
                          float* scores_out_dev, void* stream);
/* The paper regime: the row LSE comes from
 * the proxy's own prefill attention (pkv_proxy_prefill_attention, natural
 * log, fp32 [L_s, Hq, N], with the pruner's causal flag), so scoring is the
 * pooled pass alone. Otherwise as pkv_pruner_run. */
pkv_status pkv_pruner_run_lse(pkv_pruner p, const void* q_dev, const void* kp_dev, const float* lse_dev,
                              const void* kt_dev, const void* vt_dev, void* k_out_dev, void* v_out_dev,
                              int32_t* idx_out_dev, float* scores_out_dev, void* stream);
/* Same with host buffers: H2D of the inputs and D2H of the outputs are part
 * of the call (the reference-facing end-to-end form). The copies run on the
 * pruner's own copy stream, overlapped with compute: the proxy Q/K one proxy
 * layer at a time (each layer's scoring starts when it lands), then the
 * target KV (consumed only by select + compaction); the map -> select ->
 * compact tail runs per group of target layers, each group's outputs copied
 * back while the next group is mapped. Pinned host memory makes the copies
 * asynchronous. */
pkv_status pkv_pruner_run_host(pkv_pruner p, const void* q_host, const void* kp_host, const void* kt_host,
                               const void* vt_host, void* k_out_host, void* v_out_host, int32_t* idx_out_host,
                               void* stream);
/* Dual-stream form (the proxy runs asynchronously to the target
 * prefill): scoring + mapping (and, sharded by head, the score exchange) are
 * enqueued on proxy_stream; select + compaction on target_stream, gated by an
 * event recorded on proxy_stream. Arguments as pkv_pruner_run. */
pkv_status pkv_pruner_run_dual(pkv_pruner p, const void* q_dev, const void* kp_dev, const void* kt_dev,
                               const void* vt_dev, void* k_out_dev, void* v_out_dev, int32_t* idx_out_dev,
                               float* scores_out_dev, void* proxy_stream, void* target_stream);

/* Two-device proxy -> target: the pruner's
 * context device scores and maps (q, kp on it; proxy_stream there); the mapped
 * scores cross with one peer copy; select + compaction run on target_ctx's
 * device on target_stream (kt/vt/outputs live there), gated by an event.
 * scores_target_dev (nullable) receives Ŷ on the target device. Unsharded
 * pruners only. Outputs are identical to pkv_pruner_run's. */
pkv_status pkv_pruner_run_two_device(pkv_pruner p, pkv_ctx target_ctx, const void* q_dev, const void* kp_dev,
                                     const void* kt_target_dev, const void* vt_target_dev, void* k_out_target_dev,
                                     void* v_out_target_dev, int32_t* idx_out_target_dev, float* scores_target_dev,
                                     void* proxy_stream, void* target_stream);

/* Target-side consumption of the packed cache: one
 * decode query per query head over its KV head's retained rows,
 *   out[l,h,:] = softmax(q[l,h]·K_packed[l,h/g]^T · scale) · V_packed[l,h/g]
 * q bf16 [L, Hq, d] (L: layers or independent sequences), k/v_packed bf16
 * [L, Hkv, K, d] as written by pkv_compact_kv / pkv_pruner_run, out fp32
 * [L, Hq, d]. Split-K flash decoding, HBM-bound; GQA groups 1/2/4/8, d 64/128. */
pkv_status pkv_packed_decode_attention(pkv_ctx ctx, const void* q_dev, const void* k_packed_dev,
                                       const void* v_packed_dev, int64_t L, int64_t Hq, int64_t Hkv, int64_t K,
                                       int64_t d, double scale, float* out_dev, void* stream);

/* Decode over a paged pruned cache with per-(layer, KV head) lengths: slab
 * s = l * Hkv + kh holds seq_lens[s] rows, row r in page
 * block_table[s * max_blocks + r / page_size] at row r % page_size of the
 * bf16 pools [pages, page_size, d]; max_len >= every seq_lens[s] sizes the
 * split-K grid. A slab of length 0 decodes to 0. Same kernel as the packed
 * form with the row address taken through the block table. */
pkv_status pkv_paged_decode_attention(pkv_ctx ctx, const void* q_dev, const void* k_pool_dev, const void* v_pool_dev,
                                      const int32_t* block_table_dev, const int32_t* seq_lens_dev, int64_t L,
                                      int64_t Hq, int64_t Hkv, int64_t max_blocks, int64_t page_size, int64_t max_len,
                                      int64_t d, double scale, float* out_dev, void* stream);

/* ------------------------------------------- file formats -- */
/* Host-only. Little-endian, binio.hpp semantics; corrupt files return the
 * PKV_EIO_* code of the reference's IoError taxonomy (common.hpp:33-52).
 * PKVT trace: geom6 = {L_s, H_s, L_l, H_l, N, B};
 * per sample X fp32 [B, L_s, H_s, N] then Y fp32 [B, L_l, H_l, N]; meta is a
 * free one-line string (nullable). read(write(t)) is bit-exact. */
pkv_status pkv_trace_write(const char* path, const int64_t* geom6, int64_t samples, const float* x, const float* y,
                           const char* meta);
pkv_status pkv_trace_read_header(const char* path, int64_t* geom6_out, int64_t* samples_out);
/* x_out / y_out hold samples * [B, L, H, N] floats (sizes from the header). */
pkv_status pkv_trace_read(const char* path, float* x_out, float* y_out);
/* Mapper checkpoint: geometry, config, tensor directory and the
 * fp64 parameter blob in the pkv_mapper_init_params / pkv_mapper_create
 * layout. blob_out may be NULL to query count_out. */
pkv_status pkv_checkpoint_write(const char* path, const int64_t* geom5, const int64_t* cfg12, const double* blob,
                                int64_t count);
pkv_status pkv_checkpoint_read(const char* path, int64_t* geom5_out, int64_t* cfg12_out, double* blob_out,
                               int64_t* count_out);

/* ------------------------------------------------ multi-GPU -- */
/* One context pruned by `world` ranks (one process per GPU). No reference
 * code: the reference is single-threaded CPU; BASELINE.json configs[2,3].
 *   PKV_SHARD_LAYER: rank owns a contiguous block of target layers (all KV
 *     heads) and scores + maps the proxy layers they pair with (layer_pair is
 *     monotone, mapper.cpp:44-49): no collective.
 *   PKV_SHARD_HEAD: rank owns a contiguous group of target KV heads (all
 *     layers); proxy layers are split across ranks and the mapped scores are
 *     exchanged with one NCCL all-to-all (needs a pkv_comm).
 * Per-slice results are bit-identical to the 1-GPU path. */
#define PKV_SHARD_LAYER 0u
#define PKV_SHARD_HEAD 1u
#define PKV_COMM_ID_BYTES 128

typedef struct pkv_comm_s* pkv_comm;

/* The plan for (world, rank), host logic only: out8 = {t_lo, t_hi, h_lo,
 * h_hi, p_lo, p_hi, a, b} (0-based, half-open): the rank selects and compacts
 * target slices [t_lo, t_hi) x heads [h_lo, h_hi), scores and maps proxy
 * layers [p_lo, p_hi), and produces mapped scores of target layers [a, b). */
pkv_status pkv_shard_plan(const int64_t* geom5, int world, int rank, uint32_t mode, int64_t* out8);
/* NCCL communicator (libnccl.so.2 is loaded at first use): rank 0 creates the
 * id, the caller distributes it (e.g. over torch.distributed / MPI). */
pkv_status pkv_comm_unique_id(uint8_t* id_out /* PKV_COMM_ID_BYTES */);
pkv_status pkv_comm_create(pkv_ctx ctx, int world, int rank, const uint8_t* id, pkv_comm* out);
void pkv_comm_destroy(pkv_comm c);
/* A pruner for this rank's shard. comm may be NULL for PKV_SHARD_LAYER.
 * Buffers passed to run / run_dual are then shard-local: q, kp the full proxy
 * tensors (only layers [p_lo, p_hi) are read); kt, vt [t_hi-t_lo, h_hi-h_lo,
 * N, dt]; k_out, v_out [.., .., K, dt]; idx_out [.., .., K]; scores_out
 * [t_hi-t_lo, h_hi-h_lo, N]. */
pkv_status pkv_pruner_create_sharded(pkv_ctx ctx, pkv_mapper m, int64_t Hq, int64_t dp, int64_t dt, int64_t N,
                                     double rho, uint32_t score_flags, uint32_t shard_mode, int world, int rank,
                                     pkv_comm comm, pkv_pruner* out);

/* The head-group exchange as a list of point-to-point operations (host logic
 * only; the NCCL exchange inside a PKV_SHARD_HEAD pruner issues exactly these,
 * in this order, inside one ncclGroupStart/End). Each op is 5 int64:
 *   {kind (0 send, 1 recv), peer rank, element offset, element count, tag}
 * sends read y_local [b-a, H_l, N] (this rank's mapped target layers, all
 * heads), recvs write y_recv [L_l, h_hi-h_lo, N] (every target layer, this
 * rank's heads); tag = the target layer, so (peer, tag) matches a send with
 * its recv. count_out = number of ops (all of them, even past cap). */
pkv_status pkv_shard_exchange_schedule(const int64_t* geom5, int world, int rank, int64_t N, int64_t* ops_out,
                                       int64_t cap, int64_t* count_out);
/* Runs a head-group pruner's exchange alone on `stream` (y_local / y_recv as
 * above): the step pkv_pruner_run performs between mapping and select. */
pkv_status pkv_pruner_exchange(pkv_pruner p, const float* y_local_dev, float* y_recv_dev, void* stream);

#ifdef __cplusplus
}
#endif

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#endif /* PKV_CAPI_H */
