/* pkv_oracle.h — plain-C CPU restatement of the ProxyKV pruning hot path.
 *
 * TEST INFRASTRUCTURE ONLY. This is the parity checker: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it. The
 * product (libpkv_b200.so) never links it and has no CPU fallback.
 *
 * Each function cites the reference file:line it restates
 * (paths relative to /root/reference/).
 */
#ifndef PKV_ORACLE_H
#define PKV_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* proj/src/pruning.cpp:14-18. Returns 0, or 2 (ValueError) for rho∉(0,1] or n<=0. */
int pkvo_retention_count(double rho, int64_t n, int64_t* k_out);

/* proj/src/pruning.cpp:20-56 (topk_indices + topk_mask) followed by
 * proj/src/pruning.cpp:197-215 (apply_mask): per slice of length n, the k best
 * values under better(a,b) = v[a] > v[b] || (v[a] == v[b] && a < b),
 * written as a 0/1 mask [slices, n] (nullable) and ascending indices
 * [slices, k] (nullable). Values are fp32 widened to fp64 (exact, monotone).
 * Returns 2 if k∉[1,n]. NaN inputs are rejected (3). */
int pkvo_topk_select_f32(const float* scores, int64_t slices, int64_t n, int64_t k,
                         uint8_t* mask_out, int32_t* idx_asc_out);

/* Packed KV gather (no reference code): for every slice s and
 * j < k, out[s, j, :] = in[s, idx_asc[s, j], :], for K and V, 16-bit elements. */
void pkvo_compact_kv(const uint16_t* k_in, const uint16_t* v_in, const int32_t* idx_asc,
                     int64_t slices, int64_t n, int64_t k, int64_t d, uint16_t* k_out,
                     uint16_t* v_out);

/* Proxy reconstruction-importance scoring for one KV head (SPEC.md:423-431
 * accumulate_attention; X definition; north-star max-pool).
 *   q: [group, nq, d] bf16 bits (the query heads sharing this KV head)
 *   k: [nk, d] bf16 bits
 *   P[h,q,:] = softmax_keys(q_h[q] · K^T / sqrt(d))   (fp64)
 *   reduce 0 (sum): x[j] = Σ_h Σ_q P[h,q,j]
 *   reduce 1 (max): x[j] = max_h max_q P[h,q,j]
 * causal != 0 masks keys j > q + (nk - nq). Output fp32 [nk]. */
void pkvo_score_head(const uint16_t* q, const uint16_t* k, int64_t group, int64_t nq, int64_t nk,
                     int64_t d, int reduce, int causal, float* x_out);

/* Row log-sum-exp (natural log) of the scaled scores for one query head:
 * lse[q] = log Σ_j exp(q·k_j / sqrt(d))   (fp64, returned as fp32). */
void pkvo_score_lse(const uint16_t* q, const uint16_t* k, int64_t nq, int64_t nk, int64_t d,
                    int causal, float* lse_out);

/* proj/include/proxykv/rng.hpp:11-87 (splitmix64 / derive_seed / xoshiro256**)
 * and proj/src/mapper.cpp:97-164 (MapperParams::init): writes the
 * named_parameters() then named_buffers() tensors (proj/src/mapper.cpp:166-225)
 * back to back as fp64 into blob (nullable); returns the element count.
 * geom5 = {target_layers, target_heads, proxy_layers, proxy_heads, head_dim};
 * cfg12 = {d_time, encoder_layers, encoder_heads, ffn_mult, d_head, crop_len,
 *          stride, synthetic_heads, stage_conv, stage_encoder, stage_cross,
 *          normalize_input} (stage: 0 active, 1 bypass). */
int64_t pkvo_mapper_init(const int64_t* geom5, const int64_t* cfg12, uint64_t seed, double* blob);

/* Raw xoshiro256** stream, for pinning the RNG restatement:
 * Rng(seed).uniform(lo, hi) n times (rng.hpp:56-58). */
void pkvo_rng_uniform(uint64_t seed, double lo, double hi, int64_t n, double* out);
/* Rng(seed).normal() n times (rng.hpp:72-84). */
void pkvo_rng_normal(uint64_t seed, int64_t n, double* out);
/* Rng(seed).below(bound) n times (rng.hpp:61-70). */
void pkvo_rng_below(uint64_t seed, uint64_t bound, int64_t n, uint64_t* out);

#ifdef __cplusplus
}
#endif

#endif
