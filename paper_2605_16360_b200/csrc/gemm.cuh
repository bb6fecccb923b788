// gemm.cuh — persistent warp-specialised tcgen05 GEMM for the mapper's dense
// contractions (conv2 as implicit GEMM over an im2col panel, QKV / Wo / FFN
// projections, stage-3 folded projection):
//
//   C[M, N] = Σ_planes A_p[M, K] · B_q[N, K]^T   (+ fused epilogue)
//
// A and B are K-major fp16 planes loaded by TMA with 128-byte swizzle into a
// multi-stage smem ring; one elected thread issues tcgen05.mma (M=128, N=BN,
// K=16 per instruction) into a double-buffered TMEM accumulator; four
// epilogue warps drain TMEM with tcgen05.ld while the next tile's MMAs run.
//
// Precision planes (DESIGN.md §Mapper precision): NA=2 splits the activation
// into hi+lo fp16 (x = hi + lo), NB=2 splits the weights the same way; the
// MMAs A0·B0 (+ A1·B0) (+ A0·B1) accumulate into one fp32 TMEM accumulator.
// FP16F8 (mode 6, `f8`): the two corrections are e4m3 MMAs (kind::f8f6f4, half
// the tensor time of an fp16 MMA) into the SAME accumulator: with the operand
// class constants below, main = A_hi·W'_hi (fp16), corr = e4m3(A_lo·lo_mul) ·
// e4m3(W'_hi / lo_mul) + e4m3(A_hi·hi_mul) · e4m3(W'_lo / hi_mul), all in units
// of A·W' where W' = W·2^w (exact power of two, undone by acc_scale).
#pragma once

#include "internal.h"
#include "sm100.cuh"

namespace pkv {

enum GemmEpi : int {
    EPI_F32 = 0,         // out_f32 = acc + bias
    EPI_F16X = 1,        // out planes = split(acc + bias)            (QKV)
    EPI_GELU_F16X = 2,   // out planes = split(gelu(acc + bias))      (FFN1)
    EPI_RESID = 3,       // resid += acc + bias                       (Wo, FFN2)
    EPI_GELU_PE = 4,     // out_f32 = gelu(acc + bias) + pe[row % lw] (conv2 + BN folded + PE)
};

// Row scaling (EPI_F32 / EPI_GELU_PE): when row_scale is set, acc is first
// multiplied by row_scale[row]. The A-operand producers (conv1_im2col, the
// stage-3 row split) store each row pre-scaled by an exact power of two so its
// largest magnitude sits in [2^13, 2^14) — inside the fp16 range whatever the
// input scale (sum-pooled X reaches g·N_q) — and record the
// inverse power of two here; the product is then exact algebra.

// FP16F8 operand classes: a bound on |A| fixes the e4m3 multipliers so every
// e4m3 value stays <= 448 (satfinite beyond: the correction of that element
// degrades, nothing overflows) and W' = W·2^w has max |W'| in [2^(w_top-1), 2^w_top).
struct F8Class {
    float lo_mul, hi_mul;  // A_lo8 = e4m3((A − A_hi)·lo_mul), A_hi8 = e4m3(A_hi·hi_mul)
    int w_top;
};
// |A| < 2^9: LayerNorm and GELU outputs
constexpr F8Class kF8Act{1024.0f, 0.5f, 15};
// rows pre-scaled so max |row| is in [2^13, 2^14) (conv2's im2col panel, §6)
constexpr F8Class kF8Row{32.0f, 1.0f / 64.0f, 13};

struct GemmEpiParams {
    float* out_f32 = nullptr;  // EPI_F32 / EPI_GELU_PE; resid for EPI_RESID
    __half* out_h = nullptr;   // hi plane
    __half* out_l = nullptr;   // lo plane (nullptr = single plane)
    const float* bias = nullptr;
    const float* pe = nullptr;  // [lw, ldo] fp32
    const float* row_scale = nullptr;  // [M] power-of-two multipliers (see above)
    int64_t ldo = 0;            // output row stride (elements)
    int64_t lw = 1;             // rows per window (PE period)
    float acc_scale = 1.0f;     // the accumulator is multiplied by this first (FP16F8: 2^-w)
    // EPI_F16X / EPI_GELU_F16X for an FP16F8 consumer: e4m3 correction planes
    // [rows, ldo] instead of the fp16 lo plane (out_l unused)
    uint8_t* out_l8 = nullptr;  // e4m3((v − hi)·l8_mul)
    uint8_t* out_h8 = nullptr;  // e4m3(hi·h8_mul)
    float l8_mul = 1.0f, h8_mul = 1.0f;
};

struct GemmArgs {
    CUtensorMap a[2];
    CUtensorMap b[2];
    int na = 1, nb = 1;
    int64_t M = 0, N = 0, K = 0;
    int bn = 256;
    GemmEpi epi = EPI_F32;
    GemmEpiParams p;
    // raw operands (the 2-CTA path re-encodes B with 128-row boxes)
    const __half* b_ptr[2] = {nullptr, nullptr};
    int64_t ldb = 0;
    bool pair = false;  // use the CTA-pair (cta_group::2, 256x256 tile) kernel
    // FP16F8: a[1] / a8h = A's e4m3 lo / hi planes, b8[0] / b8[1] = W's e4m3 hi / lo planes (pair kernel only)
    bool f8 = false;
    CUtensorMap a8h;
    const uint8_t* b8[2] = {nullptr, nullptr};
};

// Builds the TMA maps for fp16 K-major planes: A rows of length K (row stride
// lda elements), B [N, K] (row stride ldb).
void gemm_set_a(GemmArgs& g, int plane, const __half* a, int64_t M, int64_t K, int64_t lda);
void gemm_set_b(GemmArgs& g, int plane, const __half* b, int64_t N, int64_t K, int64_t ldb);
// FP16F8: A's e4m3 planes (K-major bytes, row stride lda) and W's (hi8, lo8) [N, K]
void gemm_set_a8(GemmArgs& g, const uint8_t* lo8, const uint8_t* hi8, int64_t M, int64_t K, int64_t lda);
void gemm_set_b8(GemmArgs& g, const uint8_t* hi8, const uint8_t* lo8);
void gemm_run(const GemmArgs& g, int sm_count, cudaStream_t st);

}  // namespace pkv
