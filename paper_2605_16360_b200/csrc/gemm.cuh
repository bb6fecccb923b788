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

struct GemmEpiParams {
    float* out_f32 = nullptr;  // EPI_F32 / EPI_GELU_PE; resid for EPI_RESID
    __half* out_h = nullptr;   // hi plane
    __half* out_l = nullptr;   // lo plane (nullptr = single plane)
    const float* bias = nullptr;
    const float* pe = nullptr;  // [lw, ldo] fp32
    const float* row_scale = nullptr;  // [M] power-of-two multipliers (see above)
    int64_t ldo = 0;            // output row stride (elements)
    int64_t lw = 1;             // rows per window (PE period)
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
};

// Builds the TMA maps for fp16 K-major planes: A rows of length K (row stride
// lda elements), B [N, K] (row stride ldb).
void gemm_set_a(GemmArgs& g, int plane, const __half* a, int64_t M, int64_t K, int64_t lda);
void gemm_set_b(GemmArgs& g, int plane, const __half* b, int64_t N, int64_t K, int64_t ldb);
void gemm_run(const GemmArgs& g, int sm_count, cudaStream_t st);

}  // namespace pkv
