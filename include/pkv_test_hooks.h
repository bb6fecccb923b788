/* pkv_test_hooks.h — internal kernel entry points of libpkv_b200.so exported
 * for unit tests only (tests/test_kernels_gpu.py). Not part of the drop-in API.
 */
#ifndef PKV_TEST_HOOKS_H
#define PKV_TEST_HOOKS_H

#include "pkv_capi.h"

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* tcgen05 GEMM on fp32 inputs split into na (1|2) fp16 planes of A [M, K] and
 * nb planes of B [N, K]: out[M, N] = epi(A·B^T + bias). epi: 0 f32, 1 f16
 * planes (returned recombined as fp32), 2 gelu f16 planes, 3 residual
 * (out += ...), 4 gelu + pe[row % lw]. bn: 64 | 128 | 256. */
pkv_status pkv_test_gemm(pkv_ctx ctx, const float* a_dev, int64_t M, int64_t K, const float* b_dev, int64_t N,
                         int na, int nb, int bn, int epi, const float* bias_dev, const float* pe_dev, int64_t lw,
                         float* out_dev, void* stream);

/* Encoder self-attention (mapper.cpp:254-270) on fp32 qkv [nwin*Lw, 3*D]
 * rounded to fp16: out fp32 [nwin*Lw, D] (recombined hi+lo planes). */
pkv_status pkv_test_attention(pkv_ctx ctx, const float* qkv_dev, int64_t nwin, int64_t Lw, int64_t D, int64_t heads,
                              float* out_dev, void* stream);

/* Select path override for tests: -1 default (the streaming select for rows
 * of >= 4096 scores; PKV_SELECT_STREAM env), 0 the register-cached radix
 * kernel (select.cu), 1 the streaming kernel (select_stream.cu) at every
 * size. Returns the previous setting. */
int pkv_test_select_path(int mode);

#ifdef __cplusplus
}
#endif

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#endif
