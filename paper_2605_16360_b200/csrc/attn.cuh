#pragma once
#include <cuda_fp16.h>

#include "internal.h"

namespace pkv {
// qkv fp16 [nwin * Lw, 3 * D] -> ctx planes [nwin * Lw, ld_out] (hi, lo nullable).
void launch_encoder_attention(const __half* qkv, int64_t nwin, int64_t Lw, int64_t D, int64_t heads, __half* out_h,
                              __half* out_l, int64_t ld_out, cudaStream_t st);
}  // namespace pkv
