#pragma once
#include <cuda_fp16.h>

#include "internal.h"

namespace pkv {
void launch_split_f16(const float* x, int64_t n, __half* hi, __half* lo, cudaStream_t st);
void launch_combine_f16(const __half* hi, const __half* lo, int64_t n, float* out, cudaStream_t st);
}  // namespace pkv
