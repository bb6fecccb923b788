// decode.cuh — decode attention over the packed (pruned) KV cache (decode.cu).
#pragma once
#include <algorithm>

#include "internal.h"

namespace pkv {

struct DecodeShape {
    int64_t L = 0, Hq = 0, Hkv = 0, K = 0, d = 0;
    float scale = 0.0f;
};

// q bf16 [L, Hq, d]; K/V packed bf16 [L, Hkv, K, d]; out fp32 [L, Hq, d].
void launch_packed_decode(const DecodeShape& s, const void* q, const void* kc, const void* vc, float* out, DevBuf& ws,
                          int sm_count, cudaStream_t st);

}  // namespace pkv
