#pragma once
#include <cuda_bf16.h>

#include "internal.h"

namespace pkv {

struct ScoreShape {
    int64_t L = 0, Hq = 0, Hkv = 0, Nq = 0, Nk = 0, d = 0;
    bool causal = false;
};

void score_validate(const ScoreShape& s);
// pass 1: lse fp32 [L, Hq, Nq] (nullable) and λ rows bf16 [L, Hq, Nq, 8] (nullable)
// aux: caller-owned scratch (per context / pruner) for the fixed-reference
// pass (max |k| per KV head + one flag per query tile); null = exact kernel only
void launch_score_lse(const ScoreShape& s, const void* q, const void* k, float* lse, __nv_bfloat16* lam,
                      cudaStream_t st, DevBuf* aux);
void launch_lam_from_lse(const float* lse, int64_t rows, int64_t d, __nv_bfloat16* lam, cudaStream_t st);
// pass 2: x fp32 [L, Hkv, Nk]
void launch_score_pool(const ScoreShape& s, const void* q, const void* k, const __nv_bfloat16* lam, bool reduce_max,
                       float* x, cudaStream_t st);

}  // namespace pkv
