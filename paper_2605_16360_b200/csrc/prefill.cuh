// prefill.cuh — proxy prefill self-attention with LSE output (prefill.cu).
#pragma once
#include "score.cuh"

namespace pkv {

// O bf16 [L, Hq, Nq, d] (nullable), lse fp32 [L, Hq, Nq] natural log (nullable).
void launch_prefill_attention(const ScoreShape& s, const void* q, const void* k, const void* v, void* o, float* lse,
                              cudaStream_t st);

}  // namespace pkv
