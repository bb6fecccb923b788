// lse_chunk.cuh — the fixed-reference softmax row-sum step of scoring pass 1
// (score.cu score_lse_kernel), shared with its microbenchmark
// (tools/probe_lse_chunk.cu, which runs it from registers at the kernel's
// warp count to measure the instruction mix's own ceiling).
#pragma once

#include "sm100.cuh"

namespace pkv {

// The pass-1 scale c = log2(e)/√d as a compile-time constant (bit-identical to
// the host's kLog2e / sqrtf(d)), so the FFMA2s take it as an immediate.
template <int D>
__device__ __forceinline__ constexpr float lse_scale() {
    return D == 64 ? 0x1.715476p-3f : 0x1.0527dcp-3f;
}

template <int kPolyPairs, int D>
__device__ __forceinline__ float lse_chunk_fixed(const uint32_t (&ra)[32], const uint32_t (&rb)[32], int valid,
                                                 float nm, float mp) {
    constexpr float c = lse_scale<D>();
    using namespace sm100;
    const bool masked = __any_sync(0xffffffffu, valid < 64);
    uint64_t acc0 = pack2(0.0f, 0.0f), acc1 = acc0;
    if (!masked) {
#pragma unroll
        for (int pr = 0; pr < 32; ++pr) {
            const uint64_t s2 = pr < 16 ? pack2(__uint_as_float(ra[2 * pr]), __uint_as_float(ra[2 * pr + 1]))
                                        : pack2(__uint_as_float(rb[2 * pr - 32]), __uint_as_float(rb[2 * pr - 31]));
            uint64_t e;
            if (((pr + 1) * kPolyPairs) / 32 != (pr * kPolyPairs) / 32) {
                e = ex2_poly2_fused_s(s2, c, mp);
            } else {
                const float2 x = unpack2(ffma2_ss(s2, c, nm));
                e = pack2(ex2(x.x), ex2(x.y));
            }
            if (pr & 1) acc1 = fadd2(acc1, e);
            else acc0 = fadd2(acc0, e);
        }
    } else {
#pragma unroll
        for (int pr = 0; pr < 32; ++pr) {
            float a = pr < 16 ? __uint_as_float(ra[2 * pr]) : __uint_as_float(rb[2 * pr - 32]);
            float b = pr < 16 ? __uint_as_float(ra[2 * pr + 1]) : __uint_as_float(rb[2 * pr - 31]);
            a = 2 * pr < valid ? a : -INFINITY;
            b = 2 * pr + 1 < valid ? b : -INFINITY;
            const float2 x = unpack2(ffma2_ss(pack2(a, b), c, nm));
            const uint64_t e = pack2(ex2(x.x), ex2(x.y));
            if (pr & 1) acc1 = fadd2(acc1, e);
            else acc0 = fadd2(acc0, e);
        }
    }
    const float2 ssum = unpack2(fadd2(acc0, acc1));
    return ssum.x + ssum.y;
}

}  // namespace pkv
