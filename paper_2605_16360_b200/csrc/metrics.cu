// metrics.cu — the ranking metrics of the reference on the device (SURVEY.md
// §8(f) item 4; proj/src/pruning.cpp:58-117): per-slice Top-K overlap of two
// masks and the captured-mass ratio of a predicted mask against the scores'
// own Top-K. One CTA per slice, fp64 sums (the reference accumulates in fp64;
// only the summation order differs).
#include "internal.h"

namespace pkv {
namespace {

constexpr int kThreads = 512;

__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) red[w] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x < 32) {
        t = threadIdx.x < kThreads / 32 ? red[threadIdx.x] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    }
    __syncthreads();
    return t;  // valid in thread 0
}

// topk_overlap_per_slice (pruning.cpp:91-108): |a ∩ b| / k
__global__ void __launch_bounds__(kThreads) overlap_kernel(const uint8_t* __restrict__ a,
                                                           const uint8_t* __restrict__ b, int64_t n, int64_t k,
                                                           double* __restrict__ out) {
    __shared__ double red[kThreads / 32];
    const int64_t s = blockIdx.x;
    double c = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += kThreads) c += (a[s * n + i] && b[s * n + i]) ? 1.0 : 0.0;
    const double t = block_sum(c, red);
    if (threadIdx.x == 0) out[s] = t / (double)k;
}

// captured_mass_per_slice (pruning.cpp:58-80): Σ_pred y / Σ_topk(y) y (1 if 0)
__global__ void __launch_bounds__(kThreads) mass_kernel(const uint8_t* __restrict__ pred,
                                                        const uint8_t* __restrict__ oracle,
                                                        const float* __restrict__ y, int64_t n,
                                                        double* __restrict__ out) {
    __shared__ double red[kThreads / 32];
    const int64_t s = blockIdx.x;
    double cap = 0.0, orc = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += kThreads) {
        const double v = (double)y[s * n + i];
        cap += pred[s * n + i] ? v : 0.0;
        orc += oracle[s * n + i] ? v : 0.0;
    }
    const double tc = block_sum(cap, red);
    const double to = block_sum(orc, red);
    if (threadIdx.x == 0) out[s] = to > 0.0 ? tc / to : 1.0;
}

}  // namespace
}  // namespace pkv

using namespace pkv;

extern "C" {

pkv_status pkv_topk_overlap(pkv_ctx ctx, const uint8_t* mask_a_dev, const uint8_t* mask_b_dev, int64_t slices,
                            int64_t n, int64_t k, double* per_slice_out_dev, void* stream) {
    return guard([&] {
        require_ctx(ctx);
        PKV_REQUIRE_SHAPE(slices > 0 && n > 0, "topk_overlap extents must be positive");
        PKV_REQUIRE_VALUE(k >= 1 && k <= n, "k must be in [1, n], got ", k);
        overlap_kernel<<<(unsigned)slices, kThreads, 0, static_cast<cudaStream_t>(stream)>>>(mask_a_dev, mask_b_dev, n,
                                                                                            k, per_slice_out_dev);
        check_launch("overlap_kernel");
        count_launch(ctx);
    });
}

pkv_status pkv_captured_mass(pkv_ctx ctx, const uint8_t* mask_pred_dev, const float* y_dev, int64_t slices,
                             int64_t n, int64_t k, double* per_slice_out_dev, void* stream) {
    return guard([&] {
        require_ctx(ctx);
        PKV_REQUIRE_SHAPE(slices > 0 && n > 0, "captured_mass extents must be positive");
        PKV_REQUIRE_VALUE(k >= 1 && k <= n, "k must be in [1, n], got ", k);
        auto st = static_cast<cudaStream_t>(stream);
        auto* om = static_cast<uint8_t*>(ctx->scratch_select.get(static_cast<size_t>(slices * n)));
        launch_topk_select(y_dev, slices, n, k, om, nullptr, st);  // the oracle mask: y's own Top-K
        mass_kernel<<<(unsigned)slices, kThreads, 0, st>>>(mask_pred_dev, om, y_dev, n, per_slice_out_dev);
        check_launch("mass_kernel");
        count_launch(ctx, 2);
    });
}

}  // extern "C"
