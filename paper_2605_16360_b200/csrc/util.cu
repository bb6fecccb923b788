// util.cu — small elementwise kernels: fp32 -> fp16 hi/lo planes and back.
#include "util.cuh"

namespace pkv {
namespace {

__global__ void split_kernel(const float* __restrict__ x, int64_t n, __half* __restrict__ hi, __half* __restrict__ lo) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float v = x[i];
        const __half h = __float2half_rn(v);
        hi[i] = h;
        if (lo) lo[i] = __float2half_rn(v - __half2float(h));
    }
}

__global__ void combine_kernel(const __half* __restrict__ hi, const __half* __restrict__ lo, int64_t n,
                               float* __restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        out[i] = __half2float(hi[i]) + (lo ? __half2float(lo[i]) : 0.0f);
    }
}

}  // namespace

void launch_split_f16(const float* x, int64_t n, __half* hi, __half* lo, cudaStream_t st) {
    if (n == 0) return;
    const int64_t blocks = (n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096;
    split_kernel<<<(unsigned)blocks, 256, 0, st>>>(x, n, hi, lo);
    check_launch("split_kernel");
}

void launch_combine_f16(const __half* hi, const __half* lo, int64_t n, float* out, cudaStream_t st) {
    if (n == 0) return;
    const int64_t blocks = (n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096;
    combine_kernel<<<(unsigned)blocks, 256, 0, st>>>(hi, lo, n, out);
    check_launch("combine_kernel");
}

}  // namespace pkv
