// Microbenchmark: the ceiling of scoring pass 1's softmax row-sum instruction
// mix on its own — lse_chunk_fixed (paper_2605_16360_b200/csrc/lse_chunk.cuh,
// the exact code score_lse_kernel runs per 64-column chunk) from registers, no
// TMEM loads and no MMA, at the kernel's occupancy: one 576-thread CTA per SM,
// 16 softmax warps (4 per SM sub-partition) plus 2 idle warps. Prints the
// exponentials per clock per SM for each MUFU / FMA-polynomial split, to
// compare with score_lse_kernel's achieved rate (ncu: exponentials /
// (SMs x elapsed cycles)).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//          -I paper_2605_16360_b200/csrc -o tools/probe_lse_chunk tools/probe_lse_chunk.cu
#include <cstdio>

#include "lse_chunk.cuh"

template <int kPoly>
__global__ void __launch_bounds__(576, 1) probe(int iters, float* out, long long* cycles) {
    extern __shared__ uint8_t smem_pad[];  // one CTA per SM, as the kernel
    const int warp = threadIdx.x >> 5;
    if (warp < 2) return;  // producer / MMA warps: idle on barriers in the kernel
    uint32_t ra[32], rb[32];
    for (int i = 0; i < 32; ++i) {  // scores with a spread like the bench's logits
        ra[i] = __float_as_uint(-3.0f + 0.37f * ((threadIdx.x * 7 + i * 13) % 17));
        rb[i] = __float_as_uint(-5.0f + 0.41f * ((threadIdx.x * 5 + i * 11) % 19));
    }
    const float m0 = 3.0f;
    float lsum = 0.0f;
    __syncwarp();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const float m = m0 + (float)(it & 1) * 0.5f;  // varies: nothing hoisted out of the loop
        lsum += pkv::lse_chunk_fixed<kPoly, 64>(ra, rb, 64, -m, 12582912.0f - m);
    }
    const long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = lsum;
    if (threadIdx.x == 64) cycles[blockIdx.x] = t1 - t0;
}

template <int kPoly>
void run(int sms) {
    float* out;
    long long* cyc;
    cudaMalloc(&out, sms * 576 * 4);
    cudaMalloc(&cyc, sms * 8);
    const int iters = 4096;
    const int smem = 200 * 1024;
    cudaFuncSetAttribute(probe<kPoly>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    probe<kPoly><<<sms, 576, smem>>>(64, out, cyc);  // warm-up
    probe<kPoly><<<sms, 576, smem>>>(iters, out, cyc);
    cudaDeviceSynchronize();
    long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    const double exps = 16.0 * 32 * 64 * iters;  // per SM
    printf("poly pairs %2d of 32: %6.2f exponentials/clk/SM (%s)\n", kPoly, exps / c,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<6>(sms);
    run<8>(sms);
    run<10>(sms);
    run<12>(sms);
    run<14>(sms);
    run<16>(sms);
    return 0;
}
