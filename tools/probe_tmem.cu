// Microbenchmark: tcgen05.ld (TMEM -> registers) throughput per SM, and
// MUFU ex2 throughput, on sm_100a. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe tools/probe_tmem.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2605_16360_b200/csrc/sm100.cuh"

using namespace pkv::sm100;

template <int SHAPE>
__global__ void tmem_ld_bench(int iters, float* out, long long* cycles) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc(&slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    const uint32_t quad = warp & 3;
    const uint32_t colbase = (warp >> 2) * 64;
    float acc = 0.f;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        uint32_t r[32];
        tmem_ld32(tmem + ((quad * 32) << 16) + ((colbase + (i & 1) * 32) & 511), r);
        tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 32; ++u) acc += __uint_as_float(r[u]);
    }
    long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

__global__ void ex2_bench(int iters, float* out, long long* cycles) {
    float a[8];
    for (int j = 0; j < 8; ++j) a[j] = -0.001f * (threadIdx.x + j);
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = ex2(a[j]) - 1.0f;
    }
    long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
    float s = 0;
    for (int j = 0; j < 8; ++j) s += a[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    float* out;
    long long* cyc;
    cudaMalloc(&out, 148 * 1024 * 4);
    cudaMalloc(&cyc, 148 * 8);
    const int iters = 4096;
    for (int warps : {4, 8, 16}) {
        tmem_ld_bench<0><<<148, warps * 32>>>(iters, out, cyc);
        cudaDeviceSynchronize();
        long long c;
        cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        const double bytes = (double)warps * 32 * 32 * 4 * iters;
        printf("tcgen05.ld x32: %2d warps: %lld cycles, %.1f B/clk/SM (err=%s)\n", warps, c, bytes / c,
               cudaGetErrorString(cudaGetLastError()));
    }
    for (int warps : {4, 8, 16, 32}) {
        ex2_bench<<<148, warps * 32>>>(iters, out, cyc);
        cudaDeviceSynchronize();
        long long c;
        cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        const double n = (double)warps * 32 * 8 * iters;
        printf("ex2: %2d warps: %.2f ex2/clk/SM\n", warps, n / c);
    }
    return 0;
}
