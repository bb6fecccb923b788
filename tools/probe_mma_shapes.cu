// Probe: tensor-pipe cycles per tcgen05.mma (kind::f16, cta_group::1, M = 128,
// K = 16) by N and operand source — the shapes of the mapper's encoder
// attention (attn.cu: S = Q·Kᵀ SS with N = 64 keys, O += P·V TS with N = 64)
// against wider tiles. Each CTA's elected thread issues `reps` groups of 4
// MMAs (K = 64) back to back into one accumulator; C CTAs per SM share the
// pipe. Prints cycles per MMA instruction per SM and the implied fraction of
// the dense floor (128·N/256 cycles).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//          -I paper_2605_16360_b200/csrc -o tools/probe_mma_shapes tools/probe_mma_shapes.cu
#include <cuda_fp16.h>

#include <cstdio>

#include "sm100.cuh"

using namespace pkv::sm100;

template <int N, bool TS>
__global__ void probe(int reps, long long* cycles) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = sm;            // 128 x 64 fp16, SW128 (16 KB)
    uint8_t* sB = sm + 16384;    // N x 64 fp16, SW128 (N x 128 B)
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 16384 + 256 * 128);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
    const int tid = threadIdx.x;
    for (int i = tid; i < (16384 + N * 128) / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
    fence_proxy_async_smem();
    if (tid == 0) {
        mbar_init(bar, 1);
        fence_barrier_init();
    }
    constexpr uint32_t kCols = 256;
    if (tid < 32) tmem_alloc(slot, kCols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *slot;
    constexpr uint32_t idesc = idesc_f16(128, N, 0);
    long long t0 = 0;
    if (tid < 32) {
        if (elect_one()) {
            t0 = clock64();
            const uint64_t a = desc_sw128(sA), b = desc_sw128(sB);
            for (int rep = 0; rep < reps; ++rep) {
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    if (TS) mma_f16_ts(tmem, tmem + 128 + kk * 8, b + kk * 2, idesc, (rep | kk) != 0);
                    else mma_f16_ss(tmem, a + kk * 2, b + kk * 2, idesc, (rep | kk) != 0);
                }
            }
            mma_commit(bar);
        }
        __syncwarp();
    }
    mbar_wait(bar, 0);
    if (tid == 0) cycles[blockIdx.x] = clock64() - t0;
    tc_fence_before();
    __syncthreads();
    if (tid < 32) {
        tc_fence_after();
        tmem_dealloc(tmem, kCols);
    }
}

template <int N, bool TS>
void run(int sms, int ctas_per_sm, long long* dcyc) {
    const int smem = 16384 + 256 * 128 + 64 + 1024;
    cudaFuncSetAttribute(probe<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int reps = 2048;
    probe<N, TS><<<sms * ctas_per_sm, 128, smem>>>(16, dcyc);
    probe<N, TS><<<sms * ctas_per_sm, 128, smem>>>(reps, dcyc);
    const cudaError_t e = cudaDeviceSynchronize();
    long long c = 0;
    cudaMemcpy(&c, dcyc, 8, cudaMemcpyDeviceToHost);
    const double per = (double)c / (reps * 4.0 * ctas_per_sm);
    const double floor = 128.0 * N / 256.0;
    printf("N=%3d %s  %d CTA/SM: %6.1f cycles per MMA per SM (floor %5.1f, %3.0f %%)  %s\n", N, TS ? "TS" : "SS",
           ctas_per_sm, per, floor, 100.0 * floor / per, cudaGetErrorString(e));
}


// Overlap probe: one CTA per SM, warp 0 issues a stream of N = 64 SS MMAs
// (attn.cu's S shape) into columns [0, 64) while warps 4-11 (two per lane
// quadrant, as two co-resident attention CTAs' softmax warps) run `work`
// iterations of: kind 1 — 64 independent MUFU ex2; kind 2 — two 32-column
// tcgen05.ld of columns [128, 192) + wait::ld; kind 3 — both. Each role's
// elapsed cycles are reported; run with mma_reps = 0 or work = 0 for the solo
// numbers.
__global__ void overlap(int mma_reps, int work, int kind, long long* out, float* sink) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = sm;
    uint8_t* sB = sm + 16384;
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 16384 + 8192);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < (16384 + 8192) / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
    fence_proxy_async_smem();
    if (tid == 0) {
        mbar_init(bar, 1);
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc(slot, 256);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *slot;
    if (warp == 0) {
        long long t0 = clock64();
        if (mma_reps > 0) {
            if (elect_one()) {
                const uint64_t a = desc_sw128(sA), b = desc_sw128(sB);
                constexpr uint32_t idesc = idesc_f16(128, 64, 0);
                for (int rep = 0; rep < mma_reps; ++rep)
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) mma_f16_ss(tmem, a + kk * 2, b + kk * 2, idesc, (rep | kk) != 0);
                mma_commit(bar);
            }
            __syncwarp();
            mbar_wait(bar, 0);
        }
        if (lane_id() == 0) out[blockIdx.x * 2] = clock64() - t0;
    } else if (warp >= 4) {
        const uint32_t quad = warp & 3;
        float x = 0.001f * tid, acc = 0.0f;
        long long t0 = clock64();
        for (int it = 0; it < work; ++it) {
            if (kind & 2) {
                uint32_t r[32], q[32];
                tmem_ld32(tmem + ((quad * 32) << 16) + 128, r);
                tmem_ld32(tmem + ((quad * 32) << 16) + 160, q);
                tmem_ld_wait();
#pragma unroll
                for (int u = 0; u < 32; ++u) acc += __uint_as_float(r[u]) + __uint_as_float(q[u]);
            }
            if (kind & 1) {
                float e[8] = {};
#pragma unroll
                for (int u = 0; u < 64; ++u) e[u & 7] += ex2(x + 0.01f * u);
                x += e[0] + e[1] + e[2] + e[3] + e[4] + e[5] + e[6] + e[7];
            }
        }
        if (lane_id() == 0 && warp == 4) out[blockIdx.x * 2 + 1] = clock64() - t0;
        if (x == 1.2345f || acc == 1.2345f) sink[tid] = x + acc;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 256);
    }
}

void run_overlap(int sms, int mma_reps, int work, int kind, long long* dcyc, float* sink) {
    const int smem = 16384 + 8192 + 64 + 1024;
    overlap<<<sms, 384, smem>>>(mma_reps, work, kind, dcyc, sink);
    const cudaError_t e = cudaDeviceSynchronize();
    long long c[2] = {0, 0};
    cudaMemcpy(c, dcyc, 16, cudaMemcpyDeviceToHost);
    printf("overlap kind %d  mma groups %5d  work %5d:  mma %9lld cyc (%5.1f per MMA)  workers %9lld cyc  %s\n", kind,
           mma_reps, work, c[0], mma_reps ? (double)c[0] / (mma_reps * 4.0) : 0.0, c[1], cudaGetErrorString(e));
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    long long* dcyc;
    cudaMalloc(&dcyc, sizeof(long long) * sms * 4);
    for (int c = 1; c <= 2; ++c) {
        run<32, false>(sms, c, dcyc);
        run<64, false>(sms, c, dcyc);
        run<128, false>(sms, c, dcyc);
        run<256, false>(sms, c, dcyc);
        run<64, true>(sms, c, dcyc);
        run<128, true>(sms, c, dcyc);
    }
    float* sink;
    cudaMalloc(&sink, 4096);
    const int R = 4096, W = 2048;
    for (int kind = 1; kind <= 3; ++kind) {
        run_overlap(sms, R, 0, kind, dcyc, sink);
        run_overlap(sms, 0, W, kind, dcyc, sink);
        run_overlap(sms, R, W, kind, dcyc, sink);
    }
    return 0;
}
