// Probe: do tcgen05.mma kind::f16 and kind::f8f6f4 accumulate into the same
// TMEM tile, and is the K-major 64-byte-swizzled e4m3 operand layout (64
// fp8 = one 64-B row per K block, two K = 32 MMAs per block) read as expected?
// D[128 x 128] = A16·B16ᵀ (fp16, K = 64) + A8·B8ᵀ (e4m3, K = 64), checked
// against a double-precision host product of the same (rounded) values; also
// times N back-to-back issue groups of each kind.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe_f8mma tools/probe_f8mma.cu
#include <cuda_fp16.h>
#include <cuda_fp8.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2605_16360_b200/csrc/sm100.cuh"

using namespace pkv::sm100;

__device__ __forceinline__ void mma_f8_ss(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ uint64_t desc_sw64(const void* smem_tile) {
    const uint64_t addr = smem_u32(smem_tile);
    uint64_t d = 0;
    d |= (addr >> 4) & 0x3FFFull;
    d |= 1ull << 16;
    d |= (uint64_t)(512 >> 4) << 32;  // SBO: 8 rows x 64 B
    d |= 1ull << 46;
    d |= 4ull << 61;  // SWIZZLE_64B
    return d;
}

// a16/b16: [128][64] fp16 row-major; a8/b8: [128][64] e4m3 row-major (bytes)
__global__ void probe(const __half* a16, const __half* b16, const uint8_t* a8, const uint8_t* b8, float* out,
                      int mode, int reps, long long* cycles) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA16 = sm;            // 16 KB, SW128
    uint8_t* sB16 = sm + 16384;    // 16 KB
    uint8_t* sA8 = sm + 32768;     // 8 KB, SW64
    uint8_t* sB8 = sm + 40960;     // 8 KB
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 49152);
    uint32_t* slot = reinterpret_cast<uint32_t*>(sm + 49160);
    const int tid = threadIdx.x;
    // swizzled fills: SW128 16-B chunk c of row r at r*128 + ((c ^ (r & 7)) * 16);
    // SW64 chunk c (0..3) of row r at r*64 + ((c ^ ((r >> 1) & 3)) * 16)
    for (int i = tid; i < 128 * 8; i += blockDim.x) {
        const int r = i / 8, c = i % 8;
        *reinterpret_cast<uint4*>(sA16 + r * 128 + ((c ^ (r & 7)) * 16)) = reinterpret_cast<const uint4*>(a16 + r * 64)[c];
        *reinterpret_cast<uint4*>(sB16 + r * 128 + ((c ^ (r & 7)) * 16)) = reinterpret_cast<const uint4*>(b16 + r * 64)[c];
    }
    for (int i = tid; i < 128 * 4; i += blockDim.x) {
        const int r = i / 4, c = i % 4;
        *reinterpret_cast<uint4*>(sA8 + r * 64 + ((c ^ ((r >> 1) & 3)) * 16)) = reinterpret_cast<const uint4*>(a8 + r * 64)[c];
        *reinterpret_cast<uint4*>(sB8 + r * 64 + ((c ^ ((r >> 1) & 3)) * 16)) = reinterpret_cast<const uint4*>(b8 + r * 64)[c];
    }
    fence_proxy_async_smem();
    if (tid == 0) {
        mbar_init(bar, 1);
        fence_barrier_init();
    }
    if (tid < 32) tmem_alloc(slot, 128);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *slot;
    constexpr uint32_t idesc = idesc_f16(128, 128, 0);  // fp16 x fp16 / e4m3 x e4m3 (format 0), f32 D
    long long t0 = 0, t1 = 0;
    if (tid < 32) {
        if (elect_one()) {
            t0 = clock64();
            for (int rep = 0; rep < reps; ++rep) {
                const uint32_t acc0 = rep > 0;
                if (mode & 1) {
                    const uint64_t a = desc_sw128(sA16), b = desc_sw128(sB16);
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) mma_f16_ss(tmem, a + kk * 2, b + kk * 2, idesc, (acc0 | kk) != 0);
                }
                if (mode & 2) {
                    const uint64_t a = desc_sw64(sA8), b = desc_sw64(sB8);
#pragma unroll
                    for (int kk = 0; kk < 2; ++kk)
                        mma_f8_ss(tmem, a + kk * 2, b + kk * 2, idesc, (acc0 | (mode & 1) | kk) != 0);
                }
            }
            mma_commit(bar);
        }
        __syncwarp();
    }
    mbar_wait(bar, 0);
    if (tid == 0) {
        t1 = clock64();
        *cycles = t1 - t0;
    }
    tc_fence_after();
    if (tid < 128) {
        const uint32_t quad = tid >> 5;
        for (int c = 0; c < 128; c += 32) {
            uint32_t r[32];
            tmem_ld32(tmem + ((quad * 32) << 16) + c, r);
            tmem_ld_wait();
            for (int j = 0; j < 32; ++j) out[tid * 128 + c + j] = __uint_as_float(r[j]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (tid < 32) {
        tc_fence_after();
        tmem_dealloc(tmem, 128);
    }
}

int main() {
    const int M = 128, N = 128, K = 64;
    std::vector<__half> a16(M * K), b16(N * K);
    std::vector<uint8_t> a8(M * K), b8(N * K);
    std::vector<double> fa16(M * K), fb16(N * K), fa8(M * K), fb8(N * K);
    srand(1);
    auto rnd = [] { return (double)rand() / RAND_MAX * 2.0 - 1.0; };
    for (int i = 0; i < M * K; ++i) {
        a16[i] = __double2half(rnd());
        fa16[i] = __half2float(a16[i]);
        __nv_fp8_e4m3 e(static_cast<float>(rnd() * 8.0));
        a8[i] = e.__x;
        fa8[i] = static_cast<float>(e);
    }
    for (int i = 0; i < N * K; ++i) {
        b16[i] = __double2half(rnd());
        fb16[i] = __half2float(b16[i]);
        __nv_fp8_e4m3 e(static_cast<float>(rnd() * 8.0));
        b8[i] = e.__x;
        fb8[i] = static_cast<float>(e);
    }
    __half *da16, *db16;
    uint8_t *da8, *db8;
    float* dout;
    long long* dcyc;
    cudaMalloc(&da16, M * K * 2);
    cudaMalloc(&db16, N * K * 2);
    cudaMalloc(&da8, M * K);
    cudaMalloc(&db8, N * K);
    cudaMalloc(&dout, M * N * 4);
    cudaMalloc(&dcyc, 8);
    cudaMemcpy(da16, a16.data(), M * K * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(db16, b16.data(), N * K * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(da8, a8.data(), M * K, cudaMemcpyHostToDevice);
    cudaMemcpy(db8, b8.data(), N * K, cudaMemcpyHostToDevice);
    const int smem = 49152 + 64 + 1024;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    std::vector<float> out(M * N);
    for (int mode = 1; mode <= 3; ++mode) {
        probe<<<1, 128, smem>>>(da16, db16, da8, db8, dout, mode, 1, dcyc);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("mode %d: %s\n", mode, cudaGetErrorString(e));
            return 1;
        }
        cudaMemcpy(out.data(), dout, M * N * 4, cudaMemcpyDeviceToHost);
        double maxerr = 0, maxref = 0;
        for (int i = 0; i < M; ++i)
            for (int j = 0; j < N; ++j) {
                double r = 0;
                for (int k = 0; k < K; ++k) {
                    if (mode & 1) r += fa16[i * K + k] * fb16[j * K + k];
                    if (mode & 2) r += fa8[i * K + k] * fb8[j * K + k];
                }
                maxerr = fmax(maxerr, fabs(out[i * N + j] - r));
                maxref = fmax(maxref, fabs(r));
            }
        printf("mode %d (%s): max |D - ref| = %.3e (max |ref| %.3e)\n", mode,
               mode == 1 ? "fp16 only" : mode == 2 ? "e4m3 only" : "fp16 + e4m3 into one accumulator", maxerr, maxref);
    }
    for (int mode = 1; mode <= 3; ++mode) {
        long long cyc = 0;
        probe<<<1, 128, smem>>>(da16, db16, da8, db8, dout, mode, 512, dcyc);
        cudaDeviceSynchronize();
        cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost);
        printf("mode %d: 512 K=64 blocks in %lld cycles = %.1f cycles per 128x128x64 block\n", mode, cyc, cyc / 512.0);
    }
    return 0;
}
