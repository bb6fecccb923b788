// Microbenchmark: per-SM throughput of the instructions an exp-bound softmax
// row reduction can be built from, on sm_100a (B200). Results guide the
// MUFU/FMA split in score.cu and attn.cu.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe_exp tools/probe_exp.cu
#include <cstdint>
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#define CHAINS 8

__device__ __forceinline__ float op_ex2_f32(float x) {
    float y;
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ uint32_t op_ex2_f16x2(uint32_t x) {
    uint32_t y;
    asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x));
    return y;
}
__device__ __forceinline__ uint32_t op_ex2_bf16x2(uint32_t x) {
    uint32_t y;
    asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x));
    return y;
}

template <int OP>
__global__ void bench(int iters, uint32_t* out, long long* cycles) {
    uint32_t a[CHAINS];
    float f[CHAINS];
    uint64_t d[CHAINS];
    for (int j = 0; j < CHAINS; ++j) {
        f[j] = -0.001f * (threadIdx.x + j);
        a[j] = 0xB800B800u + j;  // f16x2 (-0.5, -0.5)-ish
        d[j] = ((uint64_t)__float_as_uint(f[j]) << 32) | __float_as_uint(f[j]);
    }
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < CHAINS; ++j) {
            if (OP == 0) {
                f[j] = op_ex2_f32(f[j]);
            } else if (OP == 1) {
                a[j] = op_ex2_f16x2(a[j]) | 0x80008000u;
            } else if (OP == 2) {
                a[j] = op_ex2_bf16x2(a[j]) | 0x80008000u;
            } else if (OP == 3) {  // cvt.rn.f16x2.f32 (pack two fp32 into f16x2)
                uint32_t r;
                asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(f[j]), "f"(__uint_as_float(a[j])));
                a[j] = r;
            } else if (OP == 4) {  // FFMA2
                uint64_t r;
                asm volatile("fma.rn.f32x2 %0, %1, %1, %1;" : "=l"(r) : "l"(d[j]));
                d[j] = r;
            } else if (OP == 5) {  // FFMA
                asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(f[j]));
            } else if (OP == 6) {  // HADD2
                asm volatile("add.rn.f16x2 %0, %0, %0;" : "+r"(a[j]));
            } else if (OP == 7) {  // cvt f16 -> f32
                float r;
                asm volatile("{.reg .f16 h; mov.b32 {h, _}, %1; cvt.f32.f16 %0, h;}" : "=f"(r) : "r"(a[j]));
                a[j] = __float_as_uint(r);
            } else if (OP == 8) {  // mixed add.f32.f16 (sm_100 PTX 8.6)
                float r;
                asm volatile("{.reg .f16 h; mov.b32 {h, _}, %1; add.rn.f32.f16 %0, h, %2;}"
                             : "=f"(r)
                             : "r"(a[j]), "f"(f[j]));
                f[j] = r;
                a[j] += 1;
            } else if (OP == 9) {  // FMNMX3
                asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(f[j]) : "f"(f[(j + 1) % CHAINS]), "f"(f[(j + 2) % CHAINS]));
            } else if (OP == 11) {  // FFMA2 + FMNMX (ALU), independent
                uint64_t r;
                asm volatile("fma.rn.f32x2 %0, %1, %1, %1;" : "=l"(r) : "l"(d[j]));
                d[j] = r;
                asm volatile("max.f32 %0, %0, %1;" : "+f"(f[j]) : "f"(f[(j + 3) % CHAINS]));
            } else if (OP == 12) {  // FFMA2 + MUFU, independent
                uint64_t r;
                asm volatile("fma.rn.f32x2 %0, %1, %1, %1;" : "=l"(r) : "l"(d[j]));
                d[j] = r;
                f[j] = op_ex2_f32(f[j]);
            } else if (OP == 13) {  // 2 FFMA + FMNMX
                asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(f[j]));
                asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+r"(a[j]));
                asm volatile("max.f32 %0, %0, %1;" : "+r"(a[(j + 1) % CHAINS]) : "f"(f[(j + 3) % CHAINS]));
            } else if (OP == 14) {  // IMAD shift-add alone
                asm volatile("mad.lo.u32 %0, %0, 8388608, %1;" : "+r"(a[j]) : "r"(a[(j + 1) % CHAINS]));
            } else if (OP == 15) {  // FFMA2 + IMAD
                uint64_t r;
                asm volatile("fma.rn.f32x2 %0, %1, %1, %1;" : "=l"(r) : "l"(d[j]));
                d[j] = r;
                asm volatile("mad.lo.u32 %0, %0, 8388608, %1;" : "+r"(a[j]) : "r"(a[(j + 1) % CHAINS]));
            } else if (OP == 16) {  // FFMA2 + FFMA2 + MUFU + FMNMX (mixed softmax-like)
                uint64_t r, r2;
                asm volatile("fma.rn.f32x2 %0, %1, %1, %1;" : "=l"(r) : "l"(d[j]));
                asm volatile("add.rn.f32x2 %0, %1, %1;" : "=l"(r2) : "l"(r));
                d[j] = r2;
                f[j] = op_ex2_f32(f[j]);
                asm volatile("max.f32 %0, %0, %1;" : "+r"(a[j]) : "f"(f[(j + 3) % CHAINS]));
            } else if (OP == 17) {  // FFMA2 distinct operands
                uint64_t r;
                asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(d[j]), "l"(d[(j + 1) % CHAINS]), "l"(d[(j + 2) % CHAINS]));
                d[j] = r;
            } else if (OP == 18) {  // FFMA2 reg x reg + imm-pair (poly step)
                uint64_t r;
                asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(d[j]), "l"(d[(j + 1) % CHAINS]), "l"(0x3E7869E53E7869E5ull));
                d[j] = r;
            } else if (OP == 19) {  // FFMA distinct operands
                asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=f"(f[j]) : "f"(f[j]), "f"(f[(j + 1) % CHAINS]), "f"(f[(j + 2) % CHAINS]));
            } else if (OP == 20) {  // FADD2 distinct
                uint64_t r;
                asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(d[j]), "l"(d[(j + 1) % CHAINS]));
                d[j] = r;
            } else if (OP == 21) {  // FFMA2 distinct + MUFU (independent)
                uint64_t r;
                asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(d[j]), "l"(d[(j + 1) % CHAINS]), "l"(d[(j + 2) % CHAINS]));
                d[j] = r;
                f[j] = op_ex2_f32(f[j]);
            } else if (OP == 22) {  // 2 x FFMA distinct + MUFU
                asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=f"(f[j]) : "f"(f[j]), "f"(f[(j + 1) % CHAINS]), "f"(f[(j + 2) % CHAINS]));
                asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=r"(a[j]) : "r"(a[j]), "r"(a[(j + 1) % CHAINS]), "r"(a[(j + 2) % CHAINS]));
                a[(j + 3) % CHAINS] = __float_as_uint(op_ex2_f32(__uint_as_float(a[(j + 3) % CHAINS])));
            } else if (OP == 23) {  // cvt.rn.bf16x2.f32 (F2FP.BF16 pack)
                uint32_t r;
                asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(f[j]), "f"(__uint_as_float(a[j])));
                a[j] = r;
            } else if (OP == 24) {  // MUFU + bf16x2 pack, independent (per pair)
                uint32_t r;
                asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(__uint_as_float(a[j])), "f"(__uint_as_float(a[(j + 1) % CHAINS])));
                a[j] = r;
                f[j] = op_ex2_f32(f[j]);
            } else if (OP == 25) {  // FFMA2 + bf16x2 pack, independent (per pair)
                uint64_t r;
                asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(d[j]), "l"(d[(j + 1) % CHAINS]), "l"(d[(j + 2) % CHAINS]));
                d[j] = r;
                uint32_t q;
                asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(q) : "f"(__uint_as_float(a[j])), "f"(__uint_as_float(a[(j + 1) % CHAINS])));
                a[j] = q;
            } else if (OP == 26) {  // 2 MUFU + FFMA2 + bf16x2 pack (per pair of exps: the MMA-summed softmax step)
                uint64_t r;
                asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(d[j]), "l"(d[(j + 1) % CHAINS]), "l"(d[(j + 2) % CHAINS]));
                d[j] = r;
                f[j] = op_ex2_f32(f[j]);
                a[(j + 3) % CHAINS] = __float_as_uint(op_ex2_f32(__uint_as_float(a[(j + 3) % CHAINS])));
                uint32_t q;
                asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(q) : "f"(__uint_as_float(a[j])), "f"(f[(j + 1) % CHAINS]));
                a[j] ^= q;
            } else if (OP == 10) {  // HFMA2 with fp32-pair output? (fma.rn.f32x2 fed from f16 is not a thing) -> F2F pair
                uint64_t r;
                asm volatile(
                    "{.reg .f16 h0, h1; .reg .f32 x0, x1; mov.b32 {h0, h1}, %1; cvt.f32.f16 x0, h0; cvt.f32.f16 x1, h1;"
                    " mov.b64 %0, {x0, x1};}"
                    : "=l"(r)
                    : "r"(a[j]));
                d[j] += r;
                a[j] ^= (uint32_t)r;
            }
        }
    }
    long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
    uint32_t s = 0;
    for (int j = 0; j < CHAINS; ++j) s += a[j] + __float_as_uint(f[j]) + (uint32_t)d[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int OP>
void run(const char* name, int elems_per_op) {
    uint32_t* out;
    long long* cyc;
    cudaMalloc(&out, 148 * 1024 * 4);
    cudaMalloc(&cyc, 148 * 8);
    const int iters = 2048;
    for (int warps : {16, 32}) {
        bench<OP><<<148, warps * 32>>>(iters, out, cyc);
        cudaDeviceSynchronize();
        long long c;
        cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        const double n = (double)warps * 32 * CHAINS * iters;
        printf("%-28s %2d warps: %7.2f inst-lanes/clk/SM  %7.2f elems/clk/SM (%s)\n", name, warps, n / c,
               n * elems_per_op / c, cudaGetErrorString(cudaGetLastError()));
    }
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    run<0>("ex2.approx.ftz.f32", 1);
    run<1>("ex2.approx.f16x2", 2);
    run<2>("ex2.approx.ftz.bf16x2", 2);
    run<3>("cvt.rn.f16x2.f32", 2);
    run<4>("fma.rn.f32x2", 2);
    run<5>("fma.rn.f32", 1);
    run<6>("add.rn.f16x2", 2);
    run<7>("cvt.f32.f16", 1);
    run<8>("add.rn.f32.f16", 1);
    run<9>("max.f32 (3-input)", 1);
    run<10>("2x cvt.f32.f16 + add", 2);
    run<11>("FFMA2 + FMNMX (per pair)", 1);
    run<12>("FFMA2 + MUFU (per pair)", 1);
    run<13>("2 FFMA + FMNMX (per trio)", 1);
    run<14>("IMAD shift-add", 1);
    run<15>("FFMA2 + IMAD (per pair)", 1);
    run<16>("FFMA2+FADD2+MUFU+FMNMX (per 4)", 1);
    run<17>("FFMA2 distinct regs", 2);
    run<18>("FFMA2 reg,reg,imm", 2);
    run<19>("FFMA distinct regs", 1);
    run<20>("FADD2 distinct regs", 2);
    run<21>("FFMA2 distinct + MUFU (/pair)", 1);
    run<22>("2 FFMA distinct + MUFU (/trio)", 1);
    run<23>("cvt.rn.bf16x2.f32", 2);
    run<24>("MUFU + bf16x2 pack (/pair)", 1);
    run<25>("FFMA2 distinct + bf16x2 pack", 1);
    run<26>("2MUFU+FFMA2+pack (/quad)", 1);
    return 0;
}
