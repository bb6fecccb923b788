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

// Variant: the scores arrive already as c·s − m (an MMA over pre-scaled,
// m-augmented operands would produce that), so MUFU pairs skip the FFMA2 and
// the polynomial's range reduction is an FADD2.
template <int kPolyPairs>
__device__ __forceinline__ float lse_chunk_pre(const uint32_t (&ra)[32], const uint32_t (&rb)[32]) {
    using namespace pkv::sm100;
    uint64_t acc0 = pack2(0.0f, 0.0f), acc1 = acc0;
#pragma unroll
    for (int pr = 0; pr < 32; ++pr) {
        const uint64_t s2 = pr < 16 ? pack2(__uint_as_float(ra[2 * pr]), __uint_as_float(ra[2 * pr + 1]))
                                    : pack2(__uint_as_float(rb[2 * pr - 32]), __uint_as_float(rb[2 * pr - 31]));
        uint64_t e;
        if (((pr + 1) * kPolyPairs) / 32 != (pr * kPolyPairs) / 32) {
            uint64_t t = fadd2(s2, pack2(12582912.0f, 12582912.0f));
            float2 tf = unpack2(t);
            tf.x = fmaxf(tf.x, 12582912.0f - 125.0f);
            tf.y = fmaxf(tf.y, 12582912.0f - 125.0f);
            t = pack2(tf.x, tf.y);
            const uint64_t f = fadd2(s2, fsub2_s(12582912.0f, t));
            uint64_t p = ffma2_ss(f, 0.05508868396282196f, 0.24260404706001282f);
            p = ffma2_ps(p, f, 0.6932762265205383f);
            p = ffma2_ps(p, f, 0.9999289512634277f);
            const float2 pf = unpack2(p);
            e = pack2(__int_as_float((__float_as_int(tf.x) << 23) + __float_as_int(pf.x)),
                      __int_as_float((__float_as_int(tf.y) << 23) + __float_as_int(pf.y)));
        } else {
            const float2 x = unpack2(s2);
            e = pack2(ex2(x.x), ex2(x.y));
        }
        if (pr & 1) acc1 = fadd2(acc1, e);
        else acc0 = fadd2(acc0, e);
    }
    const float2 ssum = unpack2(fadd2(acc0, acc1));
    return ssum.x + ssum.y;
}

template <int kPoly, bool kPre>
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
    float* stage = reinterpret_cast<float*>(smem_pad) + (warp - 2) * 32 * 64;  // per warp: 32 lanes x 64 scores
    for (int i = 0; i < 64; ++i)
        stage[((i >> 2) * 32 + (threadIdx.x & 31)) * 4 + (i & 3)] = __uint_as_float(i < 32 ? ra[i] : rb[i - 32]) - 3.0f;
    float lsum = 0.0f;
    __syncwarp();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const float m = m0 + (float)(it & 1) * 0.5f;  // varies: nothing hoisted out of the loop
        if (kPre) {
            // the pre-scaled scores come from shared memory each iteration (a
            // stand-in for the kernel's TMEM load; ptxas cannot hoist the chunk)
            const uint4* src = reinterpret_cast<const uint4*>(stage) + (threadIdx.x & 31);  // [16][32 lanes] uint4
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const uint4 u = src[32 * ((i + it) & 15)], w = src[32 * ((i + 8 + it) & 15)];
                ra[4 * i] = u.x; ra[4 * i + 1] = u.y; ra[4 * i + 2] = u.z; ra[4 * i + 3] = u.w;
                rb[4 * i] = w.x; rb[4 * i + 1] = w.y; rb[4 * i + 2] = w.z; rb[4 * i + 3] = w.w;
            }
            lsum += lse_chunk_pre<kPoly>(ra, rb);
        }
        else lsum += pkv::lse_chunk_fixed<kPoly, 64>(ra, rb, 64, -m, 12582912.0f - m);
    }
    const long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = lsum;
    if (threadIdx.x == 64) cycles[blockIdx.x] = t1 - t0;
}

template <int kPoly, bool kPre = false>
void run(int sms) {
    float* out;
    long long* cyc;
    cudaMalloc(&out, sms * 576 * 4);
    cudaMalloc(&cyc, sms * 8);
    const int iters = 4096;
    const int smem = 200 * 1024;
    cudaFuncSetAttribute(probe<kPoly, kPre>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    probe<kPoly, kPre><<<sms, 576, smem>>>(64, out, cyc);  // warm-up
    probe<kPoly, kPre><<<sms, 576, smem>>>(iters, out, cyc);
    cudaDeviceSynchronize();
    long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    const double exps = 16.0 * 32 * 64 * iters;  // per SM
    printf("%s poly pairs %2d of 32: %6.2f exponentials/clk/SM (%s)\n", kPre ? "prescaled" : "fixed    ", kPoly, exps / c,
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
    run<8, true>(sms);
    run<10, true>(sms);
    run<12, true>(sms);
    run<14, true>(sms);
    run<16, true>(sms);
    run<18, true>(sms);
    run<20, true>(sms);
    return 0;
}
