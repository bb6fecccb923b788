// select.cu — per-(layer, head) Top-K budget selection as a block-wide radix
// select with the reference's deterministic tie-break, fused with the
// ascending stream compaction of apply_mask.
//
// Replaces topk_indices / topk_mask (proj/src/pruning.cpp:20-56) and the
// retained-index lists of apply_mask (proj/src/pruning.cpp:197-215).
// Order: better(a,b) = v[a] > v[b] || (v[a] == v[b] && a < b)
// (pruning.cpp:24-31), with -0.0 == +0.0 as in the reference's `!=`.
//
// One CTA (1024 threads) per slice; HBM-bound: the slice is read once from
// HBM, the 3 later digit passes and the output pass hit L2 (slices of
// 128-680 KB, whole score tensor 16-76 MB << 126 MB L2).
#include "internal.h"

namespace pkv {
namespace {

constexpr int kThreads = 1024;
constexpr int kWarps = kThreads / 32;
constexpr int kItems = 8;  // consecutive elements per thread in the output pass

__device__ __forceinline__ uint32_t order_key(float f) {
    uint32_t u = __float_as_uint(f);
    if ((u << 1) == 0) u = 0;  // -0.0 -> +0.0
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// Block-wide exclusive scan of one uint32 per thread; also returns the total.
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* warp_sums, uint32_t& total) {
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= (uint32_t)o) x += y;
    }
    if (lane == 31) warp_sums[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = warp_sums[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= (uint32_t)o) w += y;
        }
        warp_sums[lane] = w;
    }
    __syncthreads();
    const uint32_t base = warp ? warp_sums[warp - 1] : 0u;
    total = warp_sums[kWarps - 1];
    __syncthreads();
    return base + x - v;
}

__global__ void __launch_bounds__(kThreads, 2)
    topk_select_kernel(const float* __restrict__ scores, int64_t n, int64_t k, uint8_t* __restrict__ mask,
                       int32_t* __restrict__ idx) {
    __shared__ uint32_t hist[256];
    __shared__ uint32_t warp_sums[kWarps];
    __shared__ uint32_t s_digit, s_above;

    const int64_t slice = blockIdx.x;
    const float* __restrict__ v = scores + slice * n;
    const bool vec4 = (n & 3) == 0;
    const int tid = threadIdx.x;

    // ---- radix select of the k-th largest key, 4 digit passes of 8 bits
    uint32_t prefix = 0, pmask = 0, kr = (uint32_t)k;
    for (int pass = 0; pass < 4; ++pass) {
        const int shift = 24 - 8 * pass;
        if (tid < 256) hist[tid] = 0;
        __syncthreads();
        if (vec4) {
            const float4* v4 = reinterpret_cast<const float4*>(v);
            for (int64_t i = tid; i < (n >> 2); i += kThreads) {
                const float4 f = v4[i];
                const uint32_t k0 = order_key(f.x), k1 = order_key(f.y), k2 = order_key(f.z), k3 = order_key(f.w);
                if ((k0 & pmask) == prefix) atomicAdd(&hist[(k0 >> shift) & 255u], 1u);
                if ((k1 & pmask) == prefix) atomicAdd(&hist[(k1 >> shift) & 255u], 1u);
                if ((k2 & pmask) == prefix) atomicAdd(&hist[(k2 >> shift) & 255u], 1u);
                if ((k3 & pmask) == prefix) atomicAdd(&hist[(k3 >> shift) & 255u], 1u);
            }
        } else {
            for (int64_t i = tid; i < n; i += kThreads) {
                const uint32_t key = order_key(v[i]);
                if ((key & pmask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
            }
        }
        __syncthreads();
        if (tid < 32) {
            // lane l owns bins 255-8l .. 248-8l (descending digit order)
            uint32_t c[8], s = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                c[j] = hist[255 - (tid * 8 + j)];
                s += c[j];
            }
            uint32_t incl = s;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (tid >= o) incl += y;
            }
            const uint32_t excl = incl - s;
            if (excl < kr && kr <= incl) {
                uint32_t acc = excl;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    if (acc < kr && kr <= acc + c[j]) {
                        s_digit = 255u - (uint32_t)(tid * 8 + j);
                        s_above = acc;
                    }
                    acc += c[j];
                }
            }
        }
        __syncthreads();
        prefix |= s_digit << shift;
        pmask |= 0xFFu << shift;
        kr -= s_above;
        __syncthreads();
    }
    const uint32_t kth = prefix;  // key of the k-th best value
    const uint32_t ties_taken = kr;  // lowest-index elements with key == kth to keep

    // ---- ordered output: mask bits and ascending retained indices
    uint32_t sel_base = 0, tie_base = 0;
    uint8_t* __restrict__ mrow = mask ? mask + slice * n : nullptr;
    int32_t* __restrict__ irow = idx ? idx + slice * k : nullptr;
    for (int64_t t0 = 0; t0 < n; t0 += (int64_t)kThreads * kItems) {
        const int64_t i0 = t0 + (int64_t)tid * kItems;
        uint32_t gt = 0, eq = 0;
        if (vec4 && i0 + kItems <= n) {
            const float4 a = *reinterpret_cast<const float4*>(v + i0);
            const float4 b = *reinterpret_cast<const float4*>(v + i0 + 4);
            const float f[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
            for (int j = 0; j < kItems; ++j) {
                const uint32_t key = order_key(f[j]);
                gt |= (uint32_t)(key > kth) << j;
                eq |= (uint32_t)(key == kth) << j;
            }
        } else {
#pragma unroll
            for (int j = 0; j < kItems; ++j) {
                if (i0 + j < n) {
                    const uint32_t key = order_key(v[i0 + j]);
                    gt |= (uint32_t)(key > kth) << j;
                    eq |= (uint32_t)(key == kth) << j;
                }
            }
        }
        uint32_t tot_eq;
        const uint32_t eq_excl = block_excl_scan(__popc(eq), warp_sums, tot_eq);
        uint32_t sel = gt, run = tie_base + eq_excl;
#pragma unroll
        for (int j = 0; j < kItems; ++j) {
            if (eq & (1u << j)) {
                if (run < ties_taken) sel |= 1u << j;
                ++run;
            }
        }
        uint32_t tot_sel;
        const uint32_t sel_excl = block_excl_scan(__popc(sel), warp_sums, tot_sel);
        if (irow) {
            uint32_t pos = sel_base + sel_excl;
#pragma unroll
            for (int j = 0; j < kItems; ++j) {
                if (sel & (1u << j)) irow[pos++] = (int32_t)(i0 + j);
            }
        }
        if (mrow) {
            if ((n & 7) == 0 && i0 + kItems <= n) {
                uint2 w;
                w.x = (sel & 1u) | ((sel >> 1) & 1u) << 8 | ((sel >> 2) & 1u) << 16 | ((sel >> 3) & 1u) << 24;
                w.y = ((sel >> 4) & 1u) | ((sel >> 5) & 1u) << 8 | ((sel >> 6) & 1u) << 16 | ((sel >> 7) & 1u) << 24;
                *reinterpret_cast<uint2*>(mrow + i0) = w;
            } else {
#pragma unroll
                for (int j = 0; j < kItems; ++j) {
                    if (i0 + j < n) mrow[i0 + j] = (uint8_t)((sel >> j) & 1u);
                }
            }
        }
        sel_base += tot_sel;
        tie_base += tot_eq;
        if (!mrow && sel_base >= (uint32_t)k) break;  // all indices emitted
    }
}

}  // namespace

void launch_topk_select(const float* scores, int64_t slices, int64_t n, int64_t k, uint8_t* mask, int32_t* idx,
                        cudaStream_t st) {
    if (slices == 0) return;
    topk_select_kernel<<<(unsigned)slices, kThreads, 0, st>>>(scores, n, k, mask, idx);
    check_launch("topk_select_kernel");
}

}  // namespace pkv
