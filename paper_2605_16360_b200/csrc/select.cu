// select.cu — per-(layer, head) Top-K budget selection as a block-wide radix
// select with the reference's deterministic tie-break, fused with the
// ascending stream compaction of apply_mask.
//
// Replaces topk_indices / topk_mask (proj/src/pruning.cpp:20-56) and the
// retained-index lists of apply_mask (proj/src/pruning.cpp:197-215).
// Order: better(a,b) = v[a] > v[b] || (v[a] == v[b] && a < b)
// (pruning.cpp:24-31), with -0.0 == +0.0 as in the reference's `!=`.
// fp32 scores (the device pipeline's Ŷ) use 32-bit order keys; fp64 scores
// (the reference's ScoreTensor, pkv_topk_select_f64 / pkv_topk_mask_host) use
// 64-bit keys, so the drop-in ranks arbitrary doubles exactly.
//
// One CTA (1024 threads) per slice; HBM-bound: the slice is read once from
// HBM, the 2 later digit passes and the output pass hit L2 (slices of
// 128-680 KB, whole score tensor 16-76 MB << 126 MB L2).
#include <cstdlib>

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
// fp64 scores (the reference's own ScoreTensor type, tensor.hpp:86): the same
// monotone map on the 64-bit pattern, so distinct doubles never tie.
__device__ __forceinline__ uint64_t order_key(double f) {
    uint64_t u = (uint64_t)__double_as_longlong(f);
    if ((u << 1) == 0) u = 0;
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

// Radix digit schedule (most significant first): 12/12/8 bits for 32-bit
// keys, 12 x 5 + 4 for 64-bit keys.
template <typename K>
struct Digits;
template <>
struct Digits<uint32_t> {
    static constexpr int kPasses = 3;
    __device__ static int bits(int p) { return p < 2 ? 12 : 8; }
    __device__ static int shift(int p) { return p == 0 ? 20 : (p == 1 ? 8 : 0); }
};
template <>
struct Digits<uint64_t> {
    static constexpr int kPasses = 6;
    __device__ static int bits(int p) { return p < 5 ? 12 : 4; }
    __device__ static int shift(int p) { return p < 5 ? 52 - 12 * p : 0; }
};

// Block-wide exclusive scan of one uint32 per thread; also returns the total.
template <int kT = kThreads>
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* warp_sums, uint32_t& total) {
    constexpr int kW = kT / 32;
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
        uint32_t w = lane < (uint32_t)kW ? warp_sums[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= (uint32_t)o) w += y;
        }
        if (lane < (uint32_t)kW) warp_sums[lane] = w;
    }
    __syncthreads();
    const uint32_t base = warp ? warp_sums[warp - 1] : 0u;
    total = warp_sums[kW - 1];
    __syncthreads();
    return base + x - v;
}

// Generic path (rows > 32768 elements, or fp64 scores): the row is re-read
// per digit pass (L2-resident after the first) instead of register-cached.
// T: float or double; aligned16 / mask8: the caller's pointers allow the
// float4 loads / uint2 mask stores.
template <typename T>
__global__ void __launch_bounds__(kThreads, 1)
    topk_select_kernel(const T* __restrict__ scores, int64_t n, int64_t k, uint8_t* __restrict__ mask,
                       int32_t* __restrict__ idx, bool aligned16, bool mask8) {
    using Key = decltype(order_key(T(0)));
    using D = Digits<Key>;
    __shared__ uint32_t hist[4096 + kWarps];  // + one discard bin per warp
    __shared__ uint32_t warp_sums[kWarps];
    __shared__ uint32_t s_digit, s_above;

    const int64_t slice = blockIdx.x;
    const uint32_t trash = 4096u + (threadIdx.x >> 5);
    const T* __restrict__ v = scores + slice * n;
    const bool vec4 = sizeof(T) == 4 && aligned16 && (n & 3) == 0;
    const int tid = threadIdx.x;

    // ---- radix select of the k-th largest key. Wide first digits spread
    // score rows that share a few exponent values over many bins (same-bin
    // shared atomics serialise).
    Key prefix = 0, pmask = 0;
    uint32_t kr = (uint32_t)k;
#pragma unroll 1
    for (int pass = 0; pass < D::kPasses; ++pass) {
        const int bits = D::bits(pass);
        const int shift = D::shift(pass);
        const uint32_t nb = 1u << bits, dmask = nb - 1;
        for (uint32_t j = tid; j < nb; j += kThreads) hist[j] = 0;
        __syncthreads();
        auto add = [&](Key key) {  // branch-free: non-candidates into the warp's discard bin
            atomicAdd(&hist[(key & pmask) == prefix ? (uint32_t)(key >> shift) & dmask : trash], 1u);
        };
        if (vec4) {
            const float4* v4 = reinterpret_cast<const float4*>(v);
            const int64_t n4 = n >> 2;
            for (int64_t i0 = tid; i0 < n4; i0 += 2 * kThreads) {
                float4 f[2];
#pragma unroll
                for (int u = 0; u < 2; ++u)
                    f[u] = (i0 + u * kThreads < n4) ? v4[i0 + u * kThreads] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    if (i0 + u * kThreads >= n4) break;
                    add(order_key(f[u].x));
                    add(order_key(f[u].y));
                    add(order_key(f[u].z));
                    add(order_key(f[u].w));
                }
            }
        } else {
            for (int64_t i = tid; i < n; i += kThreads) add(order_key(v[i]));
        }
        __syncthreads();
        // thread t owns bins_per_thread consecutive bins in descending digit order
        const uint32_t bpt = nb / kThreads;  // 4 (12-bit digits) or 0 (8/4-bit)
        uint32_t c[4] = {0, 0, 0, 0}, sum = 0;
        if (bpt) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                c[j] = hist[nb - 1 - (tid * 4 + j)];
                sum += c[j];
            }
        } else if ((uint32_t)tid < nb) {
            c[0] = hist[nb - 1 - tid];
            sum = c[0];
        }
        uint32_t total;
        const uint32_t excl = block_excl_scan(sum, warp_sums, total);
        if (excl < kr && kr <= excl + sum) {
            uint32_t acc = excl;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (acc < kr && kr <= acc + c[j]) {
                    s_digit = nb - 1 - (uint32_t)(bpt ? tid * 4 + j : tid);
                    s_above = acc;
                }
                acc += c[j];
            }
        }
        __syncthreads();
        prefix |= (Key)s_digit << shift;
        pmask |= (Key)dmask << shift;
        kr -= s_above;
        __syncthreads();
    }
    const Key kth = prefix;          // key of the k-th best value
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
                const Key key = order_key(f[j]);
                gt |= (uint32_t)(key > kth) << j;
                eq |= (uint32_t)(key == kth) << j;
            }
        } else {
#pragma unroll
            for (int j = 0; j < kItems; ++j) {
                if (i0 + j < n) {
                    const Key key = order_key(v[i0 + j]);
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
            if (mask8 && (n & 7) == 0 && i0 + kItems <= n) {
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

// Rows of n <= kThreads * kItems * kCacheTiles (32768) elements: the row's
// order keys are read once into registers (thread t holds the same
// consecutive-8 groups the output pass uses) and the three digit passes and
// the output pass run on them — one global read per element instead of four,
// and no key recomputation (the uncached kernel is ALU-bound on it).
constexpr int kCacheTiles = 4;

template <int kT>
__global__ void __launch_bounds__(kT, 1024 / kT)
    topk_select_cached_kernel(const float* __restrict__ scores, int64_t n, int64_t k, uint8_t* __restrict__ mask,
                              int32_t* __restrict__ idx, bool aligned16) {
    __shared__ uint32_t hist[4096 + kT / 32];  // + one discard bin per warp
    __shared__ uint32_t warp_sums[32];
    __shared__ uint32_t s_digit, s_above;
    const int tid = threadIdx.x;
    const int64_t slice = blockIdx.x;
    const int nn = (int)n;
    const uint32_t trash = 4096u + (uint32_t)(tid >> 5);
    const float* __restrict__ v = scores + slice * n;
    const int ntiles = (nn + kT * kItems - 1) / (kT * kItems);
    uint32_t key[kCacheTiles][kItems];
#pragma unroll
    for (int t = 0; t < kCacheTiles; ++t) {
        const int i0 = t * kT * kItems + tid * kItems;
        if (aligned16 && (nn & 3) == 0 && i0 + kItems <= nn) {
            const float4 a = __ldcs(reinterpret_cast<const float4*>(v + i0));
            const float4 b = __ldcs(reinterpret_cast<const float4*>(v + i0 + 4));
            key[t][0] = order_key(a.x);
            key[t][1] = order_key(a.y);
            key[t][2] = order_key(a.z);
            key[t][3] = order_key(a.w);
            key[t][4] = order_key(b.x);
            key[t][5] = order_key(b.y);
            key[t][6] = order_key(b.z);
            key[t][7] = order_key(b.w);
        } else {
#pragma unroll
            for (int j = 0; j < kItems; ++j) key[t][j] = (i0 + j < nn) ? order_key(v[i0 + j]) : 0u;
        }
    }
    // per tile: number of this thread's items that exist
    auto nvalid = [&](int t) {
        const int i0 = t * kT * kItems + tid * kItems;
        const int r = nn - i0;
        return r <= 0 ? 0 : (r >= kItems ? kItems : r);
    };
    uint32_t prefix = 0, pmask = 0, kr = (uint32_t)k;
#pragma unroll 1
    for (int pass = 0; pass < 3; ++pass) {
        const int bits = pass < 2 ? 12 : 8;
        const int shift = pass == 0 ? 20 : (pass == 1 ? 8 : 0);
        const uint32_t nb = 1u << bits, dmask = nb - 1;
        for (uint32_t j = tid; j < nb; j += kT) hist[j] = 0;
        __syncthreads();
        // branch-free: non-candidates count into this warp's discard bin
        // (ATOMS.POPC.INC merges a warp's same-address increments)
#pragma unroll
        for (int t = 0; t < kCacheTiles; ++t) {
            if (t >= ntiles) break;
            const int nv = nvalid(t);
#pragma unroll
            for (int j = 0; j < kItems; ++j) {
                const bool ok = j < nv && (key[t][j] & pmask) == prefix;
                atomicAdd(&hist[ok ? (key[t][j] >> shift) & dmask : trash], 1u);
            }
        }
        __syncthreads();
        // thread t owns bpt consecutive bins in descending digit order
        constexpr int kBpt = 4096 / kT;  // bins per thread for the 12-bit digits
        const int bpt = (int)(nb / kT) > 1 ? (int)(nb / kT) : 1;
        uint32_t c[kBpt], sum = 0;
#pragma unroll
        for (int jj = 0; jj < kBpt; ++jj) {
            const int bin = tid * bpt + jj;
            c[jj] = (jj < bpt && bin < (int)nb) ? hist[nb - 1 - bin] : 0u;
            sum += c[jj];
        }
        uint32_t total;
        const uint32_t excl = block_excl_scan<kT>(sum, warp_sums, total);
        if (excl < kr && kr <= excl + sum) {
            uint32_t acc = excl;
#pragma unroll
            for (int jj = 0; jj < kBpt; ++jj) {
                if (acc < kr && kr <= acc + c[jj]) {
                    s_digit = nb - 1 - (uint32_t)(tid * bpt + jj);
                    s_above = acc;
                }
                acc += c[jj];
            }
        }
        __syncthreads();
        prefix |= s_digit << shift;
        pmask |= dmask << shift;
        kr -= s_above;
        __syncthreads();
    }
    const uint32_t kth = prefix, ties_taken = kr;
    uint32_t sel_base = 0, tie_base = 0;
    uint8_t* __restrict__ mrow = mask ? mask + slice * n : nullptr;
    int32_t* __restrict__ irow = idx ? idx + slice * k : nullptr;
#pragma unroll
    for (int t = 0; t < kCacheTiles; ++t) {
        if (t >= ntiles) break;
        const int i0 = t * kT * kItems + tid * kItems;
        const int nv = nvalid(t);
        uint32_t gt = 0, eq = 0;
#pragma unroll
        for (int j = 0; j < kItems; ++j) {
            const uint32_t in = (uint32_t)(j < nv);
            gt |= (in & (uint32_t)(key[t][j] > kth)) << j;
            eq |= (in & (uint32_t)(key[t][j] == kth)) << j;
        }
        // one scan of (#greater, #equal) packed in 16-bit halves (< 8192 each);
        // ties go to the lowest indices: this thread takes the first
        // min(ties left - equal keys before it, #equal) of its own
        uint32_t tot;
        const uint32_t excl = block_excl_scan<kT>((uint32_t)__popc(gt) | ((uint32_t)__popc(eq) << 16), warp_sums, tot);
        const uint32_t gt_excl = excl & 0xFFFFu, eq_excl = excl >> 16;
        const uint32_t ties_left = ties_taken - min(ties_taken, tie_base);
        const uint32_t tb = min(ties_left, eq_excl);                       // ties taken before this thread
        const uint32_t mine = min(ties_left - tb, (uint32_t)__popc(eq));   // ties this thread takes
        uint32_t sel = gt, e = eq;
        for (uint32_t m = 0; m < mine; ++m) {  // lowest `mine` equal keys
            sel |= e & (0u - e);
            e &= e - 1;
        }
        if (irow) {
            uint32_t pos = sel_base + gt_excl + tb, b = sel;
            while (b) {
                const int jj = __ffs(b) - 1;
                irow[pos++] = i0 + jj;
                b &= b - 1;
            }
        }
        if (mrow) {
#pragma unroll
            for (int jj = 0; jj < kItems; ++jj)
                if (jj < nv) mrow[i0 + jj] = (uint8_t)((sel >> jj) & 1u);
        }
        const uint32_t tot_gt = tot & 0xFFFFu, tot_eq = tot >> 16;
        sel_base += tot_gt + min(ties_left, tot_eq);
        tie_base += tot_eq;
    }
}

}  // namespace

void launch_topk_select(const float* scores, int64_t slices, int64_t n, int64_t k, uint8_t* mask, int32_t* idx,
                        cudaStream_t st) {
    if (slices == 0) return;
    if (select_stream_eligible(slices, n)) {
        launch_topk_select_stream(scores, slices, n, k, mask, idx, st);
        return;
    }
    // vector loads / stores only where the caller's pointers allow them (a view
    // with a storage offset, or a row inside a larger buffer, may not)
    const bool a16 = (reinterpret_cast<uintptr_t>(scores) & 15) == 0;
    const bool m8 = (reinterpret_cast<uintptr_t>(mask) & 7) == 0;
    // register-cached rows: the smallest CTA that holds the row (more CTAs per
    // SM and shorter block scans for short rows)
    // rows of <= 8192 still take 512 threads: fewer keys per thread shorten the
    // per-slice critical path (8k rows: 22 -> 19 us; one wave of slices either way)
    static const int min_kt = getenv("PKV_SELECT_MIN_THREADS") ? atoi(getenv("PKV_SELECT_MIN_THREADS")) : 512;
    if (n <= 256 * kItems * kCacheTiles && min_kt <= 256) {
        topk_select_cached_kernel<256><<<(unsigned)slices, 256, 0, st>>>(scores, n, k, mask, idx, a16);
    } else if (n <= 512 * kItems * kCacheTiles && min_kt <= 512) {
        topk_select_cached_kernel<512><<<(unsigned)slices, 512, 0, st>>>(scores, n, k, mask, idx, a16);
    } else if (n <= (int64_t)kThreads * kItems * kCacheTiles) {
        topk_select_cached_kernel<kThreads><<<(unsigned)slices, kThreads, 0, st>>>(scores, n, k, mask, idx, a16);
    } else {
        topk_select_kernel<float><<<(unsigned)slices, kThreads, 0, st>>>(scores, n, k, mask, idx, a16, m8);
    }
    check_launch("topk_select_kernel");
}

void launch_topk_select_f64(const double* scores, int64_t slices, int64_t n, int64_t k, uint8_t* mask, int32_t* idx,
                            cudaStream_t st) {
    if (slices == 0) return;
    const bool m8 = (reinterpret_cast<uintptr_t>(mask) & 7) == 0;
    topk_select_kernel<double><<<(unsigned)slices, kThreads, 0, st>>>(scores, n, k, mask, idx, false, m8);
    check_launch("topk_select_kernel<double>");
}

}  // namespace pkv
