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
#include <algorithm>
#include <cstdlib>

#include "internal.h"
#include "sm100.cuh"

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

// ============================================================ cluster select
// Rows of up to 8 x 32768 elements, one CTA cluster of C <= 8 CTAs per slice
// (C = ceil(n / 16384)), each CTA holding a contiguous chunk of the row's order
// keys in registers (32 per thread: 4 tiles x 8 consecutive items). The slice
// is read from HBM exactly once and every SM gets a share of every long slice.
//   pass 0   12-bit digit histogram per CTA, merged across the cluster over
//            DSMEM (CTA r sums bins [r·4096/C, (r+1)·4096/C) of all C
//            histograms), the k-th key's bucket found by a distributed scan;
//   extract  the keys in that bucket (typically < 1 % of the row) are appended
//            to the leader CTA's candidate list over DSMEM;
//   finish   the leader alone runs the 12- and 8-bit digit passes on the list
//            (shared-memory only) -> the k-th key and the number of its ties
//            to keep; if the list would overflow (heavily tied rows) every CTA
//            runs those two passes on its registers with the cluster merge;
//   output   per CTA the (greater, equal) counts of its chunk are exchanged
//            over DSMEM, then each thread writes its mask bytes and ascending
//            retained indices at their slice-global positions (ties to the
//            lowest indices across the whole cluster, pruning.cpp:24-31).
constexpr int kMaxCluster = 8;
constexpr int kClusterChunk = 16384;  // target elements per CTA
constexpr bool kAggregate = false;
constexpr int kMaxSamples = 4096;
constexpr int kCandCap = 8192;

__device__ __forceinline__ uint32_t ld_dsmem(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ void st_dsmem(uint32_t addr, uint32_t v) {
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

struct ClusterSmem {
    uint32_t hist[4096 + 32];  // + one discard bin per warp
    uint32_t parts[kMaxCluster];
    uint32_t ctot[kMaxCluster];
    uint32_t gtot[kMaxCluster];
    uint32_t etot[kMaxCluster];
    uint32_t res[4];
    uint32_t warp_sums[32];
    uint4 warp_sums4[32];
    uint32_t s_digit, s_above;
    uint32_t samp[kMaxSamples];  // leader: the row sample, sorted descending
    uint32_t cand[1];  // [cap] candidate keys (leader's copy is used)
};

template <int kT>
__device__ __forceinline__ void csync(int C) {
    if (C > 1) sm100::cluster_sync();
    else __syncthreads();
}

// Remote (or own) address of a shared word in CTA q.
__device__ __forceinline__ uint32_t peer(const void* p, uint32_t q) { return sm100::mapa_shared(sm100::smem_u32(p), q); }

template <int kT>
__device__ __forceinline__ uint4 block_excl_scan4(uint4 v, uint4* ws, uint4& total) {
    constexpr int kW = kT / 32;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint4 x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint4 y;
        y.x = __shfl_up_sync(0xffffffffu, x.x, o);
        y.y = __shfl_up_sync(0xffffffffu, x.y, o);
        y.z = __shfl_up_sync(0xffffffffu, x.z, o);
        y.w = __shfl_up_sync(0xffffffffu, x.w, o);
        if (lane >= (uint32_t)o) {
            x.x += y.x;
            x.y += y.y;
            x.z += y.z;
            x.w += y.w;
        }
    }
    if (lane == 31) ws[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint4 w = lane < (uint32_t)kW ? ws[lane] : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint4 y;
            y.x = __shfl_up_sync(0xffffffffu, w.x, o);
            y.y = __shfl_up_sync(0xffffffffu, w.y, o);
            y.z = __shfl_up_sync(0xffffffffu, w.z, o);
            y.w = __shfl_up_sync(0xffffffffu, w.w, o);
            if (lane >= (uint32_t)o) {
                w.x += y.x;
                w.y += y.y;
                w.z += y.z;
                w.w += y.w;
            }
        }
        if (lane < (uint32_t)kW) ws[lane] = w;
    }
    __syncthreads();
    const uint4 base = warp ? ws[warp - 1] : make_uint4(0, 0, 0, 0);
    total = ws[kW - 1];
    __syncthreads();
    return make_uint4(base.x + x.x - v.x, base.y + x.y - v.y, base.z + x.z - v.z, base.w + x.w - v.w);
}

// Finds the digit d (bins in `hist`, nb of them, descending digit order) whose
// bucket holds the kr-th largest: the CTA's bins [lo, lo + cnt) in descending
// position order are summed from `nsrc` CTAs' histograms. Returns through
// found / f_digit / f_above only in the thread that owns the bucket.
template <int kT>
__device__ __forceinline__ void scan_bins(ClusterSmem& S, int nb, int lo, int cnt, int nsrc, uint32_t kr_local,
                                          uint32_t& part_total, bool& found, uint32_t& f_digit, uint32_t& f_above) {
    const int tid = threadIdx.x;
    const int bpt = cnt >= kT ? cnt / kT : 1;  // positions per thread (cnt is a power of two)
    const int p0 = tid * bpt, p1 = min(cnt, p0 + bpt);
    auto bin_count = [&](int pos) {
        const int bin = nb - 1 - (lo + pos);
        uint32_t v = 0;
        for (int q = 0; q < nsrc; ++q) v += nsrc == 1 ? S.hist[bin] : ld_dsmem(peer(&S.hist[bin], (uint32_t)q));
        return v;
    };
    uint32_t sum = 0;
    for (int pos = p0; pos < p1; ++pos) sum += bin_count(pos);
    uint32_t total;
    const uint32_t excl = block_excl_scan<kT>(sum, S.warp_sums, total);
    part_total = total;
    found = false;
    if (excl < kr_local && kr_local <= excl + sum) {  // one thread: walk its bins again
        uint32_t acc = excl;
        for (int pos = p0; pos < p1; ++pos) {
            const uint32_t c = bin_count(pos);
            if (acc < kr_local && kr_local <= acc + c) {
                found = true;
                f_digit = (uint32_t)(nb - 1 - (lo + pos));
                f_above = acc;
                break;
            }
            acc += c;
        }
    }
}

// One digit pass over the register-cached keys with the cluster-wide merge.
template <int kT>
__device__ __forceinline__ void cluster_pass(ClusterSmem& S, const uint32_t (&key)[4][8], const uint32_t (&vm)[4],
                                             int ntiles, uint32_t prefix, uint32_t pmask, int shift, int bits,
                                             uint32_t& kr, uint32_t& digit, int C, uint32_t rank) {
    const int tid = threadIdx.x;
    const int nb = 1 << bits;
    const uint32_t dmask = (uint32_t)nb - 1, trash = 4096u + (uint32_t)(tid >> 5);
    for (int j = tid; j < nb; j += kT) S.hist[j] = 0;
    __syncthreads();
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        if (t >= ntiles) break;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const bool ok = ((vm[t] >> j) & 1u) && (key[t][j] & pmask) == prefix;
            const uint32_t bin = ok ? (key[t][j] >> shift) & dmask : trash;
            if (kAggregate) {
                // score rows concentrate in a few exponent buckets: one atomic
                // per distinct bin per warp instead of one per lane
                const uint32_t peers = __match_any_sync(0xffffffffu, bin);
                if ((threadIdx.x & 31) == (uint32_t)(__ffs(peers) - 1)) atomicAdd(&S.hist[bin], (uint32_t)__popc(peers));
            } else {
                atomicAdd(&S.hist[bin], 1u);
            }
        }
    }
    csync<kT>(C);
    // this CTA's part of the bins (descending positions [rank·B, (rank+1)·B))
    const int B = nb / C;
    uint32_t P, f_digit = 0, f_above = 0;
    bool found;
    // the part prefix A is not known yet: scan locally first, then locate
    scan_bins<kT>(S, nb, (int)rank * B, B, C, 0xFFFFFFFFu, P, found, f_digit, f_above);
    if (tid == 0)
        for (int q = 0; q < C; ++q) st_dsmem(peer(&S.parts[rank], (uint32_t)q), P);
    csync<kT>(C);
    uint32_t A = 0;
    for (uint32_t q = 0; q < rank; ++q) A += S.parts[q];
    if (A < kr && kr <= A + P) {  // this CTA's part holds the bucket: rescan with the rank known
        scan_bins<kT>(S, nb, (int)rank * B, B, C, kr - A, P, found, f_digit, f_above);
        if (found)
            for (int q = 0; q < C; ++q) {
                st_dsmem(peer(&S.res[0], (uint32_t)q), f_digit);
                st_dsmem(peer(&S.res[1], (uint32_t)q), A + f_above);
            }
    }
    csync<kT>(C);
    digit = S.res[0];
    kr -= S.res[1];
}

// Leader-local digit pass over the candidate list.
template <int kT>
__device__ __forceinline__ void list_pass(ClusterSmem& S, int ncand, uint32_t prefix, uint32_t pmask, int shift,
                                          int bits, uint32_t& kr, uint32_t& digit) {
    const int tid = threadIdx.x;
    const int nb = 1 << bits;
    const uint32_t dmask = (uint32_t)nb - 1;
    for (int j = tid; j < nb; j += kT) S.hist[j] = 0;
    __syncthreads();
    for (int i = tid; i < ncand; i += kT) {
        const uint32_t kk = S.cand[i];
        if ((kk & pmask) == prefix) atomicAdd(&S.hist[(kk >> shift) & dmask], 1u);
    }
    __syncthreads();
    uint32_t P, f_digit = 0, f_above = 0;
    bool found;
    scan_bins<kT>(S, nb, 0, nb, 1, kr, P, found, f_digit, f_above);
    if (found) {
        S.s_digit = f_digit;
        S.s_above = f_above;
    }
    __syncthreads();
    digit = S.s_digit;
    kr -= S.s_above;
    __syncthreads();
}

template <int kT>
__global__ void __launch_bounds__(kT, 1024 / kT)
    topk_select_cluster_kernel(const float* __restrict__ scores, int64_t n, int64_t k, int chunk, int cap,
                               uint8_t* __restrict__ mask, int32_t* __restrict__ idx, int C, bool aligned16,
                               bool mask8, int probe, int ns) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    ClusterSmem& S = *reinterpret_cast<ClusterSmem*>(smem_raw);
    const int tid = threadIdx.x;
    const uint32_t rank = C > 1 ? sm100::cluster_ctarank() : 0u;
    const int64_t slice = blockIdx.x / C;
    const int64_t c0 = (int64_t)rank * chunk;
    const int nn = (int)max((int64_t)0, min((int64_t)chunk, n - c0));
    const float* __restrict__ v = scores + slice * n + c0;
    const int ntiles = (nn + kT * 8 - 1) / (kT * 8);

    uint32_t key[4][8], vm[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        const int i0 = t * kT * 8 + tid * 8;
        const int r = nn - i0;
        const int nv = r <= 0 ? 0 : (r >= 8 ? 8 : r);
        vm[t] = (1u << nv) - 1u;
        if (aligned16 && nv == 8) {
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
            for (int j = 0; j < 8; ++j) key[t][j] = j < nv ? order_key(__ldcs(v + i0 + j)) : 0u;
        }
    }

    // timing probe (PKV_SELECT_PROBE): stop after a phase (all CTAs alike)
    if (probe == 1) {
        if (key[0][0] == 0xFFFFFFFFu && key[3][7] == 1u) S.res[0] = 1;  // keep the loads
        return;
    }
    uint32_t kth = 0, ties = 0;
    bool done = false;
    if (ns > 0) {
        // ---- sample bracket: NS keys sampled evenly from the whole row (the
        // slice is L2-resident now), sorted by the leader; [lo, hi] brackets the
        // k-th key's sample rank by +-3.5 sigma (binomial), so typically a few
        // % of the row falls inside. Exactness never depends on the sample:
        // a miss just takes the radix path below.
        const int spc = ns / C;
        const int64_t gstride = n / ns;
        const float* __restrict__ row = scores + slice * n;
        if (rank == 0)
            for (int j = tid; j < 4096; j += kT) S.hist[j] = 0;
        if (C == 1) __syncthreads();
        else csync<kT>(C);  // the leader's histogram is zeroed before anyone adds
        const uint32_t hist0 = sm100::smem_u32(&S.hist[0]);
        const uint32_t hist_leader = C > 1 ? sm100::mapa_shared(hist0, 0) : hist0;
#pragma unroll 4
        for (int i = tid; i < spc; i += kT) {
            const uint32_t kk = order_key(__ldg(row + ((int64_t)rank * spc + i) * gstride));
            const uint32_t addr = hist_leader + ((kk >> 20) << 2);
            if (C > 1) asm volatile("red.shared::cluster.add.u32 [%0], 1;" ::"r"(addr) : "memory");
            else atomicAdd(&S.hist[kk >> 20], 1u);
        }
        csync<kT>(C);
        if (rank == 0) {
            // the 12-bit buckets of the sample ranks r - m and r + m bound the
            // band (bucket granularity: concentrated rows give narrow bands)
            const double pr = (double)k / (double)n;
            const int r = (int)(pr * ns);
            const int m = (int)(3.5 * sqrt((double)ns * pr * (1.0 - pr))) + 4;
            uint32_t P, dh = 0, ah = 0, dl = 0, al = 0;
            bool fh, fl;
            const bool has_hi = r - m >= 1, has_lo = r + m <= ns;
            scan_bins<kT>(S, 4096, 0, 4096, 1, has_hi ? (uint32_t)(r - m) : 0u, P, fh, dh, ah);
            if (fh) S.s_digit = dh;
            scan_bins<kT>(S, 4096, 0, 4096, 1, has_lo ? (uint32_t)(r + m) : 0u, P, fl, dl, al);
            if (fl) S.s_above = dl;
            __syncthreads();
            if (tid == 0) {
                const uint32_t hi = has_hi ? ((S.s_digit + 1) << 20) - 1u : 0xFFFFFFFFu;
                const uint32_t lo = has_lo ? S.s_above << 20 : 0u;
                for (int q = 0; q < C; ++q) {
                    st_dsmem(peer(&S.res[0], (uint32_t)q), lo);
                    st_dsmem(peer(&S.res[1], (uint32_t)q), hi);
                }
            }
        }
        csync<kT>(C);
        const uint32_t lo = S.res[0], hi = S.res[1];
        // ---- band pass: count above hi, candidates in [lo, hi]
        uint32_t cm[4], gc = 0, cc = 0;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            cm[t] = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint32_t in = (vm[t] >> j) & 1u, kk = key[t][j];
                gc += in & (uint32_t)(kk > hi);
                cm[t] |= (in & (uint32_t)(kk >= lo) & (uint32_t)(kk <= hi)) << j;
            }
            cc += __popc(cm[t]);
        }
        uint32_t tot;
        const uint32_t ex = block_excl_scan<kT>(gc | (cc << 16), S.warp_sums, tot);
        if (tid == 0)
            for (int q = 0; q < C; ++q) {
                st_dsmem(peer(&S.gtot[rank], (uint32_t)q), tot & 0xFFFFu);
                st_dsmem(peer(&S.ctot[rank], (uint32_t)q), tot >> 16);
            }
        csync<kT>(C);
        uint32_t G = 0, Call = 0, before = 0;
        for (int q = 0; q < C; ++q) {
            G += S.gtot[q];
            Call += S.ctot[q];
            if ((uint32_t)q < rank) before += S.ctot[q];
        }
        if (probe == 2) return;
        if (G < (uint32_t)k && (uint32_t)k <= G + Call && Call <= (uint32_t)cap) {  // cluster-uniform
            uint32_t pos = before + (ex >> 16);
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                if (!cm[t]) continue;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    if ((cm[t] >> j) & 1u) {
                        if (C > 1) st_dsmem(peer(&S.cand[pos], 0), key[t][j]);
                        else S.cand[pos] = key[t][j];
                        ++pos;
                    }
                }
            }
            csync<kT>(C);
            if (rank == 0) {
                uint32_t kr = (uint32_t)k - G, d0, d1, d2;
                list_pass<kT>(S, (int)Call, 0u, 0u, 20, 12, kr, d0);
                list_pass<kT>(S, (int)Call, d0 << 20, 0xFFF00000u, 8, 12, kr, d1);
                list_pass<kT>(S, (int)Call, (d0 << 20) | (d1 << 8), 0xFFFFFF00u, 0, 8, kr, d2);
                if (tid == 0)
                    for (int q = 0; q < C; ++q) {
                        st_dsmem(peer(&S.res[2], (uint32_t)q), (d0 << 20) | (d1 << 8) | d2);
                        st_dsmem(peer(&S.res[3], (uint32_t)q), kr);
                    }
            }
            csync<kT>(C);
            kth = S.res[2];
            ties = S.res[3];
            done = true;
        }
    }
    if (!done) {
    // ---- pass 0: the k-th key's 12-bit bucket
    uint32_t kr = (uint32_t)k, b0;
    cluster_pass<kT>(S, key, vm, ntiles, 0u, 0u, 20, 12, kr, b0, C, rank);

    // ---- candidates (keys in bucket b0) -> the leader's list
    uint32_t cm[4], ccount = 0;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        cm[t] = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) cm[t] |= (uint32_t)(((vm[t] >> j) & 1u) && (key[t][j] >> 20) == b0) << j;
        ccount += __popc(cm[t]);
    }
    uint32_t ctotal;
    const uint32_t cex = block_excl_scan<kT>(ccount, S.warp_sums, ctotal);
    if (tid == 0)
        for (int q = 0; q < C; ++q) st_dsmem(peer(&S.ctot[rank], (uint32_t)q), ctotal);
    csync<kT>(C);
    uint32_t all = 0, before = 0;
    for (int q = 0; q < C; ++q) {
        all += S.ctot[q];
        if ((uint32_t)q < rank) before += S.ctot[q];
    }
    if (all <= (uint32_t)cap) {
        uint32_t pos = before + cex;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            if (!cm[t]) continue;
#pragma unroll
            for (int j = 0; j < 8; ++j) {  // static indices: the keys stay in registers
                if ((cm[t] >> j) & 1u) {
                    if (C > 1) st_dsmem(peer(&S.cand[pos], 0), key[t][j]);
                    else S.cand[pos] = key[t][j];
                    ++pos;
                }
            }
        }
        csync<kT>(C);
        if (rank == 0) {
            uint32_t d1, d2;
            const uint32_t p0 = b0 << 20;
            list_pass<kT>(S, (int)all, p0, 0xFFF00000u, 8, 12, kr, d1);
            list_pass<kT>(S, (int)all, p0 | (d1 << 8), 0xFFFFFF00u, 0, 8, kr, d2);
            if (tid == 0)
                for (int q = 0; q < C; ++q) {
                    st_dsmem(peer(&S.res[2], (uint32_t)q), p0 | (d1 << 8) | d2);
                    st_dsmem(peer(&S.res[3], (uint32_t)q), kr);
                }
        }
        csync<kT>(C);
        kth = S.res[2];
        ties = S.res[3];
    } else {  // heavily tied row: the two remaining digit passes over the registers
        uint32_t d1, d2;
        const uint32_t p0 = b0 << 20;
        cluster_pass<kT>(S, key, vm, ntiles, p0, 0xFFF00000u, 8, 12, kr, d1, C, rank);
        cluster_pass<kT>(S, key, vm, ntiles, p0 | (d1 << 8), 0xFFFFFF00u, 0, 8, kr, d2, C, rank);
        kth = p0 | (d1 << 8) | d2;
        ties = kr;
    }
    }  // radix path

    if (probe == 3) return;
    // ---- output: (greater, equal) bits per tile, slice-global positions
    // (the bits are recomputed in the write loop: fewer live registers)
    auto gt_eq = [&](int t, uint32_t& g, uint32_t& e) {
        g = e = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint32_t in = (vm[t] >> j) & 1u;
            g |= (in & (uint32_t)(key[t][j] > kth)) << j;
            e |= (in & (uint32_t)(key[t][j] == kth)) << j;
        }
    };
    uint4 cnt;
    uint32_t* cp = reinterpret_cast<uint32_t*>(&cnt);
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        uint32_t g, e;
        gt_eq(t, g, e);
        cp[t] = (uint32_t)__popc(g) | ((uint32_t)__popc(e) << 16);
    }
    uint4 tot;
    const uint4 ex = block_excl_scan4<kT>(cnt, S.warp_sums4, tot);
    const uint32_t* tp = reinterpret_cast<const uint32_t*>(&tot);
    const uint32_t* ep = reinterpret_cast<const uint32_t*>(&ex);
    uint32_t G = 0, E = 0;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        G += tp[t] & 0xFFFFu;
        E += tp[t] >> 16;
    }
    if (tid == 0)
        for (int q = 0; q < C; ++q) {
            st_dsmem(peer(&S.gtot[rank], (uint32_t)q), G);
            st_dsmem(peer(&S.etot[rank], (uint32_t)q), E);
        }
    csync<kT>(C);  // last cluster-wide exchange: no DSMEM access after this
    uint32_t gb = 0, eb = 0;
    for (uint32_t q = 0; q < rank; ++q) {
        gb += S.gtot[q];
        eb += S.etot[q];
    }
    uint8_t* __restrict__ mrow = mask ? mask + slice * n + c0 : nullptr;
    int32_t* __restrict__ irow = idx ? idx + slice * k : nullptr;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        if (t >= ntiles) break;
        const uint32_t gt_before = gb + (ep[t] & 0xFFFFu), eq_before = eb + (ep[t] >> 16);
        uint32_t sel, e;
        gt_eq(t, sel, e);
        const uint32_t tb = min(ties, eq_before);
        const uint32_t mine = min(ties - tb, (uint32_t)__popc(e));
        for (uint32_t m = 0; m < mine; ++m) {
            sel |= e & (0u - e);
            e &= e - 1;
        }
        const int i0 = t * kT * 8 + tid * 8;
        if (irow) {
            uint32_t pos = gt_before + tb, b = sel;
            while (b) {
                const int j = __ffs(b) - 1;
                b &= b - 1;
                irow[pos++] = (int32_t)(c0 + i0 + j);
            }
        }
        if (mrow) {
            if (mask8 && vm[t] == 0xFFu) {
                uint2 w;
                w.x = (sel & 1u) | ((sel >> 1) & 1u) << 8 | ((sel >> 2) & 1u) << 16 | ((sel >> 3) & 1u) << 24;
                w.y = ((sel >> 4) & 1u) | ((sel >> 5) & 1u) << 8 | ((sel >> 6) & 1u) << 16 | ((sel >> 7) & 1u) << 24;
                *reinterpret_cast<uint2*>(mrow + i0) = w;
            } else {
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if ((vm[t] >> j) & 1u) mrow[i0 + j] = (uint8_t)((sel >> j) & 1u);
            }
        }
        // the next tile's positions start after this tile's whole-CTA counts
        gb += tp[t] & 0xFFFFu;
        eb += tp[t] >> 16;
    }
}

template <int kT>
void launch_cluster(const float* scores, int64_t slices, int64_t n, int64_t k, int C, int chunk, uint8_t* mask,
                    int32_t* idx, bool a16, bool m8, cudaStream_t st) {
    const int cap = kCandCap;  // candidate keys (32 KB)
    const int ns = n >= 65536 ? 4096 : (n >= 4096 ? 2048 : 0);  // sample size (0: radix path only)
    const size_t smem = sizeof(ClusterSmem) + (size_t)cap * 4;
    auto kern = topk_select_cluster_kernel<kT>;
    static std::atomic<uint64_t> once{0};
    if (first_on_device(once))
        PKV_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(slices * C));
    cfg.blockDim = dim3(kT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    static const int probe = getenv("PKV_SELECT_PROBE") ? atoi(getenv("PKV_SELECT_PROBE")) : 0;
    PKV_CUDA(cudaLaunchKernelEx(&cfg, kern, scores, n, k, chunk, cap, mask, idx, C, a16, m8, probe, ns));
}

}  // namespace

void launch_topk_select(const float* scores, int64_t slices, int64_t n, int64_t k, uint8_t* mask, int32_t* idx,
                        cudaStream_t st) {
    if (slices == 0) return;
    // vector loads / stores only where the caller's pointers allow them (a view
    // with a storage offset, or a row inside a larger buffer, may not)
    const bool a16 = (reinterpret_cast<uintptr_t>(scores) & 15) == 0;
    const bool m8 = (reinterpret_cast<uintptr_t>(mask) & 7) == 0;
    // register-cached rows: the smallest CTA that holds the row (more CTAs per
    // SM and shorter block scans for short rows)
    // rows of <= 8192 still take 512 threads: fewer keys per thread shorten the
    // per-slice critical path (8k rows: 22 -> 19 us; one wave of slices either way)
    static const int min_kt = getenv("PKV_SELECT_MIN_THREADS") ? atoi(getenv("PKV_SELECT_MIN_THREADS")) : 512;
    static const bool legacy = getenv("PKV_SELECT_LEGACY") != nullptr;  // A/B switch: one CTA per slice
    if (!legacy && n <= (int64_t)kMaxCluster * 32768) {
        int C = 1;  // power of two (the 4096 pass-0 bins split evenly)
        while (C < kMaxCluster && (int64_t)C * kClusterChunk < n) C *= 2;
        const int chunk = (int)((((n + C - 1) / C) + 7) / 8 * 8);
        const bool a16c = a16 && (n & 3) == 0;
        const bool m8c = m8 && (n & 7) == 0;
        if (chunk <= 256 * 32) launch_cluster<256>(scores, slices, n, k, C, chunk, mask, idx, a16c, m8c, st);
        else if (chunk <= 512 * 32) launch_cluster<512>(scores, slices, n, k, C, chunk, mask, idx, a16c, m8c, st);
        else launch_cluster<1024>(scores, slices, n, k, C, chunk, mask, idx, a16c, m8c, st);
        check_launch("topk_select_cluster_kernel");
        return;
    }
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
