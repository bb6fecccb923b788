// select_stream.cu — streaming Top-K select with candidate compaction (the
// library's select for rows of >= 4096 scores outside 8k-16k, where it
// measures faster than select.cu's register-cached radix kernel).
//
// Same result as select.cu, bit for bit: the K best by
//   better(a,b) = v[a] > v[b] || (v[a] == v[b] && a < b)   (pruning.cpp:24-31)
// as ascending indices (apply_mask order, pruning.cpp:197-215) and/or the 0/1
// mask (topk_mask, pruning.cpp:37-56); -0.0 == +0.0.
//
// One 512-thread CTA per slice, two CTAs per SM, nothing cached in registers
// across passes:
//   pass 1 (HBM)  4096-bin shared histogram of the top 12 order-key bits,
//                 tiles of 8192 keys, two tiles in flight;
//   pass 2 (L2)   the keys of the bin holding the k-th key are appended to a
//                 shared candidate list (low 20 bits; warp-aggregated slots);
//                 a 12 + 8-bit radix select over the list gives the k-th key
//                 (a list longer than kCand — a row concentrated in one bin —
//                 falls back to two more histogram passes over the row);
//   pass 3 (L2)   per tile: greater / equal bits, one packed block scan, ties
//                 to the lowest indices; mask bytes, and the indices through
//                 a shared list (coalesced stores).
// select.cu's uncached kernel instead runs three full 12/12/8-bit digit passes
// over the row before its output pass.
#include <cstdlib>

#include "internal.h"

namespace pkv {
namespace {

constexpr int kT = 512;           // threads per slice CTA
constexpr int kPer = 16;          // consecutive keys per thread per tile
constexpr int kTile = kT * kPer;  // 8192 keys per tile
constexpr int kW = kT / 32;
constexpr int kBins = 4096;       // top digit: key bits [31:20]
constexpr int kCand = 8192;       // shared candidate list capacity
// dynamic shared memory: histogram | candidates | the tile's retained indices
constexpr int kSmem = (kBins + kCand + kTile) * 4;

// Monotone float -> uint32 map (select.cu's order_key): f + 0.0 turns -0.0
// into +0.0 (round-to-nearest, no FTZ), then negative values are inverted and
// non-negative ones get the top bit — FADD + SHF + LOP3.
__device__ __forceinline__ uint32_t order_key(float f) {
    const uint32_t u = __float_as_uint(__fadd_rn(f, 0.0f));
    return u ^ ((uint32_t)((int32_t)u >> 31) | 0x80000000u);
}

struct Tile {
    float v[kPer];
};

// The thread's kPer consecutive scores of tile t (float4 loads when the row
// allows); returns how many exist (callers mask by it).
__device__ __forceinline__ int load_tile(const float* __restrict__ row, int64_t n, int t, bool vec, Tile& x) {
    const int64_t i0 = (int64_t)t * kTile + (int64_t)threadIdx.x * kPer;
    const int64_t r = n - i0;
    const int nv = r <= 0 ? 0 : (r >= kPer ? kPer : (int)r);
    if (vec && nv == kPer) {
        const float4* p = reinterpret_cast<const float4*>(row + i0);
#pragma unroll
        for (int q = 0; q < kPer / 4; ++q) {
            const float4 a = p[q];
            x.v[4 * q + 0] = a.x;
            x.v[4 * q + 1] = a.y;
            x.v[4 * q + 2] = a.z;
            x.v[4 * q + 3] = a.w;
        }
    } else {
#pragma unroll
        for (int j = 0; j < kPer; ++j) x.v[j] = j < nv ? row[i0 + j] : 0.0f;
    }
    return nv;
}

// Block-wide exclusive scan of one uint32 per thread; total out.
__device__ __forceinline__ uint32_t scan_excl(uint32_t v, uint32_t* ws, uint32_t& total) {
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= (uint32_t)o) x += y;
    }
    if (lane == 31) ws[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < (uint32_t)kW ? ws[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= (uint32_t)o) w += y;
        }
        if (lane < (uint32_t)kW) ws[lane] = w;
    }
    __syncthreads();
    const uint32_t base = warp ? ws[warp - 1] : 0u;
    total = ws[kW - 1];
    __syncthreads();
    return base + x - v;
}

// Digit of a smem histogram of nb bins holding the kr-th largest (1-based),
// and the count above it (descending digit order).
__device__ __forceinline__ void find_digit(const uint32_t* hist, uint32_t nb, uint32_t kr, uint32_t* ws,
                                          uint32_t* s_digit, uint32_t* s_above) {
    const uint32_t bpt = nb > (uint32_t)kT ? nb / kT : 1u;  // bins per thread (8 or 1)
    const uint32_t tid = threadIdx.x;
    uint32_t c[8], sum = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const uint32_t bin = tid * bpt + j;
        c[j] = ((uint32_t)j < bpt && bin < nb) ? hist[nb - 1 - bin] : 0u;
        sum += c[j];
    }
    uint32_t total;
    const uint32_t excl = scan_excl(sum, ws, total);
    if (excl < kr && kr <= excl + sum) {
        uint32_t acc = excl;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (acc < kr && kr <= acc + c[j]) {
                *s_digit = nb - 1 - (tid * bpt + j);
                *s_above = acc;
            }
            acc += c[j];
        }
    }
    __syncthreads();
}

__device__ __forceinline__ void zero_bins(uint32_t* hist, uint32_t nb) {
    uint4* h4 = reinterpret_cast<uint4*>(hist);
    for (uint32_t i = threadIdx.x; i < nb / 4; i += kT) h4[i] = make_uint4(0, 0, 0, 0);
}

// Per-tile key work; kFull: all kPer keys of the thread exist (no masking).
template <bool kFull>
__device__ __forceinline__ void hist_tile(const Tile& x, int nv, uint32_t* hist) {
#pragma unroll
    for (int j = 0; j < kPer; ++j)
        if (kFull || j < nv) atomicAdd(&hist[order_key(x.v[j]) >> 20], 1u);
}
template <bool kFull>
__device__ __forceinline__ uint32_t cand_bits(const Tile& x, int nv, uint32_t b1) {
    uint32_t cb = 0;
#pragma unroll
    for (int j = 0; j < kPer; ++j)
        if ((kFull || j < nv) && (order_key(x.v[j]) >> 20) == b1) cb |= 1u << j;
    return cb;
}
template <bool kFull>
__device__ __forceinline__ void gteq_bits(const Tile& x, int nv, uint32_t kth, uint32_t& gt, uint32_t& eq) {
    gt = 0, eq = 0;
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
        const uint32_t key = order_key(x.v[j]);
        if ((kFull || j < nv) && key > kth) gt |= 1u << j;
        if ((kFull || j < nv) && key == kth) eq |= 1u << j;
    }
}

__global__ void __launch_bounds__(kT, 2)
    sel_stream_kernel(const float* __restrict__ scores, int64_t n, int64_t k, bool vec, uint8_t* __restrict__ mask,
                      bool mask16, int32_t* __restrict__ idx) {
    extern __shared__ __align__(16) uint32_t dsm[];
    uint32_t* hist = dsm;                                              // [kBins]
    uint32_t* cand = dsm + kBins;                                      // [kCand]
    int32_t* s_src = reinterpret_cast<int32_t*>(dsm + kBins + kCand);  // [kTile]
    __shared__ uint32_t sw[32];
    __shared__ uint32_t s_digit, s_above, s_cnt;
    const uint32_t tid = threadIdx.x, lane = tid & 31;
    const int64_t slice = blockIdx.x;
    const float* __restrict__ row = scores + slice * n;
    const int ntiles = (int)((n + kTile - 1) / kTile);

    // ---- pass 1: histogram of the top digit (two tiles in flight)
    zero_bins(hist, kBins);
    if (tid == 0) s_cnt = 0;
    __syncthreads();
    {
        Tile a, b;
        int na = load_tile(row, n, 0, vec, a), nb = 0;
        for (int t = 0; t < ntiles; t += 2) {
            if (t + 1 < ntiles) nb = load_tile(row, n, t + 1, vec, b);
            if (na == kPer) hist_tile<true>(a, na, hist);
            else hist_tile<false>(a, na, hist);
            if (t + 1 >= ntiles) break;
            if (t + 2 < ntiles) na = load_tile(row, n, t + 2, vec, a);
            if (nb == kPer) hist_tile<true>(b, nb, hist);
            else hist_tile<false>(b, nb, hist);
        }
    }
    __syncthreads();
    find_digit(hist, kBins, (uint32_t)k, sw, &s_digit, &s_above);
    const uint32_t b1 = s_digit;
    uint32_t kr = (uint32_t)k - s_above;  // rank of the k-th key inside bin b1

    // ---- pass 2: candidates of bin b1 (low 20 key bits) into shared memory
    auto add_cands = [&](const Tile& x, int nv) {
        const uint32_t cb = nv == kPer ? cand_bits<true>(x, nv, b1) : cand_bits<false>(x, nv, b1);
        // warp-aggregated slots: inclusive warp scan of the per-thread counts
        const uint32_t c = __popc(cb);
        uint32_t xs = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, xs, o);
            if (lane >= (uint32_t)o) xs += y;
        }
        uint32_t base = 0;
        if (lane == 31 && xs) base = atomicAdd(&s_cnt, xs);
        base = __shfl_sync(0xffffffffu, base, 31) + xs - c;
        if (cb) {
#pragma unroll
            for (int j = 0; j < kPer; ++j) {
                const uint32_t pos = base + __popc(cb & ((1u << j) - 1u));
                if (((cb >> j) & 1u) && pos < (uint32_t)kCand) cand[pos] = order_key(x.v[j]) & 0xFFFFFu;
            }
        }
    };
    {
        Tile a, b;
        int na = load_tile(row, n, 0, vec, a), nb = 0;
        for (int t = 0; t < ntiles; t += 2) {
            if (t + 1 < ntiles) nb = load_tile(row, n, t + 1, vec, b);
            add_cands(a, na);
            if (t + 1 >= ntiles) break;
            if (t + 2 < ntiles) na = load_tile(row, n, t + 2, vec, a);
            add_cands(b, nb);
        }
    }
    __syncthreads();
    const uint32_t nc = s_cnt;
    uint32_t kth_low;
    if (nc <= (uint32_t)kCand) {
        // radix select over the shared list: bits [19:8], then [7:0]
        zero_bins(hist, kBins);
        __syncthreads();
        for (uint32_t i = tid; i < nc; i += kT) atomicAdd(&hist[cand[i] >> 8], 1u);
        __syncthreads();
        find_digit(hist, kBins, kr, sw, &s_digit, &s_above);
        const uint32_t dA = s_digit;
        kr -= s_above;
        zero_bins(hist, 256);
        __syncthreads();
        for (uint32_t i = tid; i < nc; i += kT) {
            const uint32_t c = cand[i];
            if ((c >> 8) == dA) atomicAdd(&hist[c & 0xFFu], 1u);
        }
        __syncthreads();
        find_digit(hist, 256, kr, sw, &s_digit, &s_above);
        kth_low = (dA << 8) | s_digit;
        kr -= s_above;
    } else {
        // concentrated row: two more histogram passes over the row
        uint32_t prefix = b1 << 20, pmask = 0xFFF00000u;
#pragma unroll 1
        for (int pass = 0; pass < 2; ++pass) {
            const int shift = pass == 0 ? 8 : 0;
            const uint32_t nb = pass == 0 ? 4096u : 256u;
            zero_bins(hist, nb);
            __syncthreads();
            for (int t = 0; t < ntiles; ++t) {
                Tile cur;
                const int nv = load_tile(row, n, t, vec, cur);
#pragma unroll
                for (int j = 0; j < kPer; ++j) {
                    const uint32_t key = order_key(cur.v[j]);
                    if (j < nv && (key & pmask) == prefix) atomicAdd(&hist[(key >> shift) & (nb - 1)], 1u);
                }
            }
            __syncthreads();
            find_digit(hist, nb, kr, sw, &s_digit, &s_above);
            prefix |= s_digit << shift;
            pmask |= (nb - 1) << shift;
            kr -= s_above;
        }
        kth_low = prefix & 0xFFFFFu;
    }
    const uint32_t kth = (b1 << 20) | kth_low;
    const uint32_t ties = kr;  // keys equal to the k-th to keep, lowest indices first

    // ---- pass 3: ordered output per tile
    uint32_t sel_base = 0, tie_base = 0;
    for (int t = 0; t < ntiles; ++t) {
        Tile cur;
        const int nv = load_tile(row, n, t, vec, cur);
        const int64_t i0 = (int64_t)t * kTile + (int64_t)tid * kPer;
        uint32_t gt, eq;
        if (nv == kPer) gteq_bits<true>(cur, nv, kth, gt, eq);
        else gteq_bits<false>(cur, nv, kth, gt, eq);
        uint32_t tot;
        const uint32_t ex = scan_excl((uint32_t)__popc(gt) | ((uint32_t)__popc(eq) << 16), sw, tot);
        const uint32_t gt_excl = ex & 0xFFFFu, eq_excl = ex >> 16;
        const uint32_t ties_left = ties - min(ties, tie_base);
        const uint32_t tb = min(ties_left, eq_excl);
        const uint32_t mine = min(ties_left - tb, (uint32_t)__popc(eq));
        uint32_t sel = gt, e = eq;
        for (uint32_t m = 0; m < mine; ++m) {
            sel |= e & (0u - e);
            e &= e - 1;
        }
        if (mask) {
            uint8_t* mrow = mask + slice * n + i0;
            if (mask16 && nv == kPer) {
                uint4 w;
                uint32_t* wp = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint32_t s4 = sel >> (4 * q);
                    wp[q] = (s4 & 1u) | ((s4 >> 1) & 1u) << 8 | ((s4 >> 2) & 1u) << 16 | ((s4 >> 3) & 1u) << 24;
                }
                *reinterpret_cast<uint4*>(mrow) = w;
            } else {
#pragma unroll
                for (int j = 0; j < kPer; ++j)
                    if (j < nv) mrow[j] = (uint8_t)((sel >> j) & 1u);
            }
        }
        const uint32_t cnt = (tot & 0xFFFFu) + min(ties_left, tot >> 16);  // retained in this tile
        if (idx) {
            // the tile's retained indices, ascending, through shared memory:
            // output rows sel_base + [0, cnt) (coalesced index stores)
            uint32_t b = sel, p = gt_excl + tb;
            while (b) {
                s_src[p++] = (int32_t)(i0 + __ffs(b) - 1);
                b &= b - 1;
            }
            __syncthreads();
            int32_t* irow = idx + slice * k + sel_base;
            for (uint32_t j = tid; j < cnt; j += kT) irow[j] = s_src[j];
            __syncthreads();  // s_src is rewritten by the next tile
        }
        sel_base += cnt;
        tie_base += tot >> 16;
    }
}

}  // namespace

std::atomic<int> g_select_mode{-1};  // pkv_test_select_path

// Where the streaming kernel is the faster one (profiles/r02_sweep.json, 256
// slices: 8k 14.5 vs 15.9 us, 32k 37 vs 38.5, 64k 64 vs 93, 128k 166 vs 183;
// the register-cached radix kernel wins at 16k, 20.7 vs 22.7 us).
bool select_stream_eligible(int64_t slices, int64_t n) {
    if (slices <= 0 || n <= 0 || n >= (int64_t(1) << 31) || slices >= (int64_t(1) << 31)) return false;
    const int forced = g_select_mode.load();
    if (forced == 0) return false;
    if (forced == 1) return true;
    return n >= 4096 && !(n > 8192 && n <= 16384);
}

void launch_topk_select_stream(const float* scores, int64_t slices, int64_t n, int64_t k, uint8_t* mask,
                               int32_t* idx, cudaStream_t st) {
    if (slices == 0) return;
    static std::atomic<uint64_t> attr_done{0};
    if (first_on_device(attr_done))
        PKV_CUDA(cudaFuncSetAttribute(sel_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    const bool vec = (reinterpret_cast<uintptr_t>(scores) & 15) == 0 && (n & 3) == 0;
    const bool m16 = (reinterpret_cast<uintptr_t>(mask) & 15) == 0 && (n & 15) == 0;
    sel_stream_kernel<<<(unsigned)slices, kT, kSmem, st>>>(scores, n, k, vec, mask, m16, idx);
    check_launch("sel_stream_kernel");
}

}  // namespace pkv

extern "C" __attribute__((visibility("default"))) int pkv_test_select_path(int mode) {
    return pkv::g_select_mode.exchange(mode);
}
