// metrics.cu — the ranking metrics of the reference on the device (SURVEY.md
// §8(f) item 4; proj/src/pruning.cpp:58-195): per-slice Top-K overlap of two
// masks, the captured-mass ratio of a predicted mask against the scores' own
// Top-K (one CTA per slice, fp64 sums; the reference accumulates in fp64, only
// the summation order differs), and Spearman's rank correlation with average
// ranks on ties (pruning.cpp:122-186): a stable LSD radix sort per slice, tie
// runs by block scans, then Pearson of the ranks in exact integer arithmetic.
#include "internal.h"

namespace pkv {
namespace {

constexpr int kThreads = 512;

__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) red[w] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x < 32) {
        t = threadIdx.x < kThreads / 32 ? red[threadIdx.x] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    }
    __syncthreads();
    return t;  // valid in thread 0
}

// topk_overlap_per_slice (pruning.cpp:91-108): |a ∩ b| / k
__global__ void __launch_bounds__(kThreads) overlap_kernel(const uint8_t* __restrict__ a,
                                                           const uint8_t* __restrict__ b, int64_t n, int64_t k,
                                                           double* __restrict__ out) {
    __shared__ double red[kThreads / 32];
    const int64_t s = blockIdx.x;
    double c = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += kThreads) c += (a[s * n + i] && b[s * n + i]) ? 1.0 : 0.0;
    const double t = block_sum(c, red);
    if (threadIdx.x == 0) out[s] = t / (double)k;
}

// captured_mass_per_slice (pruning.cpp:58-80): Σ_pred y / Σ_topk(y) y (1 if 0)
__global__ void __launch_bounds__(kThreads) mass_kernel(const uint8_t* __restrict__ pred,
                                                        const uint8_t* __restrict__ oracle,
                                                        const float* __restrict__ y, int64_t n,
                                                        double* __restrict__ out) {
    __shared__ double red[kThreads / 32];
    const int64_t s = blockIdx.x;
    double cap = 0.0, orc = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += kThreads) {
        const double v = (double)y[s * n + i];
        cap += pred[s * n + i] ? v : 0.0;
        orc += oracle[s * n + i] ? v : 0.0;
    }
    const double tc = block_sum(cap, red);
    const double to = block_sum(orc, red);
    if (threadIdx.x == 0) out[s] = to > 0.0 ? tc / to : 1.0;
}

// ---------------------------------------------------------------- Spearman
// average_ranks (pruning.cpp:122-140) of one fp32 row: one CTA per row.
// Keys are the order-preserving u32 images of the values (−0 folded onto +0:
// the reference compares doubles with <, == so they tie). Stable LSD radix
// sort, 4-bit digits, 8 passes; thread t owns the contiguous strip
// [t·E, (t+1)·E) so per-(digit, thread) counters scanned digit-major give
// every element its stable destination. Ping-pong through global scratch (the
// rows stay L2-resident). Ranks are written doubled (2·rank = first + last +
// 2 of the tie run, an integer) at the element's original position.
constexpr int kRankThreads = 512;
constexpr int kDigits = 16;

__device__ __forceinline__ uint32_t order_key(float f) {
    uint32_t u = __float_as_uint(f);
    if ((u << 1) == 0) u = 0;  // -0.0 == +0.0
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

template <typename Op>
__device__ __forceinline__ int block_scan_incl(int v, int* red, Op op, int ident) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v = op(v, t);
    }
    if (lane == 31) red[w] = v;
    __syncthreads();
    if (w == 0) {
        int t = lane < kRankThreads / 32 ? red[lane] : ident;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t = op(t, u);
        }
        red[lane] = t;
    }
    __syncthreads();
    const int r = w > 0 ? op(v, red[w - 1]) : v;
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(kRankThreads) rank_kernel(const float* __restrict__ a, const float* __restrict__ b,
                                                            int64_t slices, int n, uint32_t* __restrict__ kbuf,
                                                            uint32_t* __restrict__ ibuf,
                                                            uint32_t* __restrict__ rank2) {
    __shared__ uint32_t cnt[kDigits][kRankThreads];
    __shared__ int red[32];
    const int64_t row = blockIdx.x;  // rows [0, slices) are a, [slices, 2 slices) are b
    const float* src = row < slices ? a + row * n : b + (row - slices) * n;
    const int t = threadIdx.x;
    const int E = (n + kRankThreads - 1) / kRankThreads;
    const int lo = min(t * E, n), hi = min(lo + E, n);
    const int64_t plane = 2 * slices * (int64_t)n;  // ping-pong planes
    uint32_t* k0 = kbuf + row * n;
    uint32_t* i0 = ibuf + row * n;
    for (int pass = 0; pass < 8; ++pass) {
        const int sh = 4 * pass;
        const uint32_t* kin = k0 + (pass & 1) * plane;
        const uint32_t* iin = i0 + (pass & 1) * plane;
        uint32_t* kout = k0 + ((pass + 1) & 1) * plane;
        uint32_t* iout = i0 + ((pass + 1) & 1) * plane;
#pragma unroll
        for (int d = 0; d < kDigits; ++d) cnt[d][t] = 0;
        for (int i = lo; i < hi; ++i) {
            const uint32_t key = pass == 0 ? order_key(src[i]) : kin[i];
            ++cnt[(key >> sh) & 15][t];
        }
        __syncthreads();
        // exclusive scan over the digit-major (digit, thread) order
        uint32_t* flat = &cnt[0][0];
        constexpr int kPer = kDigits * kRankThreads / kRankThreads;  // 16 counters per thread
        uint32_t loc[kPer], sum = 0;
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
            loc[j] = flat[t * kPer + j];
            sum += loc[j];
        }
        const int incl = block_scan_incl((int)sum, red, [](int x, int y) { return x + y; }, 0);
        uint32_t run = (uint32_t)incl - sum;
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
            flat[t * kPer + j] = run;
            run += loc[j];
        }
        __syncthreads();
        for (int i = lo; i < hi; ++i) {
            const uint32_t key = pass == 0 ? order_key(src[i]) : kin[i];
            const uint32_t pos = cnt[(key >> sh) & 15][t]++;
            kout[pos] = key;
            iout[pos] = pass == 0 ? (uint32_t)i : iin[i];
        }
        __threadfence_block();
        __syncthreads();
    }
    // 8 passes: the sorted row is back in plane 0. Tie runs: first = last head
    // at or before i, last = first tail at or after i.
    const uint32_t* ks = k0;
    const uint32_t* is = i0;
    int my_head = -1, my_tail = n;
    for (int i = hi - 1; i >= lo; --i)
        if (i == 0 || ks[i] != ks[i - 1]) {
            my_head = i;
            break;
        }
    for (int i = lo; i < hi; ++i)
        if (i == n - 1 || ks[i] != ks[i + 1]) {
            my_tail = i;
            break;
        }
    // carry-ins: the last run head in the strips before t, the first run
    // tail in the strips after t (suffix min = prefix min in mirrored order)
    __shared__ int carry[kRankThreads];
    const auto imax = [](int x, int y) { return max(x, y); };
    const auto imin = [](int x, int y) { return min(x, y); };
    carry[t] = block_scan_incl(my_head, red, imax, -1);
    __syncthreads();
    int first = t > 0 ? carry[t - 1] : -1;
    __syncthreads();
    carry[t] = my_tail;
    __syncthreads();
    const int mirrored = carry[kRankThreads - 1 - t];
    __syncthreads();
    carry[kRankThreads - 1 - t] = block_scan_incl(mirrored, red, imin, INT_MAX);
    __syncthreads();
    int last = t + 1 < kRankThreads ? carry[t + 1] : n;
    // backward sweep stores the run's last position, the forward sweep adds first + 2
    uint32_t* out = rank2 + row * n;
    for (int i = hi - 1; i >= lo; --i) {
        if (i == n - 1 || ks[i] != ks[i + 1]) last = i;
        out[is[i]] = (uint32_t)last;
    }
    for (int i = lo; i < hi; ++i) {
        if (i == 0 || ks[i] != ks[i - 1]) first = i;
        out[is[i]] += (uint32_t)first + 2u;
    }
}

// pearson of the doubled ranks (pruning.cpp:142-171), exactly: with integer
// ranks, S_xy = n·Σxy − Σx·Σy in 128-bit, and the one rounding is the final
// division. 1 when both rows are constant, 0 when one is.
__device__ __forceinline__ double u128_to_double(unsigned __int128 v) {
    return (double)(uint64_t)(v >> 64) * 18446744073709551616.0 + (double)(uint64_t)v;
}

__global__ void __launch_bounds__(kThreads) pearson_kernel(const uint32_t* __restrict__ rank2, int64_t slices, int n,
                                                           double* __restrict__ out) {
    __shared__ unsigned long long red[5][kThreads / 32];
    const int64_t s = blockIdx.x;
    const uint32_t* ra = rank2 + s * n;
    const uint32_t* rb = rank2 + (slices + s) * n;
    unsigned long long sa = 0, sb = 0, sab = 0, saa = 0, sbb = 0;
    for (int i = threadIdx.x; i < n; i += kThreads) {
        const unsigned long long x = ra[i], y = rb[i];
        sa += x;
        sb += y;
        sab += x * y;
        saa += x * x;
        sbb += y * y;
    }
    unsigned long long v[5] = {sa, sb, sab, saa, sbb};
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int j = 0; j < 5; ++j) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[j] += __shfl_xor_sync(0xffffffffu, v[j], o);
        if (lane == 0) red[j][w] = v[j];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t[5] = {0, 0, 0, 0, 0};
        for (int j = 0; j < 5; ++j)
            for (int q = 0; q < kThreads / 32; ++q) t[j] += red[j][q];
        using u128 = unsigned __int128;
        const u128 N = (u128)(unsigned)n;
        // n·Σx² ≥ (Σx)² (Cauchy–Schwarz), so the centred sums are non-negative
        const u128 Saa = N * t[3] - (u128)t[0] * t[0];
        const u128 Sbb = N * t[4] - (u128)t[1] * t[1];
        const u128 p = N * t[2], q = (u128)t[0] * t[1];
        double r;
        if (Saa == 0 && Sbb == 0) {
            r = 1.0;
        } else if (Saa == 0 || Sbb == 0) {
            r = 0.0;
        } else {
            const double sab_d = p >= q ? u128_to_double(p - q) : -u128_to_double(q - p);
            r = sab_d / sqrt(u128_to_double(Saa) * u128_to_double(Sbb));
        }
        out[s] = r;
    }
}

void launch_spearman(const float* a, const float* b, int64_t slices, int64_t n, void* scratch, double* out,
                     cudaStream_t st) {
    uint32_t* kb = static_cast<uint32_t*>(scratch);
    const int64_t plane = 2 * slices * n;
    uint32_t* ib = kb + 2 * plane;
    uint32_t* r2 = ib + 2 * plane;
    rank_kernel<<<(unsigned)(2 * slices), kRankThreads, 0, st>>>(a, b, slices, (int)n, kb, ib, r2);
    check_launch("rank_kernel");
    pearson_kernel<<<(unsigned)slices, kThreads, 0, st>>>(r2, slices, (int)n, out);
    check_launch("pearson_kernel");
}

size_t spearman_scratch_bytes(int64_t slices, int64_t n) { return (size_t)(2 * slices * n) * 4 * 5; }

}  // namespace
}  // namespace pkv

using namespace pkv;

extern "C" {

pkv_status pkv_topk_overlap(pkv_ctx ctx, const uint8_t* mask_a_dev, const uint8_t* mask_b_dev, int64_t slices,
                            int64_t n, int64_t k, double* per_slice_out_dev, void* stream) {
    return guard([&] {
        require_ctx(ctx);
        PKV_REQUIRE_SHAPE(slices > 0 && n > 0, "topk_overlap extents must be positive");
        PKV_REQUIRE_VALUE(k >= 1 && k <= n, "k must be in [1, n], got ", k);
        overlap_kernel<<<(unsigned)slices, kThreads, 0, static_cast<cudaStream_t>(stream)>>>(mask_a_dev, mask_b_dev, n,
                                                                                            k, per_slice_out_dev);
        check_launch("overlap_kernel");
        count_launch(ctx);
    });
}

pkv_status pkv_captured_mass(pkv_ctx ctx, const uint8_t* mask_pred_dev, const float* y_dev, int64_t slices,
                             int64_t n, int64_t k, double* per_slice_out_dev, void* stream) {
    return guard([&] {
        require_ctx(ctx);
        PKV_REQUIRE_SHAPE(slices > 0 && n > 0, "captured_mass extents must be positive");
        PKV_REQUIRE_VALUE(k >= 1 && k <= n, "k must be in [1, n], got ", k);
        auto st = static_cast<cudaStream_t>(stream);
        auto* om = static_cast<uint8_t*>(ctx->scratch_select.get(static_cast<size_t>(slices * n)));
        launch_topk_select(y_dev, slices, n, k, om, nullptr, st);  // the oracle mask: y's own Top-K
        mass_kernel<<<(unsigned)slices, kThreads, 0, st>>>(mask_pred_dev, om, y_dev, n, per_slice_out_dev);
        check_launch("mass_kernel");
        count_launch(ctx, 2);
    });
}

pkv_status pkv_spearman(pkv_ctx ctx, const float* a_dev, const float* b_dev, int64_t slices, int64_t n,
                        double* per_slice_out_dev, void* stream) {
    return guard([&] {
        require_ctx(ctx);
        PKV_REQUIRE_SHAPE(slices > 0, "spearman needs at least one slice");
        PKV_REQUIRE_VALUE(n >= 2, "spearman needs at least two tokens per slice");
        PKV_REQUIRE_VALUE(n <= (int64_t)INT32_MAX / 2 - 2, "spearman row too long: ", n);
        void* ws = ctx->scratch_metrics.get(spearman_scratch_bytes(slices, n));
        launch_spearman(a_dev, b_dev, slices, n, ws, per_slice_out_dev, static_cast<cudaStream_t>(stream));
        count_launch(ctx, 2);
    });
}

pkv_status pkv_slice_metrics(pkv_ctx ctx, const float* y_pred_dev, const float* y_true_dev, int64_t slices, int64_t n,
                             int64_t k, double* mass_out_dev, double* overlap_out_dev, double* spearman_out_dev,
                             void* stream) {
    return guard([&] {
        require_ctx(ctx);
        PKV_REQUIRE_SHAPE(slices > 0 && n >= 2, "slice_metrics needs slices > 0 and n >= 2");
        PKV_REQUIRE_VALUE(k >= 1 && k <= n, "k must be in [1, n], got ", k);
        PKV_REQUIRE_VALUE(n <= (int64_t)INT32_MAX / 2 - 2, "slice_metrics row too long: ", n);
        auto st = static_cast<cudaStream_t>(stream);
        const size_t masks = static_cast<size_t>(2 * slices * n);
        const size_t sp = spearman_scratch_bytes(slices, n);
        auto* ws = static_cast<uint8_t*>(ctx->scratch_metrics.get(sp + ((masks + 255) & ~size_t(255))));
        uint8_t* mp = ws + sp;
        uint8_t* mt = mp + slices * n;
        launch_topk_select(y_pred_dev, slices, n, k, mp, nullptr, st);  // topk_mask(y_pred, rho)
        launch_topk_select(y_true_dev, slices, n, k, mt, nullptr, st);  // topk_mask(y_true, rho)
        mass_kernel<<<(unsigned)slices, kThreads, 0, st>>>(mp, mt, y_true_dev, n, mass_out_dev);
        check_launch("mass_kernel");
        overlap_kernel<<<(unsigned)slices, kThreads, 0, st>>>(mp, mt, n, k, overlap_out_dev);
        check_launch("overlap_kernel");
        launch_spearman(y_pred_dev, y_true_dev, slices, n, ws, spearman_out_dev, st);
        count_launch(ctx, 6);
    });
}

}  // extern "C"
