// loss.cu — the reference's training loss suite on the device, forward and
// gradient w.r.t. the logits (proj/src/loss.cpp).
//
//   total = λ_bin·bin + λ_mse·mse + λ_fine·fine + λ_global·global + λ_cos·cos
//   (loss_total, loss.cpp:324-374; a zero λ removes its term exactly)
//
// Everything is computed in fp64 from fp32 logits / scores (the reference is
// fp64 throughout; with fp32-representable inputs only the summation order
// differs). The pair terms reproduce the reference's sampling exactly: the
// same xoshiro256** streams (rng.hpp:11-60) per slice, the partial
// Fisher–Yates over the Top-K pair list (loss.cpp:91-135) and Floyd's sampling
// over (Top-K × complement) pair ranks (loss.cpp:137-214), run by one thread
// per slice on an open-addressing table in shared memory (global scratch when
// max_pairs is too large for it). The gradient is the closed form of what the
// reference's tape computes (ops.cpp backward rules: relu'(0) = 0,
// clamp_min'(x) = [x > floor], softplus' = sigmoid).
//
// Kernel order on the caller's stream:
//   select ×(|ratios| + 1) → ymax → stats (bin, mse, cos partials per block)
//   → reduce → grad (elementwise part) → sample (per slice) → pair_reduce
//   → pair loss + grad scatter (fp64 atomics) → final reduce → D2H report.
#include <cmath>
#include <cstring>

#include "internal.h"

namespace pkv {
namespace {

constexpr int kT = 256;          // elementwise / reduction blocks
constexpr int kSampleT = 512;    // per-slice sampler
constexpr uint64_t kFineStream = 0x66696e65ull;
constexpr uint64_t kGlobalStream = 0x676c6f62ull;
constexpr double kNormFloor = 1e-12;
constexpr int kMaxRatios = 32;

struct DevCfg {
    double lambda[5];  // bin, mse, fine, global, cos
    double w_ratio[kMaxRatios];
    double w_sum;
    int n_ratios;
    double epsilon, mse_exponent, margin, clip_lo, clip_hi, pair_filter_frac;
    int64_t max_pairs;
};

// ------------------------------------------------------------- rng.hpp --
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
__device__ __forceinline__ uint64_t derive_seed(uint64_t base, uint64_t stream) {
    return splitmix64(base ^ splitmix64(stream + 1));
}
__device__ __forceinline__ uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

struct Xoshiro {
    uint64_t s[4];
    __device__ explicit Xoshiro(uint64_t seed) {
        uint64_t x = seed;
        for (auto& v : s) {
            x = splitmix64(x);
            v = x;
        }
    }
    __device__ uint64_t next() {
        const uint64_t r = rotl64(s[1] * 5, 7) * 9;
        const uint64_t t = s[1] << 17;
        s[2] ^= s[0];
        s[3] ^= s[1];
        s[1] ^= s[2];
        s[0] ^= s[3];
        s[2] ^= t;
        s[3] = rotl64(s[3], 45);
        return r;
    }
    __device__ uint64_t below(uint64_t n) {  // unbiased rejection (rng.hpp:49-58)
        const uint64_t threshold = (0 - n) % n;
        for (;;) {
            const uint64_t r = next();
            if (r >= threshold) return r % n;
        }
    }
};

// open addressing, key -1 = empty; cap is a power of two ≥ 2·entries
struct Table {
    int64_t* key;
    int64_t* val;  // null for a set
    int64_t mask;
    __device__ int64_t slot(int64_t k) const {
        uint64_t h = splitmix64((uint64_t)k) & (uint64_t)mask;
        while (key[h] != -1 && key[h] != k) h = (h + 1) & (uint64_t)mask;
        return (int64_t)h;
    }
};

__device__ __forceinline__ double sigmoid_d(double x) {  // ops.cpp:216-223
    return x >= 0.0 ? 1.0 / (1.0 + exp(-x)) : exp(x) / (1.0 + exp(x));
}
__device__ __forceinline__ double softplus_d(double x) {  // ops.cpp:242-248
    return fmax(x, 0.0) + log1p(exp(-fabs(x)));
}

__device__ __forceinline__ double block_sum_d(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    double t = 0.0;
    if (w == 0) {
        t = lane < nw ? red[lane] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    }
    return t;  // thread 0
}

__device__ __forceinline__ uint32_t fkey(float f) {
    const uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float unkey(uint32_t k) {
    return __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k);
}

// s_max = vmax(y) (loss.cpp:330), via the order-preserving key
__global__ void ymax_kernel(const float* __restrict__ y, int64_t numel, uint32_t* __restrict__ out) {
    uint32_t m = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < numel; i += (int64_t)gridDim.x * blockDim.x)
        m = max(m, fkey(y[i]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// per-block partials: [bin, mse, dot, pp, tt]; blocks never straddle a batch
// (blocks_per_batch blocks cover each batch of m elements)
__global__ void __launch_bounds__(kT) stats_kernel(const float* __restrict__ z, const float* __restrict__ y,
                                                    const uint8_t* __restrict__ masks, int64_t numel, int64_t m,
                                                    int blocks_per_batch, const uint32_t* __restrict__ smax_key,
                                                    DevCfg cfg, double* __restrict__ part) {
    __shared__ double red[32];
    const int64_t b = blockIdx.x / blocks_per_batch;
    const int64_t j0 = blockIdx.x % blocks_per_batch;
    const double smax = (double)unkey(*smax_key);
    double bin = 0.0, mse = 0.0, dot = 0.0, pp = 0.0, tt = 0.0;
    for (int64_t j = j0 * kT + threadIdx.x; j < m; j += (int64_t)blocks_per_batch * kT) {
        const int64_t e = b * m + j;
        const double zz = z[e], yy = y[e];
        double tw = 0.0;
        for (int r = 0; r < cfg.n_ratios; ++r) tw += masks[r * numel + e] ? cfg.w_ratio[r] : 0.0;
        bin += cfg.w_sum * softplus_d(zz) - zz * tw;
        const double mag = smax * sigmoid_d(zz);
        const double d = mag - yy;
        mse += pow(yy + cfg.epsilon, cfg.mse_exponent) * d * d;
        dot += mag * yy;
        pp += mag * mag;
        tt += yy * yy;
    }
    const double v[5] = {bin, mse, dot, pp, tt};
#pragma unroll
    for (int q = 0; q < 5; ++q) {
        const double s = block_sum_d(v[q], red);
        if (threadIdx.x == 0) part[(int64_t)blockIdx.x * 5 + q] = s;
    }
}

// scal: [0] bin, [1] mse, [2] cos (mean over batches), [3] floor hits,
//       then per batch b: [8 + 4b ...] = dot, Pn (clamped), Tn (clamped), sqrt(pp)
__global__ void __launch_bounds__(kT) stats_reduce_kernel(const double* __restrict__ part, int64_t batch,
                                                          int blocks_per_batch, int64_t numel,
                                                          double* __restrict__ scal) {
    if (threadIdx.x != 0) return;
    double bin = 0.0, mse = 0.0, cos_acc = 0.0, hits = 0.0;
    for (int64_t b = 0; b < batch; ++b) {
        double dot = 0.0, pp = 0.0, tt = 0.0;
        for (int j = 0; j < blocks_per_batch; ++j) {
            const double* p = part + (b * blocks_per_batch + j) * 5;
            bin += p[0];
            mse += p[1];
            dot += p[2];
            pp += p[3];
            tt += p[4];
        }
        const double tn = sqrt(tt), pn = sqrt(pp);
        hits += (tn < kNormFloor ? 1.0 : 0.0) + (pn < kNormFloor ? 1.0 : 0.0);
        const double Pn = fmax(pn, kNormFloor), Tn = fmax(tn, kNormFloor);
        cos_acc += 1.0 - dot / (Pn * Tn);
        scal[8 + 4 * b + 0] = dot;
        scal[8 + 4 * b + 1] = Pn;
        scal[8 + 4 * b + 2] = Tn;
        scal[8 + 4 * b + 3] = pn;
    }
    scal[0] = bin / (double)numel;
    scal[1] = mse / (double)numel;
    scal[2] = cos_acc / (double)batch;
    scal[3] = hits;
}

// elementwise gradient of λ_bin·bin + λ_mse·mse + λ_cos·cos (written, not added)
__global__ void __launch_bounds__(kT) grad_kernel(const float* __restrict__ z, const float* __restrict__ y,
                                                   const uint8_t* __restrict__ masks, int64_t numel, int64_t m,
                                                   int64_t batch, const uint32_t* __restrict__ smax_key, DevCfg cfg,
                                                   const double* __restrict__ scal, double* __restrict__ grad) {
    const double smax = (double)unkey(*smax_key);
    const double inv_n = 1.0 / (double)numel;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < numel; e += (int64_t)gridDim.x * blockDim.x) {
        const double zz = z[e], yy = y[e];
        const double sg = sigmoid_d(zz);
        const double dsg = sg * (1.0 - sg);
        double g = 0.0;
        if (cfg.lambda[0] != 0.0) {
            double tw = 0.0;
            for (int r = 0; r < cfg.n_ratios; ++r) tw += masks[r * numel + e] ? cfg.w_ratio[r] : 0.0;
            g += cfg.lambda[0] * inv_n * (cfg.w_sum * sg - tw);
        }
        const double mag = smax * sg;
        double gmag = 0.0;
        if (cfg.lambda[1] != 0.0) gmag += cfg.lambda[1] * inv_n * pow(yy + cfg.epsilon, cfg.mse_exponent) * 2.0 * (mag - yy);
        if (cfg.lambda[4] != 0.0) {
            const int64_t b = e / m;
            const double dot = scal[8 + 4 * b], Pn = scal[8 + 4 * b + 1], Tn = scal[8 + 4 * b + 2],
                         pn = scal[8 + 4 * b + 3];
            const double gc = -cfg.lambda[4] / (double)batch;  // d(1 - cos)/dcos, mean over batches
            double dp = yy / (Pn * Tn);
            if (pn > kNormFloor) dp -= dot / (Pn * Pn * Tn) * (mag / pn);
            gmag += gc * dp;
        }
        g += gmag * smax * dsg;
        grad[e] = g;
    }
}

// Rank p of the lexicographic pair list {(a, b): a < b < k} -> (a, b)
__device__ __forceinline__ void tri_unrank(int64_t p, int64_t k, int64_t& a, int64_t& b) {
    const double kk = 2.0 * (double)k - 1.0;
    int64_t x = (int64_t)floor((kk - sqrt(fmax(kk * kk - 8.0 * (double)p, 0.0))) * 0.5);
    if (x < 0) x = 0;
    auto S = [k](int64_t t) { return t * k - t * (t + 1) / 2; };
    while (x > 0 && S(x) > p) --x;
    while (S(x + 1) <= p) ++x;
    a = x;
    b = x + 1 + (p - S(x));
}

// j-th complement index (ascending) of the ascending Top-K list `top`
__device__ __forceinline__ int64_t rest_at(const int32_t* top, int64_t k, int64_t j) {
    int64_t lo = 0, hi = k;  // count of t with top[t] - t <= j
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((int64_t)top[mid] - mid <= j) lo = mid + 1;
        else hi = mid;
    }
    return j + lo;
}

struct SampleOut {
    int64_t* fine_i;   // [slices][M] global element index
    int64_t* fine_j;
    double* fine_d;
    int64_t* glob_i;
    int64_t* glob_j;
    double* glob_w;    // clamped weight
    int64_t* cand;     // [slices][M] candidate ranks
    int64_t* counts;   // [slices][4]: fine used, fine filtered, global used, global filtered
    double* fine_abs;  // [slices] Σ|d| over kept fine pairs
    int64_t* tab;      // global fallback tables [slices][2·cap] when not in smem
};

// Emit the kept candidates (ranks in cand[0..nc)) in order with a chunked
// block scan. mode 0: fine pairs (ranks into the Top-K pair list), 1: global.
__device__ void emit_pairs(int mode, const int64_t* cand, int64_t nc, const float* row, const int32_t* top,
                           int64_t k, int64_t n, int64_t base, double threshold, double rmin, double span,
                           const DevCfg& cfg, int64_t* oi, int64_t* oj, double* od, int64_t* used_out,
                           int64_t* filt_out, double* abs_out, int* scan) {
    int64_t used = 0, filtered = 0;
    double abs_acc = 0.0;
    const int64_t m = n - k;
    for (int64_t c0 = 0; c0 < nc; c0 += kSampleT) {
        const int64_t c = c0 + threadIdx.x;
        int keep = 0;
        int64_t ia = 0, ib = 0;
        double val = 0.0;
        if (c < nc) {
            const int64_t r = cand[c];
            if (mode == 0) {
                int64_t a, b;
                tri_unrank(r, k, a, b);
                ia = top[a];
                ib = top[b];
            } else {
                ia = top[r / m];
                ib = rest_at(top, k, r % m);
            }
            const double ya = row[ia], yb = row[ib];
            const double d = ya - yb;
            keep = !(fabs(d) < threshold);
            if (mode == 0) {
                val = d;
            } else {
                const double na = span > 0.0 ? (ya - rmin) / span : 0.0;
                const double nb = span > 0.0 ? (yb - rmin) / span : 0.0;
                val = fmin(fmax(1.0 + fabs(na - nb), cfg.clip_lo), cfg.clip_hi);
            }
        }
        // block exclusive scan of keep
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) scan[w] = __popc(bal);
        __syncthreads();
        if (w == 0) {
            int v = lane < kSampleT / 32 ? scan[lane] : 0;
            int inc = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += t;
            }
            if (lane < kSampleT / 32) scan[32 + lane] = inc - v;
            if (lane == 31) scan[64] = inc;
        }
        __syncthreads();
        const int pos = scan[32 + w] + __popc(bal & ((1u << lane) - 1));
        if (keep) {
            oi[used + pos] = base + ia;
            oj[used + pos] = base + ib;
            od[used + pos] = val;
            if (mode == 0) abs_acc += fabs(val);
        }
        const int nk = scan[64];
        const int64_t chunk = (nc - c0) < (int64_t)kSampleT ? (nc - c0) : (int64_t)kSampleT;
        used += nk;
        filtered += chunk - nk;
        __syncthreads();
    }
    // Σ|d| (fine): deterministic block sum
    __shared__ double red[32];
    const double s = block_sum_d(abs_acc, red);
    if (threadIdx.x == 0) {
        *used_out = used;
        *filt_out = filtered;
        if (abs_out) *abs_out = s;
    }
}

__global__ void __launch_bounds__(kSampleT) sample_kernel(const float* __restrict__ y, const int32_t* __restrict__ top_idx,
                                                          int64_t n, int64_t k, uint64_t seed, DevCfg cfg, int fine_on,
                                                          int global_on, int64_t cap, int tab_in_smem, SampleOut o) {
    extern __shared__ __align__(16) uint8_t dsm[];
    __shared__ int scan[72];
    __shared__ double red[32];
    const int64_t s = blockIdx.x;
    const float* row = y + s * n;
    const int32_t* top = top_idx + s * k;
    const int64_t M = cfg.max_pairs;
    int64_t* cand = o.cand + s * M;
    int64_t* tkey = tab_in_smem ? reinterpret_cast<int64_t*>(dsm) : o.tab + s * 2 * cap;
    int64_t* tval = tkey + cap;

    // row max / min (fp64 of fp32; exact)
    double mx = -INFINITY, mn = INFINITY;
    for (int64_t i = threadIdx.x; i < n; i += kSampleT) {
        mx = fmax(mx, (double)row[i]);
        mn = fmin(mn, (double)row[i]);
    }
#pragma unroll
    for (int q = 16; q > 0; q >>= 1) {
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, q));
        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, q));
    }
    if ((threadIdx.x & 31) == 0) {
        red[threadIdx.x >> 5] = mx;
        scan[threadIdx.x >> 5] = 0;
    }
    __syncthreads();
    double row_max = red[0];
    for (int q = 1; q < kSampleT / 32; ++q) row_max = fmax(row_max, red[q]);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mn;
    __syncthreads();
    double row_min = red[0];
    for (int q = 1; q < kSampleT / 32; ++q) row_min = fmin(row_min, red[q]);
    __syncthreads();
    const double threshold = cfg.pair_filter_frac * row_max;

    if (fine_on) {
        // ---- fine_pairs (loss.cpp:91-135)
        const int64_t C = k * (k - 1) / 2;
        int64_t nc;
        if (C > M) {
            for (int64_t i = threadIdx.x; i < cap; i += kSampleT) tkey[i] = -1;
            __syncthreads();
            if (threadIdx.x == 0) {
                Xoshiro rng(derive_seed(derive_seed(seed, kFineStream), (uint64_t)s));
                Table t{tkey, tval, cap - 1};
                for (int64_t i = 0; i < M; ++i) {
                    const int64_t j = i + (int64_t)rng.below((uint64_t)(C - i));
                    const int64_t si = t.slot(i);
                    const int64_t vi = tkey[si] == i ? tval[si] : i;
                    const int64_t sj = t.slot(j);
                    const int64_t vj = tkey[sj] == j ? tval[sj] : j;
                    cand[i] = vj;  // position i is final
                    tkey[sj] = j;  // position j now holds the old value at i
                    tval[sj] = vi;
                }
            }
            nc = M;
        } else {
            for (int64_t p = threadIdx.x; p < C; p += kSampleT) cand[p] = p;
            nc = C;
        }
        __syncthreads();
        emit_pairs(0, cand, nc, row, top, k, n, s * n, threshold, row_min, 0.0, cfg, o.fine_i + s * M,
                   o.fine_j + s * M, o.fine_d + s * M, &o.counts[s * 4 + 0], &o.counts[s * 4 + 1], &o.fine_abs[s],
                   scan);
        __syncthreads();
    }
    if (global_on && k < n) {
        // ---- global_pairs (loss.cpp:137-214)
        const int64_t total = k * (n - k);
        int64_t nc;
        if (total <= M) {
            for (int64_t p = threadIdx.x; p < total; p += kSampleT) cand[p] = p;
            nc = total;
        } else {
            for (int64_t i = threadIdx.x; i < cap; i += kSampleT) tkey[i] = -1;
            __syncthreads();
            if (threadIdx.x == 0) {
                Xoshiro rng(derive_seed(derive_seed(seed, kGlobalStream), (uint64_t)s));
                Table t{tkey, nullptr, cap - 1};
                int64_t cnt = 0;
                for (int64_t i = total - M; i < total; ++i) {
                    const int64_t r = (int64_t)rng.below((uint64_t)(i + 1));
                    const int64_t sr = t.slot(r);
                    const int64_t v = tkey[sr] == r ? i : r;
                    const int64_t sv = v == r ? sr : t.slot(v);
                    tkey[sv] = v;
                    cand[cnt++] = v;
                }
            }
            __syncthreads();
            // ascending rank order (loss.cpp:206-207): bitonic sort over the
            // next power of two, padded with INT64_MAX (in the table's space)
            int64_t P = 1;
            while (P < M) P <<= 1;
            int64_t* sb = tkey;  // the table is no longer needed; cap >= 2M >= P
            for (int64_t i = threadIdx.x; i < P; i += kSampleT) sb[i] = i < M ? cand[i] : INT64_MAX;
            __syncthreads();
            for (int64_t kk = 2; kk <= P; kk <<= 1)
                for (int64_t jj = kk >> 1; jj > 0; jj >>= 1) {
                    for (int64_t i = threadIdx.x; i < P; i += kSampleT) {
                        const int64_t l = i ^ jj;
                        if (l > i) {
                            const bool up = (i & kk) == 0;
                            const int64_t a = sb[i], b = sb[l];
                            if ((a > b) == up) {
                                sb[i] = b;
                                sb[l] = a;
                            }
                        }
                    }
                    __syncthreads();
                }
            for (int64_t i = threadIdx.x; i < M; i += kSampleT) cand[i] = sb[i];
            nc = M;
        }
        __syncthreads();
        emit_pairs(1, cand, nc, row, top, k, n, s * n, threshold, row_min, row_max - row_min, cfg, o.glob_i + s * M,
                   o.glob_j + s * M, o.glob_w + s * M, &o.counts[s * 4 + 2], &o.counts[s * 4 + 3], nullptr, scan);
    } else if (threadIdx.x == 0) {
        o.counts[s * 4 + 2] = 0;
        o.counts[s * 4 + 3] = 0;
    }
    if (!fine_on && threadIdx.x == 0) {
        o.counts[s * 4 + 0] = 0;
        o.counts[s * 4 + 1] = 0;
        o.fine_abs[s] = 0.0;
    }
}

// pscal: [0] fine used (as double), [1] fine filtered, [2] mean_abs,
//        [3] global used, [4] global filtered, [5] fine active (used >= 2 and mean_abs > 0)
__global__ void pair_reduce_kernel(const int64_t* __restrict__ counts, const double* __restrict__ fine_abs,
                                   int64_t slices, double* __restrict__ pscal, int64_t* __restrict__ ipscal) {
    if (threadIdx.x != 0) return;
    int64_t fu = 0, ff = 0, gu = 0, gf = 0;
    double ab = 0.0;
    for (int64_t s = 0; s < slices; ++s) {
        fu += counts[s * 4 + 0];
        ff += counts[s * 4 + 1];
        gu += counts[s * 4 + 2];
        gf += counts[s * 4 + 3];
        ab += fine_abs[s];
    }
    const double mean_abs = fu > 0 ? ab / (double)fu : 0.0;
    const bool fine_active = fu >= 2 && mean_abs > 0.0;
    pscal[2] = mean_abs;
    pscal[5] = fine_active ? 1.0 : 0.0;
    ipscal[0] = fine_active ? fu : 0;  // counts->used as the reference reports it
    ipscal[1] = ff;
    ipscal[2] = gu;
    ipscal[3] = gf;
}

// per-slice partial sums of the pair losses + gradient scatter
__global__ void __launch_bounds__(kT) pair_loss_kernel(const float* __restrict__ z, SampleOut o, int64_t M,
                                                        const double* __restrict__ pscal,
                                                        const int64_t* __restrict__ ipscal, DevCfg cfg,
                                                        double* __restrict__ part, double* __restrict__ grad) {
    __shared__ double red[32];
    const int64_t s = blockIdx.x;
    const bool fine_active = pscal[5] != 0.0;
    const double mean_abs = pscal[2];
    const int64_t fu = ipscal[0], gu = ipscal[2];
    double fsum = 0.0, gsum = 0.0;
    if (fine_active) {
        const int64_t n_s = o.counts[s * 4 + 0];
        const double gscale = cfg.lambda[2] / (double)fu;
        for (int64_t p = threadIdx.x; p < n_s; p += kT) {
            const int64_t i = o.fine_i[s * M + p], j = o.fine_j[s * M + p];
            const double d = o.fine_d[s * M + p];
            const double ns = d > 0.0 ? -1.0 : (d < 0.0 ? 1.0 : 0.0);
            const double w = fabs(d) / mean_abs;
            const double arg = ((double)z[i] - (double)z[j]) * ns;
            fsum += softplus_d(arg) * w;
            if (grad && cfg.lambda[2] != 0.0) {
                const double g = gscale * w * sigmoid_d(arg) * ns;
                atomicAdd(&grad[i], g);
                atomicAdd(&grad[j], -g);
            }
        }
    }
    if (gu > 0) {
        const int64_t n_s = o.counts[s * 4 + 2];
        const double gscale = cfg.lambda[3] / (double)gu;
        for (int64_t p = threadIdx.x; p < n_s; p += kT) {
            const int64_t i = o.glob_i[s * M + p], j = o.glob_j[s * M + p];
            const double w = o.glob_w[s * M + p];
            const double h = -((double)z[i] - (double)z[j]) + cfg.margin;
            gsum += (h > 0.0 ? h : 0.0) * w;
            if (grad && cfg.lambda[3] != 0.0 && h > 0.0) {
                atomicAdd(&grad[i], -gscale * w);
                atomicAdd(&grad[j], gscale * w);
            }
        }
    }
    const double a = block_sum_d(fsum, red);
    const double b = block_sum_d(gsum, red);
    if (threadIdx.x == 0) {
        part[s * 2 + 0] = a;
        part[s * 2 + 1] = b;
    }
}

__global__ void final_kernel(const double* __restrict__ part, int64_t slices, const double* __restrict__ pscal,
                             const int64_t* __restrict__ ipscal, double* __restrict__ scal) {
    if (threadIdx.x != 0) return;
    double f = 0.0, g = 0.0;
    for (int64_t s = 0; s < slices; ++s) {
        f += part[s * 2];
        g += part[s * 2 + 1];
    }
    scal[4] = pscal[5] != 0.0 ? f / (double)ipscal[0] : 0.0;
    scal[5] = ipscal[2] > 0 ? g / (double)ipscal[2] : 0.0;
}

}  // namespace
}  // namespace pkv

using namespace pkv;

extern "C" pkv_status pkv_loss_total(pkv_ctx ctx, const float* logits_dev, const float* y_dev, const int64_t* shape,
                                     int rank, const pkv_loss_config* c, uint64_t seed, pkv_loss_report* report,
                                     double* grad_dev, void* stream) {
    return guard([&] {
        require_ctx(ctx);
        PKV_REQUIRE_VALUE(c && report && shape, "null loss argument");
        PKV_REQUIRE_SHAPE(rank >= 1, "loss tensors need at least one axis");
        int64_t numel = 1;
        for (int i = 0; i < rank; ++i) {
            PKV_REQUIRE_SHAPE(shape[i] > 0, "loss extents must be positive");
            numel *= shape[i];
        }
        // LossConfig::validate (loss.cpp:29-44), same messages
        PKV_REQUIRE_VALUE(c->lambda_mse >= 0 && c->lambda_bin >= 0 && c->lambda_fine >= 0 && c->lambda_global >= 0 &&
                              c->lambda_cos >= 0,
                          "loss coefficients must be nonnegative");
        PKV_REQUIRE_VALUE(c->n_ratios > 0 && c->ratios, "ratio set must not be empty");
        PKV_REQUIRE_VALUE(c->n_ratios <= kMaxRatios, "at most ", kMaxRatios, " ratios supported on the device");
        for (int64_t i = 0; i < c->n_ratios; ++i)
            PKV_REQUIRE_VALUE(c->ratios[i] > 0.0 && c->ratios[i] <= 1.0, "ratio ", c->ratios[i], " out of (0, 1]");
        PKV_REQUIRE_VALUE(c->clip_lo <= c->clip_hi, "clip bounds out of order: [", c->clip_lo, ", ", c->clip_hi, "]");
        PKV_REQUIRE_VALUE(c->topk_ratio_for_rank > 0.0 && c->topk_ratio_for_rank <= 1.0,
                          "topk_ratio_for_rank out of (0, 1]");
        PKV_REQUIRE_VALUE(c->pair_filter_frac >= 0.0, "pair_filter_frac must be nonnegative");
        PKV_REQUIRE_VALUE(c->max_pairs > 0, "max_pairs must be positive");
        PKV_REQUIRE_VALUE(c->mse_exponent > 0.0 && c->epsilon >= 0.0, "mse weight parameters invalid");

        auto st = static_cast<cudaStream_t>(stream);
        const int64_t n = shape[rank - 1], slices = numel / n;
        const int64_t batch = rank >= 2 ? shape[0] : 1, m = numel / batch;
        const int64_t k = (int64_t)std::ceil(c->topk_ratio_for_rank * (double)n);
        const int64_t M = c->max_pairs;
        PKV_REQUIRE_VALUE(n <= (int64_t)INT32_MAX, "row too long");

        DevCfg dc{};
        dc.lambda[0] = c->lambda_bin;
        dc.lambda[1] = c->lambda_mse;
        dc.lambda[2] = c->lambda_fine;
        dc.lambda[3] = c->lambda_global;
        dc.lambda[4] = c->lambda_cos;
        double rmin = c->ratios[0];
        for (int64_t i = 1; i < c->n_ratios; ++i) rmin = std::min(rmin, c->ratios[i]);
        dc.n_ratios = (int)c->n_ratios;
        for (int64_t i = 0; i < c->n_ratios; ++i) {
            dc.w_ratio[i] = std::pow(rmin / c->ratios[i], c->gamma);
            dc.w_sum += dc.w_ratio[i];
        }
        dc.epsilon = c->epsilon;
        dc.mse_exponent = c->mse_exponent;
        dc.margin = c->margin;
        dc.clip_lo = c->clip_lo;
        dc.clip_hi = c->clip_hi;
        dc.pair_filter_frac = c->pair_filter_frac;
        dc.max_pairs = M;

        int64_t cap = 1;
        while (cap < 2 * M) cap <<= 1;
        const size_t smem_tab = (size_t)cap * 16;
        const bool tab_smem = smem_tab <= 160 * 1024;

        // ---- workspace
        const int bpb = (int)std::max<int64_t>(1, std::min<int64_t>((m + kT - 1) / kT, 4 * ctx->sm_count / batch + 1));
        auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
        const size_t masks_b = al((size_t)(c->n_ratios + 1) * numel);
        const size_t top_b = al((size_t)(slices * k) * 4);
        const size_t part_b = al((size_t)(batch * bpb) * 5 * 8);
        const size_t scal_b = al((size_t)(8 + 4 * batch) * 8);
        const size_t pairs_b = al((size_t)(slices * M) * 8);
        const size_t counts_b = al((size_t)slices * 4 * 8);
        const size_t tab_b = tab_smem ? 0 : al((size_t)(slices * 2 * cap) * 8);
        const size_t ppart_b = al((size_t)slices * 2 * 8);
        const size_t total_b = masks_b + top_b + part_b + scal_b + 7 * pairs_b + counts_b + al((size_t)slices * 8) +
                               tab_b + ppart_b + 256 + 256;
        uint8_t* w = static_cast<uint8_t*>(ctx->scratch_metrics.get(total_b));
        uint8_t* masks = w;
        w += masks_b;
        int32_t* top = reinterpret_cast<int32_t*>(w);
        w += top_b;
        double* part = reinterpret_cast<double*>(w);
        w += part_b;
        double* scal = reinterpret_cast<double*>(w);
        w += scal_b;
        SampleOut o{};
        o.fine_i = reinterpret_cast<int64_t*>(w);
        o.fine_j = reinterpret_cast<int64_t*>(w + pairs_b);
        o.fine_d = reinterpret_cast<double*>(w + 2 * pairs_b);
        o.glob_i = reinterpret_cast<int64_t*>(w + 3 * pairs_b);
        o.glob_j = reinterpret_cast<int64_t*>(w + 4 * pairs_b);
        o.glob_w = reinterpret_cast<double*>(w + 5 * pairs_b);
        o.cand = reinterpret_cast<int64_t*>(w + 6 * pairs_b);
        w += 7 * pairs_b;
        o.counts = reinterpret_cast<int64_t*>(w);
        w += counts_b;
        o.fine_abs = reinterpret_cast<double*>(w);
        w += al((size_t)slices * 8);
        o.tab = tab_smem ? nullptr : reinterpret_cast<int64_t*>(w);
        w += tab_b;
        double* ppart = reinterpret_cast<double*>(w);
        w += ppart_b;
        double* pscal = reinterpret_cast<double*>(w);   // 8 doubles
        int64_t* ipscal = reinterpret_cast<int64_t*>(w + 64);
        uint32_t* smax_key = reinterpret_cast<uint32_t*>(w + 128);

        // ---- masks: one per ratio (loss_bin) + the rank Top-K with indices
        for (int64_t r = 0; r < c->n_ratios; ++r) {
            const int64_t kr = (int64_t)std::ceil(c->ratios[r] * (double)n);
            launch_topk_select(y_dev, slices, n, kr, masks + r * numel, nullptr, st);
        }
        launch_topk_select(y_dev, slices, n, k, masks + c->n_ratios * numel, top, st);
        PKV_CUDA(cudaMemsetAsync(smax_key, 0, 4, st));
        ymax_kernel<<<4 * ctx->sm_count, kT, 0, st>>>(y_dev, numel, smax_key);
        check_launch("ymax_kernel");
        uint32_t smax_host_key = 0;
        PKV_CUDA(cudaMemcpyAsync(&smax_host_key, smax_key, 4, cudaMemcpyDeviceToHost, st));
        stats_kernel<<<(unsigned)(batch * bpb), kT, 0, st>>>(logits_dev, y_dev, masks, numel, m, bpb, smax_key, dc,
                                                             part);
        check_launch("stats_kernel");
        stats_reduce_kernel<<<1, 32, 0, st>>>(part, batch, bpb, numel, scal);
        check_launch("stats_reduce_kernel");
        PKV_CUDA(cudaStreamSynchronize(st));
        const uint32_t u = smax_host_key;
        float smax_f;
        {
            const uint32_t bits = (u & 0x80000000u) ? (u & 0x7FFFFFFFu) : ~u;
            std::memcpy(&smax_f, &bits, 4);
        }
        PKV_REQUIRE_VALUE(smax_f > 0.0f, "degenerate oracle: batch ground-truth maximum must be positive, got ",
                          (double)smax_f);
        if (grad_dev) {
            grad_kernel<<<8 * ctx->sm_count, kT, 0, st>>>(logits_dev, y_dev, masks, numel, m, batch, smax_key, dc, scal,
                                                          grad_dev);
            check_launch("grad_kernel");
        }
        const int fine_on = 1, global_on = 1;  // the terms are reported even when their λ is 0
        const size_t dyn = tab_smem ? smem_tab : 0;
        if (dyn > 48 * 1024)
            PKV_CUDA(cudaFuncSetAttribute(sample_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
        sample_kernel<<<(unsigned)slices, kSampleT, dyn, st>>>(y_dev, top, n, k, seed, dc, fine_on, global_on, cap,
                                                                tab_smem ? 1 : 0, o);
        check_launch("sample_kernel");
        pair_reduce_kernel<<<1, 32, 0, st>>>(o.counts, o.fine_abs, slices, pscal, ipscal);
        check_launch("pair_reduce_kernel");
        pair_loss_kernel<<<(unsigned)slices, kT, 0, st>>>(logits_dev, o, M, pscal, ipscal, dc, ppart, grad_dev);
        check_launch("pair_loss_kernel");
        final_kernel<<<1, 32, 0, st>>>(ppart, slices, pscal, ipscal, scal);
        check_launch("final_kernel");
        double hs[6];
        int64_t hi[4];
        PKV_CUDA(cudaMemcpyAsync(hs, scal, sizeof(hs), cudaMemcpyDeviceToHost, st));
        PKV_CUDA(cudaMemcpyAsync(hi, ipscal, sizeof(hi), cudaMemcpyDeviceToHost, st));
        PKV_CUDA(cudaStreamSynchronize(st));
        count_launch(ctx, (int)c->n_ratios + 9 + (grad_dev ? 1 : 0));

        pkv_loss_report& r = *report;
        r = pkv_loss_report{};
        r.s_max = (double)smax_f;
        r.bin = hs[0];
        r.mse = hs[1];
        r.cos = hs[2];
        r.cos_floor_hits = (int64_t)hs[3];
        r.fine = hs[4];
        r.global = hs[5];
        r.fine_used = hi[0];
        r.fine_filtered = hi[1];
        r.global_used = hi[2];
        r.global_filtered = hi[3];
        r.weighted_bin = c->lambda_bin * r.bin;
        r.weighted_mse = c->lambda_mse * r.mse;
        r.weighted_fine = c->lambda_fine * r.fine;
        r.weighted_global = c->lambda_global * r.global;
        r.weighted_cos = c->lambda_cos * r.cos;
        double total = 0.0;
        bool any = false;
        const double terms[5][2] = {{r.bin, c->lambda_bin},
                                    {r.mse, c->lambda_mse},
                                    {r.fine, c->lambda_fine},
                                    {r.global, c->lambda_global},
                                    {r.cos, c->lambda_cos}};
        for (const auto& t : terms) {
            if (t[1] == 0.0) continue;  // exact removal (loss.cpp:355-361)
            total = any ? total + t[0] * t[1] : t[0] * t[1];
            any = true;
        }
        r.total = any ? total : 0.0;
    });
}
