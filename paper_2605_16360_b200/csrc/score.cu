// score.cu — proxy reconstruction-importance scoring (SPEC.md:423-431
// accumulate_attention; X definition; north-star max-pool), flash
// style on tcgen05 so the N_q×N_k attention matrix is never materialised:
//
//   pass 1 (score_lse_kernel):  S = Q·Kᵀ (M = 128 queries, N = 256 keys) into
//     double-buffered TMEM; 16 softmax warps (4 column segments x 4 TMEM lane
//     quadrants) sum exp2(c·s − m) per row segment in registers against a
//     fixed per-row reference m = ⌈c·|q|·max|k|⌉ + 1 (Cauchy–Schwarz: no
//     running max), merged through smem at the end; 10 of 32 exponential
//     pairs are a degree-3 polynomial on the FMA pipe to offload MUFU
//     (FA4-style), with m folded into the range reduction; writes lse[q] and
//     the bf16 triple (hi, mid, lo) of λ_q = √d·lse_q. A row whose largest
//     term falls below 2^-40 flags its tile; the exact running-max variant of
//     the kernel then redoes only the flagged tiles.
//   pass 2 (score_pool_kernel): S' = K·Qᵀ − λ (two M = 128 key blocks = 256
//     keys per CTA, N = 128 queries per tile), the −λ_q column folded into the
//     MMA as 3 extra K columns (K_aug = 1, Q_aug = −(hi, mid, lo)); one thread
//     per key row reduces over queries in registers: max mode = one FMNMX3 per
//     2 elements (max_q P = exp2(c·max_q S'), c = log2(e)/√d); sum mode =
//     exp2 + FADD per element.
// GQA: pass 2 walks the queries of all heads of a KV head's group.
//
// q bf16 [L, Hq, Nq, d], k bf16 [L, Hkv, Nk, d]; d ∈ {64, 128}.
#include <cstdlib>

#include <mutex>

#include "lse_chunk.cuh"
#include "score.cuh"
#include "sm100.cuh"

namespace pkv {
namespace {

using namespace sm100;

constexpr float kLog2e = 1.4426950408889634f;

template <int D>
struct P1 {
    static constexpr int kBQ = 128, kBK = 256;
    static constexpr int kSegs = 4;  // column segments per tile (one warp per segment and TMEM lane quadrant)
    static constexpr int kSegCols = kBK / kSegs;
    static constexpr int kSoftWarps = 4 * kSegs;
    static constexpr int kThreads = 64 + 32 * kSoftWarps;  // warp 0 TMA, warp 1 TMEM+MMA
    static constexpr int kPanels = D / 64;
    static constexpr int kQBytes = kBQ * D * 2;
    static constexpr int kKBytes = kBK * D * 2;
    static constexpr int kStages = D == 64 ? 3 : 2;
    static constexpr int kSmem = 1024 + kQBytes + kStages * kKBytes + 256 + kSegs * kBQ * 8;
};

template <int D>
struct P2 {
    static constexpr int kBK = 128, kBlocks = 2, kBQ = 128;
    static constexpr int kThreads = 128 + 32 * 4 * kBlocks;
    static constexpr int kPanels = D / 64;
    static constexpr int kKBytes = kBK * D * 2;  // per key block
    static constexpr int kAugA = 2 * kBK * 16;  // [ones pattern | zeros], 16 B rows
    static constexpr int kQBytes = kBQ * D * 2;
    static constexpr int kLBytes = kBQ * 16;
    static constexpr int kStageBytes = kQBytes + kLBytes;
    static constexpr int kStages = D == 64 ? 4 : 3;
    static constexpr int kSmem = 1024 + kBlocks * kKBytes + kAugA + kStages * kStageBytes + 256;
};

// No-swizzle K-major descriptor: 8-row core matrices of 16 B rows (128 B
// contiguous), SBO between 8-row groups, LBO between the two 8-element K halves.
__device__ __forceinline__ uint64_t desc_noswz(const void* p, uint32_t lbo, uint32_t sbo) {
    const uint64_t addr = smem_u32(p);
    uint64_t d = 0;
    d |= (addr >> 4) & 0x3FFFull;
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= 1ull << 46;  // version, layout type 0 = SWIZZLE_NONE
    return d;
}

__device__ __forceinline__ void write_lam(__nv_bfloat16* dst, float lam) {
    const __nv_bfloat16 hi = __float2bfloat16_rn(lam);
    const float r1 = lam - __bfloat162float(hi);
    const __nv_bfloat16 mid = __float2bfloat16_rn(r1);
    const __nv_bfloat16 lo = __float2bfloat16_rn(r1 - __bfloat162float(mid));
    __align__(16) __nv_bfloat16 v[8];
    v[0] = __hneg(hi);
    v[1] = __hneg(mid);
    v[2] = __hneg(lo);
#pragma unroll
    for (int u = 3; u < 8; ++u) v[u] = __float2bfloat16_rn(0.0f);
    *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(v);
}

// One 64-column chunk of a softmax row segment: online (max, Σexp2) update.
// valid = number of leading columns that count (masked tail / causal diagonal).
template <int kPolyPairs>
__device__ __forceinline__ void lse_chunk(const uint32_t (&ra)[32], const uint32_t (&rb)[32], int valid, float c_log2,
                                          float& m, float& lsum) {
    float v[64];
#pragma unroll
    for (int u = 0; u < 32; ++u) {
        v[u] = __uint_as_float(ra[u]);
        v[32 + u] = __uint_as_float(rb[u]);
    }
    const bool masked = __any_sync(0xffffffffu, valid < 64);  // warp-uniform: tail / diagonal tiles
    if (masked) {
#pragma unroll
        for (int u = 0; u < 64; ++u) v[u] = (u < valid) ? v[u] : -INFINITY;
    }
    // max as a tree (8 independent FMNMX3 chains) to keep the dependency short
    float mt[8];
#pragma unroll
    for (int t8 = 0; t8 < 8; ++t8) mt[t8] = fmaxf(v[t8], v[t8 + 8]);
#pragma unroll
    for (int u = 16; u < 64; u += 16)
#pragma unroll
        for (int t8 = 0; t8 < 8; ++t8) mt[t8] = max3f(mt[t8], v[u + t8], v[u + t8 + 8]);
    const float cm = max3f(max3f(mt[0], mt[1], mt[2]), max3f(mt[3], mt[4], mt[5]), fmaxf(mt[6], mt[7]));
    // integer running max (log2 domain): lets the polynomial path fold the
    // offset into its range reduction (ex2_poly2_fused)
    const float mn = fmaxf(m, ceilf(cm * c_log2));
    if (mn == -INFINITY) return;
    // packed fp32x2: FFMA2 for the arguments, FADD2 for the sums; of the 32
    // pairs, kPolyPairs go through the FMA-pipe polynomial, spread evenly
    // (Bresenham), the rest through MUFU. Masked chunks take the MUFU path only.
    const uint64_t cc = pack2(c_log2, c_log2), nm = pack2(-mn, -mn);
    const uint64_t mp = pack2(12582912.0f - mn, 12582912.0f - mn);
    uint64_t acc0 = pack2(0.0f, 0.0f), acc1 = acc0;
    if (!masked) {
#pragma unroll
        for (int pr = 0; pr < 32; ++pr) {
            const uint64_t s2 = pack2(v[2 * pr], v[2 * pr + 1]);
            uint64_t e;
            if (((pr + 1) * kPolyPairs) / 32 != (pr * kPolyPairs) / 32) {
                e = ex2_poly2_fused(s2, cc, mp);
            } else {
                const float2 x = unpack2(ffma2(s2, cc, nm));
                e = pack2(ex2(x.x), ex2(x.y));
            }
            if (pr & 1) acc1 = fadd2(acc1, e);
            else acc0 = fadd2(acc0, e);
        }
    } else {
#pragma unroll
        for (int pr = 0; pr < 32; ++pr) {
            const float2 x = unpack2(ffma2(pack2(v[2 * pr], v[2 * pr + 1]), cc, nm));
            const uint64_t e = pack2(ex2(x.x), ex2(x.y));
            if (pr & 1) acc1 = fadd2(acc1, e);
            else acc0 = fadd2(acc0, e);
        }
    }
    const float2 ssum = unpack2(fadd2(acc0, acc1));
    lsum = lsum * ex2(m - mn) + (ssum.x + ssum.y);
    m = mn;
}

// The same over a fixed per-row reference m (an upper bound of every score of
// the row, so no running max, no max tree and no rescale): all exponents are
// <= 0 and the sum keeps full relative precision as long as the row's largest
// term is not far below 1 (checked by the caller).
// max_k |k| per (layer, KV head) slab: the Cauchy–Schwarz score bound's K side
__global__ void kmax_norm_kernel(const __nv_bfloat16* __restrict__ k, int64_t rows, int d, float* __restrict__ out) {
    const int64_t slab = blockIdx.x;
    const __nv_bfloat16* kp = k + slab * rows * d;
    float mx = 0.0f;
    for (int64_t r = threadIdx.x; r < rows; r += blockDim.x) {
        const uint4* row = reinterpret_cast<const uint4*>(kp + r * d);
        float s = 0.0f;
        for (int c = 0; c < d / 8; ++c) {
            const uint4 u = __ldg(row + c);
            const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float a = __uint_as_float(w[i] << 16), b = __uint_as_float(w[i] & 0xFFFF0000u);
                s = fmaf(a, a, fmaf(b, b, s));
            }
        }
        mx = fmaxf(mx, s);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    __shared__ float red[32];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        float m = 0.0f;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = fmaxf(m, red[w]);
        out[slab] = sqrtf(m);
    }
}

// ---------------------------------------------------------------- pass 1 --
// kFixed: rows use the fixed Cauchy–Schwarz reference ceil(c·|q|·max|k|) + 1
// (kmax) and flag their query tile when its largest term falls below 2^-40
// (tile_flags; the exact kernel then redoes those tiles). !kFixed with
// tile_flags: exact running-max kernel restricted to the flagged tiles.
template <int D, int kPolyPairs, bool kFixed>
__global__ void __launch_bounds__(P1<D>::kThreads, 1)
    score_lse_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk, int Hq, int Hkv,
                     int Nq, int Nk, int causal, float c_log2, float* __restrict__ lse_out,
                     __nv_bfloat16* __restrict__ lam_out, const float* __restrict__ kmax,
                     uint32_t* __restrict__ tile_flags) {
    using C = P1<D>;
    const int64_t tile_id = ((int64_t)blockIdx.z * Hq + blockIdx.y) * gridDim.x + blockIdx.x;
    if (!kFixed && tile_flags != nullptr && tile_flags[tile_id] == 0) return;  // CTA-uniform, before any barrier
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = smem;
    uint8_t* sK = sQ + C::kQBytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sK + C::kStages * C::kKBytes);
    uint64_t* bar_q = bars;
    uint64_t* k_full = bars + 1;
    uint64_t* k_empty = k_full + C::kStages;
    uint64_t* s_full = k_empty + C::kStages;
    uint64_t* s_empty = s_full + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_empty + 2);
    float2* part = reinterpret_cast<float2*>(reinterpret_cast<uint8_t*>(bars) + 256);  // [segs][128] (m, l)

    const uint32_t warp = warp_id(), lane = lane_id();
    const int q0 = blockIdx.x * C::kBQ, h = blockIdx.y, l = blockIdx.z;
    const int g = Hq / Hkv;
    const int qslab = l * Hq + h, kslab = l * Hkv + h / g;
    const int off = Nk - Nq;  // causal: key j allowed iff j <= q + off
    int n_kv = (Nk + C::kBK - 1) / C::kBK;
    if (causal) {
        const int last_key = q0 + C::kBQ - 1 + off;
        const int t = last_key < 0 ? 0 : last_key / C::kBK + 1;
        n_kv = t < n_kv ? t : n_kv;
    }

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tq);
        tma_prefetch(&tk);
        mbar_init(bar_q, 1);
        for (int s = 0; s < C::kStages; ++s) {
            mbar_init(&k_full[s], 1);
            mbar_init(&k_empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&s_full[s], 1);
            mbar_init(&s_empty[s], C::kSoftWarps);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (elect_one() && n_kv > 0) {
            mbar_arrive_expect_tx(bar_q, C::kQBytes);
            for (int p = 0; p < C::kPanels; ++p) tma_load_3d(sQ + p * (C::kBQ * 128), &tq, bar_q, p * 64, q0, qslab);
            for (int j = 0; j < n_kv; ++j) {
                const int st = j % C::kStages;
                mbar_wait(&k_empty[st], ((j / C::kStages) & 1) ^ 1);
                mbar_arrive_expect_tx(&k_full[st], C::kKBytes);
                uint8_t* dst = sK + st * C::kKBytes;
                for (int p = 0; p < C::kPanels; ++p)
                    tma_load_3d(dst + p * (C::kBK * 128), &tk, &k_full[st], p * 64, j * C::kBK, kslab);
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t idesc = idesc_f16(C::kBQ, C::kBK, 1);
        if (n_kv > 0) mbar_wait(bar_q, 0);
        for (int j = 0; j < n_kv; ++j) {
            const int st = j % C::kStages, sb = j & 1;
            mbar_wait(&k_full[st], (j / C::kStages) & 1);
            mbar_wait(&s_empty[sb], ((j >> 1) & 1) ^ 1);
            tc_fence_after();
            if (elect_one()) {
#pragma unroll
                for (int p = 0; p < C::kPanels; ++p) {
                    const uint64_t a = desc_sw128(sQ + p * (C::kBQ * 128));
                    const uint64_t b = desc_sw128(sK + st * C::kKBytes + p * (C::kBK * 128));
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        mma_f16_ss(tmem + sb * C::kBK, a + kk * 2, b + kk * 2, idesc, (p | kk) != 0);
                }
                mma_commit(&s_full[sb]);
                mma_commit(&k_empty[st]);
            }
            __syncwarp();
        }
    } else {
        const uint32_t quad = warp & 3;
        const int seg = (warp - 2) >> 2;  // column segment of the 256-key tile (quad = warp % 4)
        const int r = quad * 32 + lane;
        const int q = q0 + r;
        const int kmax_k = causal ? (q + off + 1 < Nk ? q + off + 1 : Nk) : Nk;  // keys [0, kmax_k) allowed
        float m = -INFINITY, lsum = 0.0f;  // m in the log2 (scaled) domain
        constexpr int kChunks = C::kSegCols / 64;
        float fnm = 0.0f, fmp = 0.0f;
        for (int j = 0; j < n_kv; ++j) {
            const int sb = j & 1;
            mbar_wait(&s_full[sb], (j >> 1) & 1);
            tc_fence_after();
            if (kFixed && j == 0) {  // Q has landed (S_0 is done): |q| of this row from the swizzled tile
                float qn2 = 0.0f;
#pragma unroll
                for (int p = 0; p < C::kPanels; ++p)
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const uint4 u = *reinterpret_cast<const uint4*>(sQ + p * (C::kBQ * 128) + r * 128 +
                                                                        ((c ^ (r & 7)) * 16));
                        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const float a = __uint_as_float(w[i] << 16), b = __uint_as_float(w[i] & 0xFFFF0000u);
                            qn2 = fmaf(a, a, fmaf(b, b, qn2));
                        }
                    }
                m = ceilf(c_log2 * sqrtf(qn2) * __ldg(kmax + kslab)) + 1.0f;
                fnm = -m;
                fmp = 12582912.0f - m;
            }
            const uint32_t base = tmem + ((quad * 32) << 16) + sb * C::kBK + seg * C::kSegCols;
            uint32_t ra[32], rb[32];
            tmem_ld64(base, ra, rb);
            tmem_ld_wait();
#pragma unroll
            for (int c = 0; c < kChunks; ++c) {
                uint32_t na[32], nb[32];
                if (c + 1 < kChunks) {  // prefetch the next 64 columns while this chunk computes
                    tmem_ld64(base + 64 * (c + 1), na, nb);  // one MIO op (shared with MUFU) per chunk
                } else {
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&s_empty[sb]);
                }
                if (kFixed)
                    lsum += lse_chunk_fixed<kPolyPairs, D>(ra, rb, kmax_k - (j * C::kBK + seg * C::kSegCols + 64 * c),
                                                           fnm, fmp);
                else
                    lse_chunk<kPolyPairs>(ra, rb, kmax_k - (j * C::kBK + seg * C::kSegCols + 64 * c), c_log2, m,
                                          lsum);
                if (c + 1 < kChunks) {
                    tmem_ld_wait();
#pragma unroll
                    for (int u = 0; u < 32; ++u) {
                        asm volatile("" : "+r"(na[u]), "+r"(nb[u]));  // pin the reads after wait::ld
                        ra[u] = na[u];
                        rb[u] = nb[u];
                    }
                }
            }
        }
        part[seg * C::kBQ + r] = make_float2(m, lsum);
        named_bar_sync(1, 32 * C::kSoftWarps);
        if (seg == 0 && q < Nq) {
            float M = -INFINITY;
#pragma unroll
            for (int s = 0; s < C::kSegs; ++s) M = fmaxf(M, part[s * C::kBQ + r].x);
            float L = 0.0f;
#pragma unroll
            for (int s = 0; s < C::kSegs; ++s) {
                const float2 pm = part[s * C::kBQ + r];
                L += pm.y * ex2(pm.x - M);
            }
            // fixed reference far above the row's scores: the exact kernel redoes the tile
            if (kFixed && !(L >= 0x1p-40f)) atomicOr(&tile_flags[tile_id], 1u);  // any row flags the tile
            const float lse2 = M + __log2f(L);  // log2 Σ exp2(c·s)
            const int64_t row = (int64_t)qslab * Nq + q;
            if (lse_out) lse_out[row] = lse2 / kLog2e;
            if (lam_out) write_lam(lam_out + row * 8, lse2 / c_log2);  // √d·lse (raw-score units)
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// λ rows from a caller-supplied natural-log LSE (proxy prefill).
__global__ void lam_from_lse_kernel(const float* __restrict__ lse, int64_t rows, float sqrt_d,
                                    __nv_bfloat16* __restrict__ lam_out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows) return;
    write_lam(lam_out + i * 8, lse[i] * sqrt_d);
}

// ---------------------------------------------------------------- pass 2 --
template <int D, bool kMax>
__global__ void __launch_bounds__(P2<D>::kThreads, 1)
    score_pool_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                      const __grid_constant__ CUtensorMap tlam, int Hq, int Hkv, int Nq, int Nk, int causal,
                      float c_log2, float* __restrict__ x_out) {
    using C = P2<D>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sK = smem;  // [blocks][panels][128 rows x 128 B]
    uint8_t* sAug = sK + C::kBlocks * C::kKBytes;
    uint8_t* sQ = sAug + C::kAugA;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sQ + C::kStages * C::kStageBytes);
    uint64_t* bar_k = bars;
    uint64_t* q_full = bars + 1;
    uint64_t* q_empty = q_full + C::kStages;
    uint64_t* s_full = q_empty + C::kStages;
    uint64_t* s_empty = s_full + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_empty + 2);

    const uint32_t warp = warp_id(), lane = lane_id();
    const int k0 = blockIdx.x * (C::kBK * C::kBlocks), kh = blockIdx.y, l = blockIdx.z;
    const int g = Hq / Hkv;
    const int kslab = l * Hkv + kh;
    const int off = Nk - Nq;
    const int tiles_per_head = (Nq + C::kBQ - 1) / C::kBQ;
    // causal: query tiles whose every query is earlier than k0 - off are skipped
    int first_tile = 0;
    if (causal) {
        const int qmin = k0 - off;
        first_tile = qmin <= 0 ? 0 : qmin / C::kBQ;
        if (first_tile > tiles_per_head) first_tile = tiles_per_head;
    }
    const int tiles_h = tiles_per_head - first_tile;
    const int n_tiles = g * tiles_h;

    // K_aug: row r = [1, 1, 1, 0, 0, 0, 0, 0] then an all-zero K half.
    for (int i = threadIdx.x; i < C::kAugA / 16; i += C::kThreads) {
        uint4 v = make_uint4(0, 0, 0, 0);
        if (i < C::kBK) {
            const uint32_t one = 0x3F80u;  // bf16 1.0
            v.x = one | (one << 16);
            v.y = one;
        }
        reinterpret_cast<uint4*>(sAug)[i] = v;
    }
    fence_proxy_async_smem();
    if (warp == 0 && lane == 0) {
        tma_prefetch(&tq);
        tma_prefetch(&tk);
        tma_prefetch(&tlam);
        mbar_init(bar_k, 1);
        for (int s = 0; s < C::kStages; ++s) {
            mbar_init(&q_full[s], 1);
            mbar_init(&q_empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&s_full[s], 1);
            mbar_init(&s_empty[s], 4 * C::kBlocks);
        }
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (elect_one() && n_tiles > 0) {
            mbar_arrive_expect_tx(bar_k, C::kBlocks * C::kKBytes);
            for (int b = 0; b < C::kBlocks; ++b)
                for (int p = 0; p < C::kPanels; ++p)
                    tma_load_3d(sK + b * C::kKBytes + p * (C::kBK * 128), &tk, bar_k, p * 64, k0 + b * C::kBK, kslab);
            for (int j = 0; j < n_tiles; ++j) {
                const int st = j % C::kStages;
                const int hh = j / tiles_h, qt = first_tile + j % tiles_h;
                const int qslab = l * Hq + kh * g + hh;
                mbar_wait(&q_empty[st], ((j / C::kStages) & 1) ^ 1);
                mbar_arrive_expect_tx(&q_full[st], C::kStageBytes);
                uint8_t* dst = sQ + st * C::kStageBytes;
                for (int p = 0; p < C::kPanels; ++p)
                    tma_load_3d(dst + p * (C::kBQ * 128), &tq, &q_full[st], p * 64, qt * C::kBQ, qslab);
                tma_load_3d(dst + C::kQBytes, &tlam, &q_full[st], 0, qt * C::kBQ, qslab);
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t idesc = idesc_f16(C::kBK, C::kBQ, 1);
        if (n_tiles > 0) mbar_wait(bar_k, 0);
        for (int j = 0; j < n_tiles; ++j) {
            const int st = j % C::kStages, sb = j & 1;
            mbar_wait(&q_full[st], (j / C::kStages) & 1);
            mbar_wait(&s_empty[sb], ((j >> 1) & 1) ^ 1);
            tc_fence_after();
            if (elect_one()) {
                uint8_t* qs = sQ + st * C::kStageBytes;
                const uint64_t a_aug = desc_noswz(sAug, C::kBK * 16, 128);
                const uint64_t b_aug = desc_noswz(qs + C::kQBytes, 0, 128);
#pragma unroll
                for (int b = 0; b < C::kBlocks; ++b) {
                    const uint32_t d = tmem + (sb * C::kBlocks + b) * C::kBQ;
#pragma unroll
                    for (int p = 0; p < C::kPanels; ++p) {
                        const uint64_t a = desc_sw128(sK + b * C::kKBytes + p * (C::kBK * 128));
                        const uint64_t bq = desc_sw128(qs + p * (C::kBQ * 128));
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk) mma_f16_ss(d, a + kk * 2, bq + kk * 2, idesc, (p | kk) != 0);
                    }
                    // − λ_q: K_aug (ones; zero second K half via LBO) · Q_aug (−hi, −mid, −lo)
                    mma_f16_ss(d, a_aug, b_aug, idesc, 1);
                }
                mma_commit(&s_full[sb]);
                mma_commit(&q_empty[st]);
            }
            __syncwarp();
        }
    } else if (warp >= 4) {
        const uint32_t quad = warp & 3;
        const int blk = (warp - 4) >> 2;
        const int r = quad * 32 + lane;
        const int key = k0 + blk * C::kBK + r;
        const int qmin = key - off;  // causal: queries >= qmin see this key
        float acc = kMax ? -INFINITY : 0.0f;
        for (int j = 0; j < n_tiles; ++j) {
            const int sb = j & 1;
            const int qbase = (first_tile + j % tiles_h) * C::kBQ;
            const int lo_col = causal ? max(qmin - qbase, 0) : 0;  // columns [lo_col, hi_col) valid
            const int hi_col = min(Nq - qbase, C::kBQ);
            mbar_wait(&s_full[sb], (j >> 1) & 1);
            tc_fence_after();
            const uint32_t base = tmem + ((quad * 32) << 16) + (sb * C::kBlocks + blk) * C::kBQ;
            uint32_t r0[32], r1[32], r2[32], r3[32];
            tmem_ld32(base, r0);
            tmem_ld32(base + 32, r1);
            tmem_ld32(base + 64, r2);
            tmem_ld32(base + 96, r3);
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_empty[sb]);
            float v[128];
#pragma unroll
            for (int u = 0; u < 32; ++u) {
                v[u] = __uint_as_float(r0[u]);
                v[32 + u] = __uint_as_float(r1[u]);
                v[64 + u] = __uint_as_float(r2[u]);
                v[96 + u] = __uint_as_float(r3[u]);
            }
            const bool full = lo_col == 0 && hi_col == C::kBQ;
            if (kMax) {
                if (!full) {
#pragma unroll
                    for (int u = 0; u < 128; ++u) v[u] = (u >= lo_col && u < hi_col) ? v[u] : -INFINITY;
                }
                float mt[8];
#pragma unroll
                for (int t8 = 0; t8 < 8; ++t8) mt[t8] = fmaxf(v[t8], v[t8 + 8]);
#pragma unroll
                for (int u = 16; u < 128; u += 16)
#pragma unroll
                    for (int t8 = 0; t8 < 8; ++t8) mt[t8] = max3f(mt[t8], v[u + t8], v[u + t8 + 8]);
                acc = max3f(acc, max3f(mt[0], mt[1], mt[2]),
                            max3f(max3f(mt[3], mt[4], mt[5]), mt[6], mt[7]));
            } else {
                float s0 = 0.0f, s1 = 0.0f, s2 = 0.0f, s3 = 0.0f;
#pragma unroll
                for (int u = 0; u < 128; u += 4) {
                    const float e0 = ex2(v[u] * c_log2), e1 = ex2(v[u + 1] * c_log2);
                    const float e2 = ex2(v[u + 2] * c_log2), e3 = ex2_poly(v[u + 3] * c_log2);
                    if (full) {
                        s0 += e0;
                        s1 += e1;
                        s2 += e2;
                        s3 += e3;
                    } else {
                        s0 += (u >= lo_col && u < hi_col) ? e0 : 0.0f;
                        s1 += (u + 1 >= lo_col && u + 1 < hi_col) ? e1 : 0.0f;
                        s2 += (u + 2 >= lo_col && u + 2 < hi_col) ? e2 : 0.0f;
                        s3 += (u + 3 >= lo_col && u + 3 < hi_col) ? e3 : 0.0f;
                    }
                }
                acc += (s0 + s1) + (s2 + s3);
            }
        }
        if (key < Nk) x_out[(int64_t)kslab * Nk + key] = kMax ? ex2(acc * c_log2) : acc;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

template <typename K>
void set_smem(K kern, int bytes) {
    PKV_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
}

template <int D>
void run_lse(const ScoreShape& s, const void* q, const void* k, float* lse, __nv_bfloat16* lam, cudaStream_t st,
             const float* kmax = nullptr, uint32_t* tile_flags = nullptr) {
    using C = P1<D>;
    static std::atomic<uint64_t> once{0};
    static int poly = 10;
    using KernT = decltype(&score_lse_kernel<D, 12, false>);
    static KernT table[2][7] = {{score_lse_kernel<D, 6, false>, score_lse_kernel<D, 8, false>,
                                 score_lse_kernel<D, 10, false>, score_lse_kernel<D, 12, false>,
                                 score_lse_kernel<D, 14, false>, score_lse_kernel<D, 16, false>,
                                 score_lse_kernel<D, 18, false>},
                                {score_lse_kernel<D, 6, true>, score_lse_kernel<D, 8, true>,
                                 score_lse_kernel<D, 10, true>, score_lse_kernel<D, 12, true>,
                                 score_lse_kernel<D, 14, true>, score_lse_kernel<D, 16, true>,
                                 score_lse_kernel<D, 18, true>}};
    if (first_on_device(once)) {
        for (auto& row : table)
            for (KernT kf : row) set_smem(kf, C::kSmem);
        if (const char* e = getenv("PKV_POLY_PAIRS")) poly = atoi(e);  // tuning knob: 6..18 of 32 pairs
    }
    const CUtensorMap tq = make_tmap_3d(q, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, D, s.Nq, s.L * s.Hq, D * 2, D * 2 * s.Nq,
                                        64, C::kBQ, 1, CU_TENSOR_MAP_SWIZZLE_128B);
    const CUtensorMap tk = make_tmap_3d(k, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, D, s.Nk, s.L * s.Hkv, D * 2, D * 2 * s.Nk,
                                        64, C::kBK, 1, CU_TENSOR_MAP_SWIZZLE_128B);
    const dim3 grid((unsigned)((s.Nq + C::kBQ - 1) / C::kBQ), (unsigned)s.Hq, (unsigned)s.L);
    const int pi = poly <= 6 ? 0 : poly <= 8 ? 1 : poly <= 10 ? 2 : poly <= 12 ? 3 : poly <= 14 ? 4 : poly <= 16 ? 5 : 6;
    const float c = kLog2e / sqrtf((float)D);
    if (kmax) {  // fixed-reference pass, then the exact kernel on the flagged tiles only
        table[1][pi]<<<grid, C::kThreads, C::kSmem, st>>>(tq, tk, (int)s.Hq, (int)s.Hkv, (int)s.Nq, (int)s.Nk,
                                                          s.causal ? 1 : 0, c, lse, lam, kmax, tile_flags);
        check_launch("score_lse_kernel<fixed>");
    }
    table[0][pi]<<<grid, C::kThreads, C::kSmem, st>>>(tq, tk, (int)s.Hq, (int)s.Hkv, (int)s.Nq, (int)s.Nk,
                                                      s.causal ? 1 : 0, c, lse, lam, nullptr, tile_flags);
    check_launch("score_lse_kernel");
}

template <int D>
void run_pool(const ScoreShape& s, const void* q, const void* k, const __nv_bfloat16* lam, bool reduce_max, float* x,
              cudaStream_t st) {
    using C = P2<D>;
    static std::atomic<uint64_t> once{0};
    if (first_on_device(once)) {
        set_smem(score_pool_kernel<D, true>, C::kSmem);
        set_smem(score_pool_kernel<D, false>, C::kSmem);
    }
    const CUtensorMap tq = make_tmap_3d(q, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, D, s.Nq, s.L * s.Hq, D * 2, D * 2 * s.Nq,
                                        64, C::kBQ, 1, CU_TENSOR_MAP_SWIZZLE_128B);
    const CUtensorMap tk = make_tmap_3d(k, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, D, s.Nk, s.L * s.Hkv, D * 2, D * 2 * s.Nk,
                                        64, C::kBK, 1, CU_TENSOR_MAP_SWIZZLE_128B);
    const CUtensorMap tl = make_tmap_3d(lam, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 8, s.Nq, s.L * s.Hq, 16, 16 * s.Nq, 8,
                                        C::kBQ, 1, CU_TENSOR_MAP_SWIZZLE_NONE);
    const int keys_per_cta = C::kBK * C::kBlocks;
    const dim3 grid((unsigned)((s.Nk + keys_per_cta - 1) / keys_per_cta), (unsigned)s.Hkv, (unsigned)s.L);
    const float c = kLog2e / sqrtf((float)D);
    if (reduce_max) {
        score_pool_kernel<D, true><<<grid, C::kThreads, C::kSmem, st>>>(tq, tk, tl, (int)s.Hq, (int)s.Hkv, (int)s.Nq,
                                                                       (int)s.Nk, s.causal ? 1 : 0, c, x);
    } else {
        score_pool_kernel<D, false><<<grid, C::kThreads, C::kSmem, st>>>(tq, tk, tl, (int)s.Hq, (int)s.Hkv,
                                                                        (int)s.Nq, (int)s.Nk, s.causal ? 1 : 0, c, x);
    }
    check_launch("score_pool_kernel");
}

}  // namespace

void score_validate(const ScoreShape& s) {
    PKV_REQUIRE_SHAPE(s.L > 0 && s.Hq > 0 && s.Hkv > 0 && s.Nq > 0 && s.Nk > 0, "score extents must be positive");
    PKV_REQUIRE_SHAPE(s.Hq % s.Hkv == 0, "query heads ", s.Hq, " not a multiple of KV heads ", s.Hkv);
    PKV_REQUIRE(s.d == 64 || s.d == 128, PKV_ECONFIG, "GPU scoring supports head_dim 64 or 128, got ", s.d);
    PKV_REQUIRE(s.L * s.Hq <= 65535 && s.Nq < (int64_t(1) << 31) && s.Nk < (int64_t(1) << 31), PKV_ECONFIG,
                "score shape too large for one launch");
    PKV_REQUIRE(!s.causal || s.Nk >= s.Nq, PKV_ECONFIG, "causal scoring needs Nk >= Nq");
}

bool score_fixed_enabled() {
    static const bool on = [] {
        const char* e = getenv("PKV_SCORE_FIXED");
        return !(e && atoi(e) == 0);
    }();
    return on;
}

void launch_score_lse(const ScoreShape& s, const void* q, const void* k, float* lse, __nv_bfloat16* lam,
                      cudaStream_t st, DevBuf* aux) {
    const float* kmax = nullptr;
    uint32_t* flags = nullptr;
    if (aux && score_fixed_enabled()) {
        const int64_t slabs = s.L * s.Hkv, tiles = s.L * s.Hq * ((s.Nq + 127) / 128);
        const int64_t kbytes = (slabs * 4 + 255) & ~int64_t(255);
        auto* w = static_cast<uint8_t*>(aux->get((size_t)(kbytes + tiles * 4)));
        float* km = reinterpret_cast<float*>(w);
        flags = reinterpret_cast<uint32_t*>(w + kbytes);
        PKV_CUDA(cudaMemsetAsync(flags, 0, (size_t)tiles * 4, st));
        kmax_norm_kernel<<<(unsigned)slabs, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(k), s.Nk, (int)s.d, km);
        check_launch("kmax_norm_kernel");
        kmax = km;
    }
    if (s.d == 64) run_lse<64>(s, q, k, lse, lam, st, kmax, flags);
    else run_lse<128>(s, q, k, lse, lam, st, kmax, flags);
}

void launch_lam_from_lse(const float* lse, int64_t rows, int64_t d, __nv_bfloat16* lam, cudaStream_t st) {
    lam_from_lse_kernel<<<(unsigned)((rows + 255) / 256), 256, 0, st>>>(lse, rows, sqrtf((float)d), lam);
    check_launch("lam_from_lse_kernel");
}

void launch_score_pool(const ScoreShape& s, const void* q, const void* k, const __nv_bfloat16* lam, bool reduce_max,
                       float* x, cudaStream_t st) {
    if (s.d == 64) run_pool<64>(s, q, k, lam, reduce_max, x, st);
    else run_pool<128>(s, q, k, lam, reduce_max, x, st);
}

}  // namespace pkv
