// gemm.cu — see gemm.cuh. Persistent, warp-specialised tcgen05 GEMM.
//   warp 0 : TMA producer (one elected lane)
//   warp 1 : MMA issuer (one elected lane)
//   warp 2 : TMEM allocator
//   warps 4-7 : epilogue (thread = accumulator row; TMEM lane quadrant = warp % 4)
#include <cuda_fp8.h>

#include "gemm.cuh"

namespace pkv {
namespace {

using namespace sm100;

constexpr int kBM = 128;
constexpr int kBK = 64;  // one 128-B swizzle atom of fp16
constexpr int kEpiGroups = 2;  // epilogue warpgroups, each owning BN / kEpiGroups columns
constexpr int kThreads = 128 + 128 * kEpiGroups;
constexpr int kABytes = kBM * kBK * 2;
// per epilogue warp: 32x32 fp32 staging tile (row stride 33: conflict-free)
constexpr int kStageLd = 33;
constexpr int kStageBufBytes = 4 * kEpiGroups * 32 * kStageLd * 4;


template <int BN, int NA, int NB>
struct Cfg {
    static constexpr int kBBytes = BN * kBK * 2;
    static constexpr int kStageBytes = NA * kABytes + NB * kBBytes;
    static constexpr int kBudget = 227 * 1024 - 2048 - kStageBufBytes;
    static constexpr int kStagesRaw = kBudget / kStageBytes;
    static constexpr int kStages = kStagesRaw > 6 ? 6 : kStagesRaw;
    static constexpr int kSmem = 1024 + kStages * kStageBytes + 256 + kStageBufBytes;
    static constexpr uint32_t kTmemCols = (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128 : (2 * BN <= 256) ? 256 : 512;
    static_assert(kStages >= 2, "not enough shared memory for 2 stages");
};

// Warp-cooperative epilogue for a 32-row x 32-column accumulator chunk:
// thread t holds row (row0 + t). The chunk is transposed through a padded smem
// tile so global loads/stores are row-contiguous across the warp (128 B fp32
// rows, or two 64 B fp16 rows per instruction) instead of 32 scattered
// per-thread rows (partial-sector traffic).
// gelu_fast (sm100.cuh) on a packed pair: the FMA-pipe work as FFMA2/FMUL2.
__device__ __forceinline__ float2 gelu_fast2(float x0, float x1) {
    const uint64_t z = fmul2(pack2(fabsf(x0), fabsf(x1)), pack2(0.70710678118654752f, 0.70710678118654752f));
    const float2 zd = unpack2(ffma2(pack2(0.3275911f, 0.3275911f), z, pack2(1.0f, 1.0f)));
    const uint64_t t = pack2(rcp_approx(zd.x), rcp_approx(zd.y));
    uint64_t q = ffma2(pack2(1.061405429f, 1.061405429f), t, pack2(-1.453152027f, -1.453152027f));
    q = ffma2(q, t, pack2(1.421413741f, 1.421413741f));
    q = ffma2(q, t, pack2(-0.284496736f, -0.284496736f));
    q = ffma2(q, t, pack2(0.254829592f, 0.254829592f));
    const float2 a = unpack2(fmul2(fmul2(z, pack2(-1.4426950408889634f, -1.4426950408889634f)), z));
    const uint64_t e = pack2(ex2(a.x), ex2(a.y));
    const float2 h = unpack2(fmul2(fmul2(pack2(0.5f * x0, 0.5f * x1), fmul2(q, t)), e));
    return make_float2(x0 >= 0.0f ? x0 - h.x : h.x, x1 >= 0.0f ? x1 - h.y : h.y);
}

// Per-row epilogue of a 32-column accumulator chunk (thread = row; the row's
// 32 columns are contiguous in global memory: 16-byte vector accesses, the L2
// merges the warp's partial sectors). res: residual row slice (EPI_RESID).
template <int EPI>
__device__ __forceinline__ void epilogue_row(const GemmEpiParams& p, int64_t row, int64_t col0, int64_t M, int64_t N,
                                             const uint32_t (&r)[32], const float4 (&res)[8]) {
    if (row >= M) return;
    const bool full = col0 + 32 <= N;
    float v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]) * p.acc_scale;
    if ((EPI == EPI_F32 || EPI == EPI_GELU_PE) && p.row_scale) {
        const float rs = __ldg(p.row_scale + row);
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] *= rs;
    }
    if (p.bias) {
        if (full) {
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
                const float4 b = __ldg(reinterpret_cast<const float4*>(p.bias + col0 + j));
                v[j] += b.x;
                v[j + 1] += b.y;
                v[j + 2] += b.z;
                v[j + 3] += b.w;
            }
        } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
                if (col0 + j < N) v[j] += __ldg(p.bias + col0 + j);
        }
    }
    if (EPI == EPI_GELU_F16X || EPI == EPI_GELU_PE) {
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
            const float2 g = gelu_fast2(v[j], v[j + 1]);
            v[j] = g.x;
            v[j + 1] = g.y;
        }
    }
    const int64_t base = row * p.ldo + col0;
    if (EPI == EPI_F16X || EPI == EPI_GELU_F16X) {
        if (full) {
#pragma unroll
            for (int j = 0; j < 32; j += 8) {
                uint32_t hi[4], lo[4];
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const __half2 h = __floats2half2_rn(v[j + 2 * t], v[j + 2 * t + 1]);
                    const float2 hf = __half22float2(h);
                    const __half2 l = __floats2half2_rn(v[j + 2 * t] - hf.x, v[j + 2 * t + 1] - hf.y);
                    hi[t] = *reinterpret_cast<const uint32_t*>(&h);
                    lo[t] = *reinterpret_cast<const uint32_t*>(&l);
                }
                *reinterpret_cast<uint4*>(p.out_h + base + j) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
                if (p.out_l) *reinterpret_cast<uint4*>(p.out_l + base + j) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
            }
        } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                if (col0 + j >= N) continue;
                const __half hi = __float2half_rn(v[j]);
                p.out_h[base + j] = hi;
                if (p.out_l) p.out_l[base + j] = __float2half_rn(v[j] - __half2float(hi));
            }
        }
        return;
    }
    if (EPI == EPI_GELU_PE && p.pe) {
        const float* pe = p.pe + (row % p.lw) * p.ldo + col0;
        if (full) {
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
                const float4 e = __ldg(reinterpret_cast<const float4*>(pe + j));
                v[j] += e.x;
                v[j + 1] += e.y;
                v[j + 2] += e.z;
                v[j + 3] += e.w;
            }
        } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
                if (col0 + j < N) v[j] += __ldg(pe + j);
        }
    }
    if (EPI == EPI_RESID) {
        if (full) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                v[4 * j] += res[j].x;
                v[4 * j + 1] += res[j].y;
                v[4 * j + 2] += res[j].z;
                v[4 * j + 3] += res[j].w;
            }
        } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
                if (col0 + j < N) v[j] += p.out_f32[base + j];
        }
    }
    float* out = p.out_f32 + base;
    if (full) {
#pragma unroll
        for (int j = 0; j < 32; j += 4) *reinterpret_cast<float4*>(out + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
    } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
            if (col0 + j < N) out[j] = v[j];
    }
}

// kF8Out: the e4m3 output planes (p.out_l8 / out_h8) are compiled in only for
// the FP16F8 kernels (their register cost would spill the FP16X3 GELU epilogue)
template <int EPI, bool kF8Out = false>
__device__ __forceinline__ void epilogue_coalesced(const GemmEpiParams& p, int64_t row0, int64_t col0, int64_t M,
                                                   int64_t N, const uint32_t (&r)[32], float* stg) {
    const int lane = threadIdx.x & 31;
    if (EPI == EPI_GELU_PE) {  // GELU-heavy, fp32 out: per-row (measured faster than the transpose)
        const float4 none[8] = {};
        epilogue_row<EPI>(p, row0 + lane, col0, M, N, r, none);
        return;
    }
    const float as = p.acc_scale;
#pragma unroll
    for (int j = 0; j < 32; ++j) stg[lane * kStageLd + j] = __uint_as_float(r[j]) * as;
    __syncwarp();
    // warp-uniform fast path: the whole 32x32 chunk is in bounds (no per-row
    // checks, fully unrolled so independent rows overlap)
    const bool full = row0 + 32 <= M && col0 + 32 <= N;
    if (EPI == EPI_F16X || EPI == EPI_GELU_F16X) {
        const int half = lane >> 4, cp = (lane & 15) * 2;
        const int64_t col = col0 + cp;
        const bool c0ok = col < N, c1ok = col + 1 < N;
        const float b0 = (p.bias && c0ok) ? __ldg(p.bias + col) : 0.0f;
        const float b1 = (p.bias && c1ok) ? __ldg(p.bias + col + 1) : 0.0f;
        if (full) {
            __half* oh = p.out_h + (row0 + half) * p.ldo + col;
            __half* ol = p.out_l ? p.out_l + (row0 + half) * p.ldo + col : nullptr;
            const int64_t step = 2 * p.ldo;
#pragma unroll
            for (int rr = 0; rr < 32; rr += 2) {
                float x0 = stg[(rr + half) * kStageLd + cp] + b0;
                float x1 = stg[(rr + half) * kStageLd + cp + 1] + b1;
                if (EPI == EPI_GELU_F16X) {  // packed FFMA2/FMUL2 form of gelu_fast
                    const float2 g = gelu_fast2(x0, x1);
                    x0 = g.x;
                    x1 = g.y;
                }
                const __half2 hi = __floats2half2_rn(x0, x1);
                const float2 hb = __half22float2(hi);
                *reinterpret_cast<__half2*>(oh + (rr >> 1) * step) = hi;
                if (kF8Out && p.out_l8) {
                    const int64_t o8 = (row0 + rr + half) * p.ldo + col;
                    *reinterpret_cast<__nv_fp8x2_storage_t*>(p.out_l8 + o8) = __nv_cvt_float2_to_fp8x2(
                        make_float2((x0 - hb.x) * p.l8_mul, (x1 - hb.y) * p.l8_mul), __NV_SATFINITE, __NV_E4M3);
                    *reinterpret_cast<__nv_fp8x2_storage_t*>(p.out_h8 + o8) = __nv_cvt_float2_to_fp8x2(
                        make_float2(hb.x * p.h8_mul, hb.y * p.h8_mul), __NV_SATFINITE, __NV_E4M3);
                } else if (ol) {
                    *reinterpret_cast<__half2*>(ol + (rr >> 1) * step) = __floats2half2_rn(x0 - hb.x, x1 - hb.y);
                }
            }
        } else {
#pragma unroll 4
            for (int rr = 0; rr < 32; rr += 2) {
                const int64_t row = row0 + rr + half;
                if (row >= M) continue;
                float x0 = stg[(rr + half) * kStageLd + cp] + b0;
                float x1 = stg[(rr + half) * kStageLd + cp + 1] + b1;
                if (EPI == EPI_GELU_F16X) {
                    x0 = gelu_fast(x0);
                    x1 = gelu_fast(x1);
                }
                const __half2 hi = __floats2half2_rn(x0, x1);
                const float2 hb = __half22float2(hi);
                const int64_t o = row * p.ldo + col;
                if (c1ok) {
                    *reinterpret_cast<__half2*>(p.out_h + o) = hi;
                    if (kF8Out && p.out_l8) {
                        *reinterpret_cast<__nv_fp8x2_storage_t*>(p.out_l8 + o) = __nv_cvt_float2_to_fp8x2(
                            make_float2((x0 - hb.x) * p.l8_mul, (x1 - hb.y) * p.l8_mul), __NV_SATFINITE, __NV_E4M3);
                        *reinterpret_cast<__nv_fp8x2_storage_t*>(p.out_h8 + o) = __nv_cvt_float2_to_fp8x2(
                            make_float2(hb.x * p.h8_mul, hb.y * p.h8_mul), __NV_SATFINITE, __NV_E4M3);
                    } else if (p.out_l) {
                        *reinterpret_cast<__half2*>(p.out_l + o) = __floats2half2_rn(x0 - hb.x, x1 - hb.y);
                    }
                } else if (c0ok) {
                    p.out_h[o] = __low2half(hi);
                    if (kF8Out && p.out_l8) {
                        p.out_l8[o] = __nv_cvt_float_to_fp8((x0 - hb.x) * p.l8_mul, __NV_SATFINITE, __NV_E4M3);
                        p.out_h8[o] = __nv_cvt_float_to_fp8(hb.x * p.h8_mul, __NV_SATFINITE, __NV_E4M3);
                    } else if (p.out_l) {
                        p.out_l[o] = __float2half_rn(x0 - hb.x);
                    }
                }
            }
        }
    } else {
        const int64_t col = col0 + lane;
        const bool cok = col < N;
        const float b = (p.bias && cok) ? __ldg(p.bias + col) : 0.0f;
        float* out = p.out_f32 + row0 * p.ldo + col;
        if (full) {
            // all global loads of the chunk are issued before any use (32 in flight per lane)
            if (EPI == EPI_RESID) {
                float extra[32];  // all residual loads in flight before any use
#pragma unroll
                for (int rr = 0; rr < 32; ++rr) extra[rr] = out[rr * p.ldo];
#pragma unroll
                for (int rr = 0; rr < 32; ++rr) out[rr * p.ldo] = stg[rr * kStageLd + lane] + b + extra[rr];
            } else {
                int pr = (int)(row0 % p.lw);  // window position of row0 (PE table is L2-resident)
                const float* rsc = (EPI == EPI_F32 || EPI == EPI_GELU_PE) ? p.row_scale : nullptr;
#pragma unroll 8
                for (int rr = 0; rr < 32; ++rr) {
                    float x = stg[rr * kStageLd + lane];
                    if (rsc) x *= __ldg(rsc + row0 + rr);
                    x += b;
                    if (EPI == EPI_GELU_PE) {
                        x = gelu_fast(x);
                        if (p.pe) x += __ldg(p.pe + (int64_t)pr * p.ldo + col);
                        if (++pr == p.lw) pr = 0;
                    }
                    out[rr * p.ldo] = x;
                }
            }
        } else {
            float extra[32];
            if (EPI == EPI_RESID || (EPI == EPI_GELU_PE && p.pe)) {
                int pr = 0;
                if (EPI == EPI_GELU_PE) pr = (int)(row0 % p.lw);
#pragma unroll
                for (int rr = 0; rr < 32; ++rr) {
                    const bool ok = cok && row0 + rr < M;
                    if (EPI == EPI_RESID) {
                        extra[rr] = ok ? out[rr * p.ldo] : 0.0f;
                    } else {
                        extra[rr] = ok ? __ldg(p.pe + (int64_t)pr * p.ldo + col) : 0.0f;
                        if (++pr == p.lw) pr = 0;
                    }
                }
            }
#pragma unroll
            for (int rr = 0; rr < 32; ++rr) {
                if (!cok || row0 + rr >= M) continue;
                float x = stg[rr * kStageLd + lane];
                if ((EPI == EPI_F32 || EPI == EPI_GELU_PE) && p.row_scale) x *= __ldg(p.row_scale + row0 + rr);
                x += b;
                if (EPI == EPI_GELU_PE) {
                    x = gelu_fast(x);
                    if (p.pe) x += extra[rr];
                }
                if (EPI == EPI_RESID) x += extra[rr];
                out[rr * p.ldo] = x;
            }
        }
    }
    __syncwarp();
}

// Residual epilogue (resid += acc + bias) for a 32x32 chunk whose residual
// values were prefetched by the caller (res[rr] = out[row0 + rr][col0 + lane]).
__device__ __forceinline__ void epilogue_resid_pref(const GemmEpiParams& p, int64_t row0, int64_t col0, int64_t M,
                                                    int64_t N, const uint32_t (&r)[32], const float (&res)[32],
                                                    float* stg) {
    const int lane = threadIdx.x & 31;
    const float as = p.acc_scale;
#pragma unroll
    for (int j = 0; j < 32; ++j) stg[lane * kStageLd + j] = __uint_as_float(r[j]) * as;
    __syncwarp();
    const int64_t col = col0 + lane;
    const bool cok = col < N;
    const float b = (p.bias && cok) ? __ldg(p.bias + col) : 0.0f;
    float* out = p.out_f32 + row0 * p.ldo + col;
    if (cok && row0 + 32 <= M) {
#pragma unroll
        for (int rr = 0; rr < 32; ++rr) out[rr * p.ldo] = stg[rr * kStageLd + lane] + b + res[rr];
    } else {
#pragma unroll
        for (int rr = 0; rr < 32; ++rr)
            if (cok && row0 + rr < M) out[rr * p.ldo] = stg[rr * kStageLd + lane] + b + res[rr];
    }
    __syncwarp();
}

__device__ __forceinline__ void resid_prefetch(const GemmEpiParams& p, int64_t row0, int64_t col0, int64_t M,
                                               int64_t N, float (&res)[32]) {
    const int64_t col = col0 + (threadIdx.x & 31);
    const float* src = p.out_f32 + row0 * p.ldo + col;
#pragma unroll
    for (int rr = 0; rr < 32; ++rr) res[rr] = (col < N && row0 + rr < M) ? src[rr * p.ldo] : 0.0f;
}

template <int BN, int NA, int NB, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tA0, const __grid_constant__ CUtensorMap tA1,
                const __grid_constant__ CUtensorMap tB0, const __grid_constant__ CUtensorMap tB1, GemmEpiParams p,
                int64_t M, int64_t N, int64_t K) {
    using C = Cfg<BN, NA, NB>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes);
    uint64_t* empty = full + C::kStages;
    uint64_t* tfull = empty + C::kStages;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    float* stagebuf = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(tempty) + 256) +
                      (warp_id() >= 4 ? (warp_id() - 4) * 32 * kStageLd : 0);

    const uint32_t warp = warp_id(), lane = lane_id();
    const int64_t tiles_m = (M + kBM - 1) / kBM, tiles_n = (N + BN - 1) / BN;
    const int64_t tiles = tiles_m * tiles_n;
    const int num_kb = (int)((K + kBK - 1) / kBK);

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tA0);
        tma_prefetch(&tB0);
        if (NA > 1) tma_prefetch(&tA1);
        if (NB > 1) tma_prefetch(&tB1);
        for (int s = 0; s < C::kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 4 * kEpiGroups);
        }
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc(tmem_slot, C::kTmemCols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (elect_one()) {
            int stage = 0;
            uint32_t phase = 0;
            for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
                const int32_t m0 = (int32_t)((t / tiles_n) * kBM);
                const int32_t n0 = (int32_t)((t % tiles_n) * BN);
                for (int kb = 0; kb < num_kb; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* st = smem + stage * C::kStageBytes;
                    mbar_arrive_expect_tx(&full[stage], C::kStageBytes);
                    tma_load_2d(st, &tA0, &full[stage], kb * kBK, m0);
                    if (NA > 1) tma_load_2d(st + kABytes, &tA1, &full[stage], kb * kBK, m0);
                    tma_load_2d(st + NA * kABytes, &tB0, &full[stage], kb * kBK, n0);
                    if (NB > 1) tma_load_2d(st + NA * kABytes + C::kBBytes, &tB1, &full[stage], kb * kBK, n0);
                    if (++stage == C::kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t idesc = idesc_f16(kBM, BN, 0);
        int stage = 0;
        uint32_t phase = 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
            mbar_wait(&tempty[acc], acc_phase ^ 1);
            tc_fence_after();
            const uint32_t d = tmem_base + acc * BN;
            for (int kb = 0; kb < num_kb; ++kb) {
                mbar_wait(&full[stage], phase);
                tc_fence_after();
                if (elect_one()) {
                    uint8_t* st = smem + stage * C::kStageBytes;
                    const uint64_t a0 = desc_sw128(st);
                    const uint64_t a1 = desc_sw128(st + kABytes);
                    const uint64_t b0 = desc_sw128(st + NA * kABytes);
                    const uint64_t b1 = desc_sw128(st + NA * kABytes + C::kBBytes);
#pragma unroll
                    for (int kk = 0; kk < kBK / 16; ++kk) {
                        const uint64_t off = (uint64_t)(kk * 2);  // +32 B within the swizzle atom
                        mma_f16_ss(d, a0 + off, b0 + off, idesc, (kb | kk) != 0);
                        if (NA > 1) mma_f16_ss(d, a1 + off, b0 + off, idesc, 1);
                        if (NB > 1) mma_f16_ss(d, a0 + off, b1 + off, idesc, 1);
                    }
                    mma_commit(&empty[stage]);
                }
                __syncwarp();
                if (++stage == C::kStages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            if (elect_one()) mma_commit(&tfull[acc]);
            __syncwarp();
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    } else if (warp >= 4) {
        const uint32_t quad = warp & 3;
        const int cg = (int)(warp - 4) >> 2;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
            const int64_t m0 = (t / tiles_n) * kBM;
            const int64_t n0 = (t % tiles_n) * BN;
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const int64_t row = m0 + quad * 32 + lane;
            const uint32_t taddr = tmem_base + ((quad * 32) << 16) + acc * BN;
            // this warp's column group; the next chunk's TMEM load overlaps the
            // current chunk's epilogue math (double-buffered registers)
            const int cbeg = cg * (BN / kEpiGroups), cend = cbeg + BN / kEpiGroups;
            uint32_t r[2][32];
            tmem_ld32(taddr + cbeg, r[0]);
            tmem_ld_wait();
#pragma unroll 1
            for (int c0 = cbeg; c0 < cend; c0 += 64) {
                if (c0 + 32 < cend) tmem_ld32(taddr + c0 + 32, r[1]);
                if (n0 + c0 < N) epilogue_coalesced<EPI>(p, row - lane, n0 + c0, M, N, r[0], stagebuf);
                tmem_ld_wait();
                if (c0 + 32 < cend) {
                    if (c0 + 64 < cend) tmem_ld32(taddr + c0 + 64, r[0]);
                    if (n0 + c0 + 32 < N) epilogue_coalesced<EPI>(p, row - lane, n0 + c0 + 32, M, N, r[1], stagebuf);
                    tmem_ld_wait();
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem_base, C::kTmemCols);
    }
}

template <int BN, int NA, int NB, int EPI>
void launch(const GemmArgs& g, int sm_count, cudaStream_t st) {
    using C = Cfg<BN, NA, NB>;
    auto kern = gemm_kernel<BN, NA, NB, EPI>;
    static std::atomic<uint64_t> attr_set{0};
    if (first_on_device(attr_set)) PKV_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
    const int64_t tiles = ((g.M + kBM - 1) / kBM) * ((g.N + BN - 1) / BN);
    const int grid = (int)(tiles < sm_count ? tiles : sm_count);
    kern<<<grid, kThreads, C::kSmem, st>>>(g.a[0], g.a[1], g.b[0], g.b[1], g.p, g.M, g.N, g.K);
    check_launch("gemm_kernel");
}

template <int BN, int NA, int NB>
void dispatch_epi(const GemmArgs& g, int sm, cudaStream_t st) {
    switch (g.epi) {
        case EPI_F32: return launch<BN, NA, NB, EPI_F32>(g, sm, st);
        case EPI_F16X: return launch<BN, NA, NB, EPI_F16X>(g, sm, st);
        case EPI_GELU_F16X: return launch<BN, NA, NB, EPI_GELU_F16X>(g, sm, st);
        case EPI_RESID: return launch<BN, NA, NB, EPI_RESID>(g, sm, st);
        case EPI_GELU_PE: return launch<BN, NA, NB, EPI_GELU_PE>(g, sm, st);
    }
}

template <int BN>
void dispatch_planes(const GemmArgs& g, int sm, cudaStream_t st) {
    if (g.na == 1 && g.nb == 1) return dispatch_epi<BN, 1, 1>(g, sm, st);
    if (g.na == 2 && g.nb == 1) return dispatch_epi<BN, 2, 1>(g, sm, st);
    if (g.na == 1 && g.nb == 2) return dispatch_epi<BN, 1, 2>(g, sm, st);
    if (g.na == 2 && g.nb == 2) return dispatch_epi<BN, 2, 2>(g, sm, st);
    throw Error{PKV_ECONFIG, cat("unsupported GEMM plane combination na=", g.na, " nb=", g.nb)};
}

// ------------------------------------------------------------ CTA pair ----
// cta_group::2 variant: a cluster of 2 CTAs computes a 256x256 tile. CTA r
// loads A rows [m0 + 128r, +128) and B rows [n0 + 128r, +128) (half of each
// operand per SM); the leader issues tcgen05.mma.cta_group::2 (M = 256), each
// CTA's TMEM receives its 128 accumulator rows x 256 columns. Per-SM operand
// traffic drops by a third vs the 128x256 single-CTA tile, which lets the
// 4-plane FP16X3 stages fit 3-deep.
// pair kernel epilogue width per epilogue kind: 16 warps (64 accumulator
// columns each) for the GELU + hi/lo-split FFN1 epilogue, whose per-tile work
// bounds that GEMM; 8 elsewhere (the residual path needs the registers and the
// 3-deep operand ring that the larger staging buffer would cost)
// FP16F8 halves the correction MMAs' tensor time, so its QKV (F16X) epilogue gets
// 16 warps too (measured: QKV 12 % faster in mode 6, no gain in mode 3)
__host__ __device__ constexpr int epi_groups2(int epi, bool f8) {
    return (epi == EPI_GELU_F16X || (f8 && epi == EPI_F16X)) ? 4 : 2;
}

template <int NA, int NB, int EPI, bool F8 = false>
struct Cfg2 {
    static constexpr int kEpiGroups2 = epi_groups2(EPI, F8);
    static constexpr int kThreads2 = 128 + 128 * kEpiGroups2;
    static constexpr int kStageBufBytes2 = 4 * kEpiGroups2 * 32 * kStageLd * 4;
    static constexpr int kHalf = 128 * kBK * 2;  // 16 KB: one operand half-tile plane
    static constexpr int kStageBytes = (NA + NB) * kHalf;
    static constexpr int kBudget = 227 * 1024 - 2048 - kStageBufBytes2;
    static constexpr int kStagesRaw = kBudget / kStageBytes;
    static constexpr int kStages = kStagesRaw > 6 ? 6 : kStagesRaw;
    static constexpr int kSmem = 1024 + kStages * kStageBytes + 256 + kStageBufBytes2;
};

// F8 (FP16F8, NA = NB = 2): each stage holds [A16 16 KB | A8lo 8 KB | A8hi 8 KB |
// B16 16 KB | B8hi 8 KB | B8lo 8 KB] per CTA (the same 64 KB as FP16X3); per
// 64-wide K block: 4 fp16 MMAs A16·B16 + 2 e4m3 MMAs A8lo·B8hi + 2 A8hi·B8lo
// (tA1 / tA2 = A8lo / A8hi maps, tB1 / tB2 = B8hi / B8lo, SWIZZLE_64B).
template <int NA, int NB, int EPI, bool F8 = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Cfg2<NA, NB, EPI, F8>::kThreads2, 1)
    gemm2_kernel(const __grid_constant__ CUtensorMap tA0, const __grid_constant__ CUtensorMap tA1,
                 const __grid_constant__ CUtensorMap tB0, const __grid_constant__ CUtensorMap tB1,
                 const __grid_constant__ CUtensorMap tA2, const __grid_constant__ CUtensorMap tB2, GemmEpiParams p,
                 int64_t M, int64_t N, int64_t K) {
    static_assert(!F8 || (NA == 2 && NB == 2), "FP16F8 uses the two-plane stage layout");
    using C = Cfg2<NA, NB, EPI, F8>;
    constexpr int kEpiGroups2 = C::kEpiGroups2;
    constexpr int BN = 256;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes);
    uint64_t* empty = full + C::kStages;
    uint64_t* tfull = empty + C::kStages;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    float* stagebuf = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(tempty) + 256) +
                      (warp_id() >= 4 ? (warp_id() - 4) * 32 * kStageLd : 0);

    const uint32_t warp = warp_id(), lane = lane_id();
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    const int64_t tiles_m = (M + 255) / 256, tiles_n = (N + BN - 1) / BN;
    const int64_t tiles = tiles_m * tiles_n;
    const int64_t cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
    const int num_kb = (int)((K + kBK - 1) / kBK);

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tA0);
        tma_prefetch(&tB0);
        if (NA > 1) tma_prefetch(&tA1);
        if (NB > 1) tma_prefetch(&tB1);
        if (F8) {
            tma_prefetch(&tA2);
            tma_prefetch(&tB2);
        }
        for (int s = 0; s < C::kStages; ++s) {
            mbar_init(&full[s], 1);   // leader: arrive.expect_tx(both halves); bytes of both CTAs land here
            mbar_init(&empty[s], 1);  // multicast commit from the leader's MMA
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 8 * kEpiGroups2);  // epilogue warps of both CTAs (leader's copy is used)
        }
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc_2sm(tmem_slot, 512);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (elect_one()) {
            int stage = 0;
            uint32_t phase = 0;
            for (int64_t t = cluster; t < tiles; t += nclusters) {
                const int32_t m0 = (int32_t)((t / tiles_n) * 256 + rank * 128);
                const int32_t n0 = (int32_t)((t % tiles_n) * BN + rank * 128);
                for (int kb = 0; kb < num_kb; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* st = smem + stage * C::kStageBytes;
                    if (leader) mbar_arrive_expect_tx(&full[stage], 2 * C::kStageBytes);
                    tma_load_2d_2sm(st, &tA0, &full[stage], kb * kBK, m0);
                    if (F8) {
                        tma_load_2d_2sm(st + C::kHalf, &tA1, &full[stage], kb * kBK, m0);
                        tma_load_2d_2sm(st + C::kHalf + C::kHalf / 2, &tA2, &full[stage], kb * kBK, m0);
                        tma_load_2d_2sm(st + 2 * C::kHalf, &tB0, &full[stage], kb * kBK, n0);
                        tma_load_2d_2sm(st + 3 * C::kHalf, &tB1, &full[stage], kb * kBK, n0);
                        tma_load_2d_2sm(st + 3 * C::kHalf + C::kHalf / 2, &tB2, &full[stage], kb * kBK, n0);
                    } else {
                        if (NA > 1) tma_load_2d_2sm(st + C::kHalf, &tA1, &full[stage], kb * kBK, m0);
                        tma_load_2d_2sm(st + NA * C::kHalf, &tB0, &full[stage], kb * kBK, n0);
                        if (NB > 1) tma_load_2d_2sm(st + (NA + 1) * C::kHalf, &tB1, &full[stage], kb * kBK, n0);
                    }
                    if (++stage == C::kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (leader) {
            constexpr uint32_t idesc = idesc_f16(256, BN, 0);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int64_t t = cluster; t < tiles; t += nclusters) {
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d = tmem_base + acc * BN;
                for (int kb = 0; kb < num_kb; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    if (elect_one()) {
                        uint8_t* st = smem + stage * C::kStageBytes;
                        if (F8) {
                            const uint64_t a0 = desc_sw128(st), b0 = desc_sw128(st + 2 * C::kHalf);
                            const uint64_t a8l = desc_sw64(st + C::kHalf);
                            const uint64_t a8h = desc_sw64(st + C::kHalf + C::kHalf / 2);
                            const uint64_t b8h = desc_sw64(st + 3 * C::kHalf);
                            const uint64_t b8l = desc_sw64(st + 3 * C::kHalf + C::kHalf / 2);
#pragma unroll
                            for (int kk = 0; kk < kBK / 16; ++kk)
                                mma_f16_ss_2sm(d, a0 + kk * 2, b0 + kk * 2, idesc, (kb | kk) != 0);
#pragma unroll
                            for (int kk = 0; kk < kBK / 32; ++kk) {  // e4m3: K = 32 (32 B) per MMA
                                mma_f8_ss_2sm(d, a8l + kk * 2, b8h + kk * 2, idesc, 1);
                                mma_f8_ss_2sm(d, a8h + kk * 2, b8l + kk * 2, idesc, 1);
                            }
                        } else {
                            const uint64_t a0 = desc_sw128(st);
                            const uint64_t a1 = desc_sw128(st + C::kHalf);
                            const uint64_t b0 = desc_sw128(st + NA * C::kHalf);
                            const uint64_t b1 = desc_sw128(st + (NA + 1) * C::kHalf);
#pragma unroll
                            for (int kk = 0; kk < kBK / 16; ++kk) {
                                const uint64_t off = (uint64_t)(kk * 2);
                                mma_f16_ss_2sm(d, a0 + off, b0 + off, idesc, (kb | kk) != 0);
                                if (NA > 1) mma_f16_ss_2sm(d, a1 + off, b0 + off, idesc, 1);
                                if (NB > 1) mma_f16_ss_2sm(d, a0 + off, b1 + off, idesc, 1);
                            }
                        }
                        mma_commit_2sm(&empty[stage], 0x3);
                    }
                    __syncwarp();
                    if (++stage == C::kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                if (elect_one()) mma_commit_2sm(&tfull[acc], 0x3);
                __syncwarp();
                if (++acc == 2) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
        }
    } else if (warp >= 4) {
        const uint32_t quad = warp & 3;
        const int cg = (int)(warp - 4) >> 2;
        const uint32_t tempty_leader = mapa_shared(smem_u32(&tempty[0]), 0);
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int64_t t = cluster; t < tiles; t += nclusters) {
            const int64_t m0 = (t / tiles_n) * 256 + rank * 128;
            const int64_t n0 = (t % tiles_n) * BN;
            const int64_t row = m0 + quad * 32 + lane;
            const uint32_t taddr = tmem_base + ((quad * 32) << 16) + acc * BN;
            // this warp's column group; the next chunk's TMEM load overlaps the
            // current chunk's epilogue math (double-buffered registers)
            const int cbeg = cg * (BN / kEpiGroups2), cend = cbeg + BN / kEpiGroups2;
            if (EPI == EPI_RESID) {
                // residual reads do not depend on the MMA: the first chunk's are
                // issued before waiting for the accumulator, each next chunk's
                // before the current chunk's stores
                float res[32], nxt[32];
                resid_prefetch(p, row - lane, n0 + cbeg, M, N, res);
                mbar_wait(&tfull[acc], acc_phase);
                tc_fence_after();
#pragma unroll 1
                for (int c0 = cbeg; c0 < cend; c0 += 32) {
                    uint32_t r[32];
                    tmem_ld32(taddr + c0, r);
                    if (c0 + 32 < cend) resid_prefetch(p, row - lane, n0 + c0 + 32, M, N, nxt);
                    tmem_ld_wait();
                    if (n0 + c0 < N) epilogue_resid_pref(p, row - lane, n0 + c0, M, N, r, res, stagebuf);
#pragma unroll
                    for (int u = 0; u < 32; ++u) res[u] = nxt[u];
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(tempty_leader + acc * 8);
                if (++acc == 2) {
                    acc = 0;
                    acc_phase ^= 1;
                }
                continue;
            }
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            uint32_t r[2][32];
            tmem_ld32(taddr + cbeg, r[0]);
            tmem_ld_wait();
#pragma unroll 1
            for (int c0 = cbeg; c0 < cend; c0 += 64) {
                if (c0 + 32 < cend) tmem_ld32(taddr + c0 + 32, r[1]);
                if (n0 + c0 < N) epilogue_coalesced<EPI, F8>(p, row - lane, n0 + c0, M, N, r[0], stagebuf);
                tmem_ld_wait();
                if (c0 + 32 < cend) {
                    if (c0 + 64 < cend) tmem_ld32(taddr + c0 + 64, r[0]);
                    if (n0 + c0 + 32 < N) epilogue_coalesced<EPI, F8>(p, row - lane, n0 + c0 + 32, M, N, r[1], stagebuf);
                    tmem_ld_wait();
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(tempty_leader + acc * 8);
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    }
    tc_fence_before();
    cluster_sync();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc_2sm(tmem_base, 512);
    }
}

template <int NA, int NB, int EPI, bool F8 = false>
void launch2(const GemmArgs& g, int sm_count, cudaStream_t st) {
    using C = Cfg2<NA, NB, EPI, F8>;
    auto kern = gemm2_kernel<NA, NB, EPI, F8>;
    static std::atomic<uint64_t> attr_set{0};
    if (first_on_device(attr_set)) PKV_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
    // B re-encoded with 128-row boxes (each CTA of the pair loads half of the N tile)
    CUtensorMap b[2];
    for (int q = 0; q < (F8 ? 1 : NB); ++q) {
        b[q] = make_tmap_2d(g.b_ptr[q], CU_TENSOR_MAP_DATA_TYPE_FLOAT16, (uint64_t)g.K, (uint64_t)g.N,
                            (uint64_t)g.ldb * 2, kBK, 128, CU_TENSOR_MAP_SWIZZLE_128B);
    }
    if (NB == 1) b[1] = b[0];
    CUtensorMap a2 = g.a[0], b2 = b[0];
    if (F8) {  // B planes: [0] fp16 hi, then e4m3 hi / lo (64-B rows, 128-row boxes)
        b[1] = make_tmap_2d(g.b8[0], CU_TENSOR_MAP_DATA_TYPE_UINT8, (uint64_t)g.K, (uint64_t)g.N, (uint64_t)g.K, kBK,
                            128, CU_TENSOR_MAP_SWIZZLE_64B);
        b2 = make_tmap_2d(g.b8[1], CU_TENSOR_MAP_DATA_TYPE_UINT8, (uint64_t)g.K, (uint64_t)g.N, (uint64_t)g.K, kBK, 128,
                          CU_TENSOR_MAP_SWIZZLE_64B);
        a2 = g.a8h;
    }
    const int64_t tiles = ((g.M + 255) / 256) * ((g.N + 255) / 256);
    int64_t clusters = tiles < sm_count / 2 ? tiles : sm_count / 2;
    kern<<<(unsigned)(2 * clusters), C::kThreads2, C::kSmem, st>>>(g.a[0], g.a[1], b[0], b[1], a2, b2, g.p, g.M, g.N,
                                                                   g.K);
    check_launch("gemm2_kernel");
}

template <int NA, int NB>
void dispatch2_epi(const GemmArgs& g, int sm, cudaStream_t st) {
    switch (g.epi) {
        case EPI_F32: return launch2<NA, NB, EPI_F32>(g, sm, st);
        case EPI_F16X: return launch2<NA, NB, EPI_F16X>(g, sm, st);
        case EPI_GELU_F16X: return launch2<NA, NB, EPI_GELU_F16X>(g, sm, st);
        case EPI_RESID: return launch2<NA, NB, EPI_RESID>(g, sm, st);
        case EPI_GELU_PE: return launch2<NA, NB, EPI_GELU_PE>(g, sm, st);
    }
}

void dispatch2(const GemmArgs& g, int sm, cudaStream_t st) {
    if (g.f8) {
        switch (g.epi) {
            case EPI_F16X: return launch2<2, 2, EPI_F16X, true>(g, sm, st);
            case EPI_GELU_F16X: return launch2<2, 2, EPI_GELU_F16X, true>(g, sm, st);
            case EPI_RESID: return launch2<2, 2, EPI_RESID, true>(g, sm, st);
            case EPI_GELU_PE: return launch2<2, 2, EPI_GELU_PE, true>(g, sm, st);
            default: throw Error{PKV_ECONFIG, "FP16F8 GEMM: unsupported epilogue"};
        }
    }
    if (g.na == 1 && g.nb == 1) return dispatch2_epi<1, 1>(g, sm, st);
    if (g.na == 2 && g.nb == 1) return dispatch2_epi<2, 1>(g, sm, st);
    if (g.na == 1 && g.nb == 2) return dispatch2_epi<1, 2>(g, sm, st);
    if (g.na == 2 && g.nb == 2) return dispatch2_epi<2, 2>(g, sm, st);
    throw Error{PKV_ECONFIG, cat("unsupported GEMM plane combination na=", g.na, " nb=", g.nb)};
}

}  // namespace

void gemm_set_a(GemmArgs& g, int plane, const __half* a, int64_t M, int64_t K, int64_t lda) {
    g.a[plane] = make_tmap_2d(a, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, (uint64_t)K, (uint64_t)M, (uint64_t)lda * 2, kBK, kBM,
                              CU_TENSOR_MAP_SWIZZLE_128B);
    if (plane == 0 && g.na < 1) g.na = 1;
    if (plane == 1) g.na = 2;
    g.M = M;
    g.K = K;
}

void gemm_set_b(GemmArgs& g, int plane, const __half* b, int64_t N, int64_t K, int64_t ldb) {
    g.b[plane] = make_tmap_2d(b, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, (uint64_t)K, (uint64_t)N, (uint64_t)ldb * 2, kBK,
                              (uint32_t)g.bn, CU_TENSOR_MAP_SWIZZLE_128B);
    if (plane == 1) g.nb = 2;
    g.N = N;
    g.b_ptr[plane] = b;
    g.ldb = ldb;
}

void gemm_set_a8(GemmArgs& g, const uint8_t* lo8, const uint8_t* hi8, int64_t M, int64_t K, int64_t lda) {
    g.a[1] = make_tmap_2d(lo8, CU_TENSOR_MAP_DATA_TYPE_UINT8, (uint64_t)K, (uint64_t)M, (uint64_t)lda, kBK, kBM,
                          CU_TENSOR_MAP_SWIZZLE_64B);
    g.a8h = make_tmap_2d(hi8, CU_TENSOR_MAP_DATA_TYPE_UINT8, (uint64_t)K, (uint64_t)M, (uint64_t)lda, kBK, kBM,
                         CU_TENSOR_MAP_SWIZZLE_64B);
    g.na = 2;
    g.f8 = true;
}

void gemm_set_b8(GemmArgs& g, const uint8_t* hi8, const uint8_t* lo8) {
    g.b8[0] = hi8;
    g.b8[1] = lo8;
    g.nb = 2;
}

void gemm_run(const GemmArgs& g, int sm_count, cudaStream_t st) {
    if (g.M == 0 || g.N == 0) return;
    PKV_REQUIRE(!g.f8 || g.pair, PKV_ECONFIG, "FP16F8 GEMMs run on the CTA-pair kernel (M, N >= 256)");
    if (g.pair) return dispatch2(g, sm_count, st);
    switch (g.bn) {
        case 256: return dispatch_planes<256>(g, sm_count, st);
        case 128: return dispatch_planes<128>(g, sm_count, st);
        case 64: return dispatch_planes<64>(g, sm_count, st);
        default: throw Error{PKV_ECONFIG, cat("unsupported GEMM tile N ", g.bn)};
    }
}

}  // namespace pkv
