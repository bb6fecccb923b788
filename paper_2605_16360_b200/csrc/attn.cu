// attn.cu — the mapper encoder's multi-head self-attention
// (proj/src/mapper.cpp:254-270: softmax(q·kᵀ/√64)·v, non-causal, per window),
// as a flash-style tcgen05 kernel: S = Q·Kᵀ into TMEM, online softmax in
// registers (one thread per query row), P (fp16) staged to swizzled smem,
// O_tile = P·V into TMEM, rescaled accumulation in registers. The N_w×N_w
// score matrix is never materialised.
//
// Input: qkv fp16 [rows, 3·D] (q | k | v, head h at columns h·64 of each),
// rows = window·Lw + t. Output: ctx hi/lo fp16 planes [rows, D].
//
// CTA = (query tile of 128 rows, head, window). Warps: 0 TMA, 1 MMA, 2 TMEM
// alloc, 4-7 softmax/epilogue.
#include "attn.cuh"
#include "sm100.cuh"

namespace pkv {
namespace {

using namespace sm100;

constexpr int kBQ = 128, kBK = 128, kD = 64;
constexpr int kStages = 3;
constexpr int kTileBytes = 128 * kD * 2;  // 16 KB: Q, K or V tile
constexpr int kPBytes = kBQ * kBK * 2;    // 32 KB: two 64-key swizzle panels
constexpr int kThreads = 256;
constexpr int kSmem = 1024 + kTileBytes * (1 + 2 * kStages) + kPBytes + 256;
constexpr uint32_t kTmemCols = 512;  // S[2] (2x128) + O (64)
constexpr uint32_t kColO = 256;

// Byte offset of fp16 element (row, col) in a K-major, 128-B-swizzled panel
// (rows of 128 B; 16-B chunk index XOR (row % 8)).
__device__ __forceinline__ uint32_t sw128_off(uint32_t row, uint32_t col) {
    const uint32_t chunk = (col >> 3) ^ (row & 7);
    return row * 128 + chunk * 16 + (col & 7) * 2;
}

__global__ void __launch_bounds__(kThreads, 1)
    attn_kernel(const __grid_constant__ CUtensorMap tqkv, __half* __restrict__ out_h, __half* __restrict__ out_l,
                int64_t ld_out, int Lw, int D, float scale_log2) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = smem;
    uint8_t* sK = sQ + kTileBytes;
    uint8_t* sV = sK + kStages * kTileBytes;
    uint8_t* sP = sV + kStages * kTileBytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sP + kPBytes);
    uint64_t* bar_q = bars;
    uint64_t* kv_full = bars + 1;
    uint64_t* kv_empty = kv_full + kStages;
    uint64_t* s_full = kv_empty + kStages;
    uint64_t* s_empty = s_full + 2;
    uint64_t* p_full = s_empty + 2;
    uint64_t* o_full = p_full + 1;
    uint64_t* o_empty = o_full + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_empty + 1);

    const uint32_t warp = warp_id(), lane = lane_id();
    const int q0 = blockIdx.x * kBQ, head = blockIdx.y, win = blockIdx.z;
    const int n_kv = (Lw + kBK - 1) / kBK;

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tqkv);
        mbar_init(bar_q, 1);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&kv_full[s], 1);
            mbar_init(&kv_empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&s_full[s], 1);
            mbar_init(&s_empty[s], 4);
        }
        mbar_init(p_full, 4);
        mbar_init(o_full, 1);
        mbar_init(o_empty, 4);
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc(tmem_slot, kTmemCols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (elect_one()) {
            mbar_arrive_expect_tx(bar_q, kTileBytes);
            tma_load_3d(sQ, &tqkv, bar_q, head * kD, q0, win);
            for (int j = 0; j < n_kv; ++j) {
                const int st = j % kStages;
                mbar_wait(&kv_empty[st], ((j / kStages) & 1) ^ 1);
                mbar_arrive_expect_tx(&kv_full[st], 2 * kTileBytes);
                tma_load_3d(sK + st * kTileBytes, &tqkv, &kv_full[st], D + head * kD, j * kBK, win);
                tma_load_3d(sV + st * kTileBytes, &tqkv, &kv_full[st], 2 * D + head * kD, j * kBK, win);
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t idesc_s = idesc_f16(kBQ, kBK, 0);
        constexpr uint32_t idesc_o = idesc_f16(kBQ, kD, 0, 0, 1);  // B (V) is MN-major
        mbar_wait(bar_q, 0);
        auto do_pv = [&](int i) {
            mbar_wait(p_full, i & 1);
            mbar_wait(o_empty, (i & 1) ^ 1);
            tc_fence_after();
            if (elect_one()) {
                const uint8_t* v = sV + (i % kStages) * kTileBytes;
#pragma unroll
                for (int kk = 0; kk < kBK / 16; ++kk) {
                    const uint64_t a = desc_sw128(sP + (kk >> 2) * (kPBytes / 2)) + (uint64_t)((kk & 3) * 2);
                    const uint64_t b = desc_sw128_mn(v + kk * 16 * 128, 8192);
                    mma_f16_ss(tmem + kColO, a, b, idesc_o, kk > 0);
                }
                mma_commit(o_full);
                mma_commit(&kv_empty[i % kStages]);
            }
            __syncwarp();
        };
        for (int j = 0; j < n_kv; ++j) {
            const int st = j % kStages, sb = j & 1;
            mbar_wait(&kv_full[st], (j / kStages) & 1);
            mbar_wait(&s_empty[sb], ((j >> 1) & 1) ^ 1);
            tc_fence_after();
            if (elect_one()) {
                const uint64_t a = desc_sw128(sQ);
                const uint64_t b = desc_sw128(sK + st * kTileBytes);
#pragma unroll
                for (int kk = 0; kk < kD / 16; ++kk) {
                    mma_f16_ss(tmem + sb * kBK, a + kk * 2, b + kk * 2, idesc_s, kk > 0);
                }
                mma_commit(&s_full[sb]);
            }
            __syncwarp();
            if (j >= 1) do_pv(j - 1);
        }
        do_pv(n_kv - 1);
    } else if (warp >= 4) {
        const uint32_t quad = warp & 3;
        const uint32_t row = quad * 32 + lane;
        const uint32_t lane_addr = (quad * 32) << 16;
        float m = -INFINITY, l = 0.0f;
        float o[kD];
#pragma unroll
        for (int c = 0; c < kD; ++c) o[c] = 0.0f;
        for (int j = 0; j < n_kv; ++j) {
            const int sb = j & 1;
            const int valid = Lw - j * kBK;  // keys beyond are masked
            mbar_wait(&s_full[sb], (j >> 1) & 1);
            tc_fence_after();
            const uint32_t sbase = tmem + lane_addr + sb * kBK;
            float tmax = -INFINITY;
#pragma unroll
            for (int c0 = 0; c0 < kBK; c0 += 32) {
                uint32_t r[32];
                tmem_ld32(sbase + c0, r);
                tmem_ld_wait();
#pragma unroll
                for (int t = 0; t < 32; t += 2) {
                    const float a = (c0 + t < valid) ? __uint_as_float(r[t]) : -INFINITY;
                    const float b = (c0 + t + 1 < valid) ? __uint_as_float(r[t + 1]) : -INFINITY;
                    tmax = max3f(tmax, a, b);
                }
            }
            const float mx = fmaxf(m, tmax * scale_log2);
            const float alpha = ex2(m - mx);
            float rs = 0.0f;
#pragma unroll
            for (int c0 = 0; c0 < kBK; c0 += 32) {
                uint32_t r[32];
                tmem_ld32(sbase + c0, r);
                tmem_ld_wait();
                uint8_t* panel = sP + (c0 >> 6) * (kPBytes / 2);
#pragma unroll
                for (int t = 0; t < 32; t += 8) {
                    __align__(16) __half2 h[4];
#pragma unroll
                    for (int u = 0; u < 8; u += 2) {
                        const int c = c0 + t + u;
                        const float p0 = (c < valid) ? ex2(fmaf(__uint_as_float(r[t + u]), scale_log2, -mx)) : 0.0f;
                        const float p1 = (c + 1 < valid) ? ex2(fmaf(__uint_as_float(r[t + u + 1]), scale_log2, -mx)) : 0.0f;
                        const __half2 hp = __floats2half2_rn(p0, p1);
                        const float2 back = __half22float2(hp);
                        rs += back.x + back.y;
                        h[u >> 1] = hp;
                    }
                    *reinterpret_cast<uint4*>(panel + sw128_off(row, (c0 & 63) + t)) = *reinterpret_cast<uint4*>(h);
                }
            }
            tc_fence_before();
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&s_empty[sb]);
                mbar_arrive(p_full);
            }
            l = l * alpha + rs;
            mbar_wait(o_full, j & 1);
            tc_fence_after();
#pragma unroll
            for (int c0 = 0; c0 < kD; c0 += 32) {
                uint32_t r[32];
                tmem_ld32(tmem + lane_addr + kColO + c0, r);
                tmem_ld_wait();
#pragma unroll
                for (int t = 0; t < 32; ++t) o[c0 + t] = fmaf(o[c0 + t], alpha, __uint_as_float(r[t]));
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(o_empty);
            m = mx;
        }
        if (q0 + (int)row < Lw) {
            const float inv = 1.0f / l;
            const int64_t base = ((int64_t)win * Lw + q0 + row) * ld_out + head * kD;
#pragma unroll
            for (int c = 0; c < kD; c += 8) {
                __align__(16) __half hi[8];
                __align__(16) __half lo[8];
#pragma unroll
                for (int t = 0; t < 8; ++t) {
                    const float v = o[c + t] * inv;
                    hi[t] = __float2half_rn(v);
                    lo[t] = __float2half_rn(v - __half2float(hi[t]));
                }
                *reinterpret_cast<uint4*>(out_h + base + c) = *reinterpret_cast<const uint4*>(hi);
                if (out_l) *reinterpret_cast<uint4*>(out_l + base + c) = *reinterpret_cast<const uint4*>(lo);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem, kTmemCols);
    }
}

}  // namespace

void launch_encoder_attention(const __half* qkv, int64_t nwin, int64_t Lw, int64_t D, int64_t heads, __half* out_h,
                              __half* out_l, int64_t ld_out, cudaStream_t st) {
    PKV_REQUIRE(D == heads * kD, PKV_ECONFIG, "GPU encoder attention needs d_time / encoder_heads == 64, got ", D,
                "/", heads);
    PKV_REQUIRE(nwin <= 65535, PKV_ECONFIG, "too many windows per launch: ", nwin);
    static bool attr = false;
    if (!attr) {
        PKV_CUDA(cudaFuncSetAttribute(attn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
        attr = true;
    }
    const CUtensorMap t = make_tmap_3d(qkv, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, (uint64_t)(3 * D), (uint64_t)Lw,
                                       (uint64_t)nwin, (uint64_t)(3 * D) * 2, (uint64_t)(3 * D) * 2 * Lw, kD, 128, 1,
                                       CU_TENSOR_MAP_SWIZZLE_128B);
    const dim3 grid((unsigned)((Lw + kBQ - 1) / kBQ), (unsigned)heads, (unsigned)nwin);
    const float scale_log2 = 1.4426950408889634f / sqrtf((float)kD);
    attn_kernel<<<grid, kThreads, kSmem, st>>>(t, out_h, out_l, ld_out, (int)Lw, (int)D, scale_log2);
    check_launch("attn_kernel");
}

}  // namespace pkv
