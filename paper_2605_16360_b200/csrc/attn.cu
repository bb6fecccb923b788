// attn.cu — the mapper encoder's multi-head self-attention
// (proj/src/mapper.cpp:254-270: softmax(q·kᵀ/√64)·v, non-causal, per window),
// as a flash-style tcgen05 kernel; the N_w×N_w score matrix never leaves the SM.
//
// CTA = (256 queries = two 128-row tiles A/B, head, window); K/V tiles are
// loaded once by TMA and shared by both query tiles.
//   warp 0     TMA producer + TMEM allocator
//   warp 1     MMA issuer (one elected lane)
//   warps 2-5 / 6-9: softmax for tile A / B (one thread per query row)
// TMEM (512 columns): S_A | S_B (128 each) | O_A | O_B | P_A | P_B (64 each).
// Per key tile j and query tile t:
//   S_t = Q_t·K_jᵀ -> TMEM. The softmax warps read S once, in two 64-key
//   halves, and evaluate P = 2^(c·s − m) against the running (integer, log2)
//   max m while tracking the tile max; kPolyPairs of the 64 pairs run on the
//   FMA pipe, the rest on MUFU. P is packed to fp16 and stored to P_t with
//   tcgen05.st; O_t += P_t·V_j takes its A operand straight from TMEM, so P
//   never touches shared memory. If the tile max exceeds m by more than 2^15
//   (fp16 headroom; always on the first tile) the row max is raised, O and the
//   sum are rescaled and P is recomputed from S, which is still resident.
// Epilogue: O / l -> ctx hi/lo fp16 planes.
//
// Input: qkv fp16 [rows, 3·D] (q | k | v, head h at columns h·64 of each),
// rows = window·Lw + t. Output: ctx hi/lo fp16 planes [rows, ld_out].
#include "attn.cuh"
#include "sm100.cuh"

namespace pkv {
namespace {

using namespace sm100;

constexpr int kBQ = 128, kBK = 128, kD = 64;
constexpr int kTiles = 2;  // query tiles per CTA
constexpr int kStages = 3;
constexpr int kTileBytes = 128 * kD * 2;     // 16 KB: one Q, K or V tile
constexpr int kThreads = 64 + 128 * kTiles;  // 320 threads
constexpr int kSmem = 1024 + kTileBytes * (kTiles + 2 * kStages) + 256;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kColO = 256, kColP = 384;
constexpr float kHeadroom = 15.0f;  // P <= 2^15 < fp16 max
constexpr int kPolyPairs = 16;      // of the 32 exponential pairs per 64-key half

__device__ __forceinline__ uint32_t pack_half2(float a, float b) {
    const __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&h);
}

// 64 scores (two 32-column TMEM loads) -> 32 fp16 pairs of P = 2^(c·s − m)
// stored to TMEM at p_col; returns the raw max (or -inf) and adds Σp to acc.
template <bool kMask>
__device__ __forceinline__ float p_half(uint32_t s_col, uint32_t p_col, int valid, uint64_t cc, uint64_t nm,
                                        uint64_t mp, uint64_t& acc0, uint64_t& acc1) {
    uint32_t r[2][32];
    tmem_ld32(s_col, r[0]);
    tmem_ld32(s_col + 32, r[1]);
    tmem_ld_wait();
    if (kMask) {
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int u = 0; u < 32; ++u)
                if (c * 32 + u >= valid) r[c][u] = __float_as_uint(-INFINITY);
    }
    float mt[4];
#pragma unroll
    for (int t4 = 0; t4 < 4; ++t4) mt[t4] = fmaxf(__uint_as_float(r[0][t4]), __uint_as_float(r[0][t4 + 4]));
    uint32_t pk[16];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        const uint32_t* rr = r[i >> 4];
        const float a = __uint_as_float(rr[2 * (i & 15)]), b = __uint_as_float(rr[2 * (i & 15) + 1]);
        if (i >= 4) mt[i & 3] = max3f(mt[i & 3], a, b);
        const uint64_t s2 = pack2(a, b);
        uint64_t e;
        if (!kMask && ((i + 1) * kPolyPairs) / 32 != (i * kPolyPairs) / 32) {
            e = ex2_poly2_fused(s2, cc, mp);
        } else {
            const float2 x = unpack2(ffma2(s2, cc, nm));
            e = pack2(ex2(x.x), ex2(x.y));
        }
        if (i & 1) acc1 = fadd2(acc1, e);
        else acc0 = fadd2(acc0, e);
        const float2 ef = unpack2(e);
        pk[i & 15] = pack_half2(ef.x, ef.y);
        if ((i & 15) == 15) tmem_st16(p_col + (i & 16), pk);
    }
    return fmaxf(fmaxf(mt[0], mt[1]), fmaxf(mt[2], mt[3]));
}

__global__ void __launch_bounds__(kThreads, 1)
    attn_kernel(const __grid_constant__ CUtensorMap tqkv, __half* __restrict__ out_h, __half* __restrict__ out_l,
                int64_t ld_out, int Lw, int D, float scale_log2) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = smem;                       // [kTiles] tiles
    uint8_t* sK = sQ + kTiles * kTileBytes;   // [kStages]
    uint8_t* sV = sK + kStages * kTileBytes;  // [kStages]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sV + kStages * kTileBytes);
    uint64_t* bar_q = bars;
    uint64_t* kv_full = bars + 1;
    uint64_t* kv_empty = kv_full + kStages;
    uint64_t* s_full = kv_empty + kStages;  // [kTiles]
    uint64_t* s_empty = s_full + kTiles;    // [kTiles]
    uint64_t* p_full = s_empty + kTiles;    // [kTiles]
    uint64_t* o_done = p_full + kTiles;     // [kTiles]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + kTiles);

    const uint32_t warp = warp_id(), lane = lane_id();
    const int q0 = blockIdx.x * (kBQ * kTiles), head = blockIdx.y, win = blockIdx.z;
    const int n_kv = (Lw + kBK - 1) / kBK;

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tqkv);
        mbar_init(bar_q, 1);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&kv_full[s], 1);
            mbar_init(&kv_empty[s], 1);
        }
        for (int t = 0; t < kTiles; ++t) {
            mbar_init(&s_full[t], 1);
            mbar_init(&s_empty[t], 4);
            mbar_init(&p_full[t], 4);
            mbar_init(&o_done[t], 1);
        }
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc(tmem_slot, kTmemCols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (elect_one()) {
            mbar_arrive_expect_tx(bar_q, kTiles * kTileBytes);
            for (int t = 0; t < kTiles; ++t) tma_load_3d(sQ + t * kTileBytes, &tqkv, bar_q, head * kD, q0 + t * kBQ, win);
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
        auto issue_s = [&](int j, int t) {
            if (elect_one()) {
                const uint64_t a = desc_sw128(sQ + t * kTileBytes);
                const uint64_t b = desc_sw128(sK + (j % kStages) * kTileBytes);
#pragma unroll
                for (int kk = 0; kk < kD / 16; ++kk) mma_f16_ss(tmem + t * kBK, a + kk * 2, b + kk * 2, idesc_s, kk > 0);
                mma_commit(&s_full[t]);
            }
            __syncwarp();
        };
        mbar_wait(&kv_full[0], 0);
        tc_fence_after();
        for (int t = 0; t < kTiles; ++t) issue_s(0, t);
        for (int j = 0; j < n_kv; ++j) {
            const uint8_t* v = sV + (j % kStages) * kTileBytes;
            if (j + 1 < n_kv) mbar_wait(&kv_full[(j + 1) % kStages], ((j + 1) / kStages) & 1);
            for (int t = 0; t < kTiles; ++t) {
                if (j + 1 < n_kv) {  // S_t(j+1) as soon as the softmax has read S_t(j)
                    mbar_wait(&s_empty[t], j & 1);
                    tc_fence_after();
                    issue_s(j + 1, t);
                }
                mbar_wait(&p_full[t], j & 1);
                tc_fence_after();
                if (elect_one()) {
                    // O_t += P_t·V_j: A = P_t from TMEM (8 columns = 16 keys per MMA)
#pragma unroll
                    for (int kk = 0; kk < kBK / 16; ++kk) {
                        const uint64_t b = desc_sw128_mn(v + kk * 16 * 128, 8192);
                        mma_f16_ts(tmem + kColO + t * kD, tmem + kColP + t * 64 + kk * 8, b, idesc_o,
                                   (j > 0 || kk > 0) ? 1u : 0u);
                    }
                    mma_commit(&o_done[t]);
                    if (t == kTiles - 1) mma_commit(&kv_empty[j % kStages]);
                }
                __syncwarp();
            }
        }
    } else {
        // softmax warps 2..9: tile = (warp - 2) / 4; TMEM lane quadrant = warp % 4
        // (warps 2,3,4,5 cover quadrants 2,3,0,1 — all four row blocks of the tile)
        const int t = (int)(warp - 2) >> 2;
        const uint32_t quad = warp & 3;
        const uint32_t row = quad * 32 + lane;
        const uint32_t lane_addr = (quad * 32) << 16;
        const uint32_t s_addr = tmem + lane_addr + t * kBK;
        const uint32_t o_addr = tmem + lane_addr + kColO + t * kD;
        const uint32_t p_addr = tmem + lane_addr + kColP + t * 64;
        const uint64_t cc = pack2(scale_log2, scale_log2);
        float m = -INFINITY, l = 0.0f;  // m: integer, log2 domain (-inf before the first tile)
        for (int j = 0; j < n_kv; ++j) {
            const int valid = Lw - j * kBK;  // keys beyond are masked
            const bool tail = valid < kBK;   // uniform across the CTA
            mbar_wait(&s_full[t], j & 1);
            tc_fence_after();
            if (j > 0) mbar_wait(&o_done[t], (j - 1) & 1);  // P_t free, O_t stable
            tc_fence_after();
            float rmax;
            uint64_t acc0, acc1;
            for (int attempt = 0;; ++attempt) {
                const uint64_t nm = pack2(-m, -m), mp = pack2(12582912.0f - m, 12582912.0f - m);
                acc0 = pack2(0.0f, 0.0f);
                acc1 = acc0;
                float h0, h1;
                if (tail) {
                    h0 = p_half<true>(s_addr, p_addr, valid, cc, nm, mp, acc0, acc1);
                    h1 = p_half<true>(s_addr + 64, p_addr + 32, valid - 64, cc, nm, mp, acc0, acc1);
                } else {
                    h0 = p_half<false>(s_addr, p_addr, kBK, cc, nm, mp, acc0, acc1);
                    h1 = p_half<false>(s_addr + 64, p_addr + 32, kBK, cc, nm, mp, acc0, acc1);
                }
                rmax = fmaxf(h0, h1) * scale_log2;
                // warp-uniform (tcgen05.ld/st are warp-collective): raise the
                // running max if any row's P would exceed the fp16 headroom
                if (!__any_sync(0xffffffffu, rmax > m + kHeadroom) || attempt > 0) break;
                const float mn = fmaxf(m, ceilf(rmax));
                const float alpha = ex2(m - mn);  // 0 when m = -inf
                l *= alpha;
                m = mn;
                if (j > 0) {
#pragma unroll
                    for (int c = 0; c < kD; c += 32) {
                        uint32_t o[32];
                        tmem_ld32(o_addr + c, o);
                        tmem_ld_wait();
#pragma unroll
                        for (int u = 0; u < 32; ++u) o[u] = __float_as_uint(__uint_as_float(o[u]) * alpha);
                        tmem_st32(o_addr + c, o);
                    }
                }
            }
            const float2 rs = unpack2(fadd2(acc0, acc1));
            l += rs.x + rs.y;
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&s_empty[t]);
                mbar_arrive(&p_full[t]);
            }
        }
        mbar_wait(&o_done[t], (n_kv - 1) & 1);
        tc_fence_after();
        const int qrow = q0 + t * kBQ + (int)row;
        const float inv = 1.0f / l;
        const int64_t base = ((int64_t)win * Lw + qrow) * ld_out + head * kD;
#pragma unroll
        for (int c0 = 0; c0 < kD; c0 += 32) {
            uint32_t o[32];
            tmem_ld32(o_addr + c0, o);
            tmem_ld_wait();
            if (qrow < Lw) {
#pragma unroll
                for (int c = 0; c < 32; c += 8) {
                    __align__(16) __half hi[8];
                    __align__(16) __half lo[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        const float v = __uint_as_float(o[c + e]) * inv;
                        hi[e] = __float2half_rn(v);
                        lo[e] = __float2half_rn(v - __half2float(hi[e]));
                    }
                    *reinterpret_cast<uint4*>(out_h + base + c0 + c) = *reinterpret_cast<const uint4*>(hi);
                    if (out_l) *reinterpret_cast<uint4*>(out_l + base + c0 + c) = *reinterpret_cast<const uint4*>(lo);
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
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
    const dim3 grid((unsigned)((Lw + kBQ * kTiles - 1) / (kBQ * kTiles)), (unsigned)heads, (unsigned)nwin);
    const float scale_log2 = 1.4426950408889634f / sqrtf((float)kD);
    attn_kernel<<<grid, kThreads, kSmem, st>>>(t, out_h, out_l, ld_out, (int)Lw, (int)D, scale_log2);
    check_launch("attn_kernel");
}

}  // namespace pkv
