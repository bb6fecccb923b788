// attn.cu — the mapper encoder's multi-head self-attention
// (proj/src/mapper.cpp:254-270: softmax(q·kᵀ/√64)·v, non-causal, per window),
// as a flash-style tcgen05 kernel; the N_w×N_w score matrix never leaves the SM.
//
// CTA = (256 queries = two 128-row tiles A/B, head, window); K/V tiles are
// loaded once by TMA and shared by both query tiles.
//   warp 0     TMA producer          warp 1   MMA issuer (one elected lane)
//   warp 0 also allocates TMEM;       warps 2-5 / 6-9: softmax for tile A / B
// Per key tile j and query tile t:
//   S_t = Q_t·K_jᵀ -> TMEM; softmax warps (one thread per row) load the row,
//   compute P = 2^(c·s − m) with a lazily updated running max m (rescale O
//   only when the row max grows by > 2^8, FA4-style), 1 in 4 exponentials on
//   the FMA pipe; P (fp16) -> swizzled smem; O_t += P·V_j accumulates in TMEM.
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
constexpr int kTileBytes = 128 * kD * 2;  // 16 KB: one Q, K or V tile
constexpr int kPBytes = kBQ * kBK * 2;    // 32 KB: two 64-key swizzle panels
constexpr int kThreads = 64 + 128 * kTiles;  // 320 threads -> up to 204 registers per thread
constexpr int kSmem = 1024 + kTileBytes * (kTiles + 2 * kStages) + kTiles * kPBytes + 256;
constexpr uint32_t kTmemCols = 512;  // S_A, S_B (128 each) | O_A, O_B (64 each)
constexpr uint32_t kColO = 256;
constexpr float kRescale = 8.0f;  // log2 of the lazy-rescale threshold

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
    uint8_t* sQ = smem;                          // [kTiles] tiles
    uint8_t* sK = sQ + kTiles * kTileBytes;      // [kStages]
    uint8_t* sV = sK + kStages * kTileBytes;     // [kStages]
    uint8_t* sP = sV + kStages * kTileBytes;     // [kTiles] x 32 KB
    uint64_t* bars = reinterpret_cast<uint64_t*>(sP + kTiles * kPBytes);
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
            const int st = j % kStages;
            mbar_wait(&s_empty[t], (j & 1) ^ 1);
            tc_fence_after();
            if (elect_one()) {
                const uint64_t a = desc_sw128(sQ + t * kTileBytes);
                const uint64_t b = desc_sw128(sK + st * kTileBytes);
#pragma unroll
                for (int kk = 0; kk < kD / 16; ++kk) mma_f16_ss(tmem + t * kBK, a + kk * 2, b + kk * 2, idesc_s, kk > 0);
                mma_commit(&s_full[t]);
            }
            __syncwarp();
        };
        auto issue_pv = [&](int j, int t) {
            mbar_wait(&p_full[t], j & 1);
            tc_fence_after();
            if (elect_one()) {
                const uint8_t* v = sV + (j % kStages) * kTileBytes;
                const uint8_t* p = sP + t * kPBytes;
#pragma unroll
                for (int kk = 0; kk < kBK / 16; ++kk) {
                    const uint64_t a = desc_sw128(p + (kk >> 2) * (kPBytes / 2)) + (uint64_t)((kk & 3) * 2);
                    const uint64_t b = desc_sw128_mn(v + kk * 16 * 128, 8192);
                    mma_f16_ss(tmem + kColO + t * kD, a, b, idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
                }
                mma_commit(&o_done[t]);
            }
            __syncwarp();
        };
        mbar_wait(&kv_full[0], 0);
        for (int t = 0; t < kTiles; ++t) issue_s(0, t);
        for (int j = 0; j < n_kv; ++j) {
            if (j + 1 < n_kv) {
                mbar_wait(&kv_full[(j + 1) % kStages], ((j + 1) / kStages) & 1);
                for (int t = 0; t < kTiles; ++t) issue_s(j + 1, t);
            }
            for (int t = 0; t < kTiles; ++t) issue_pv(j, t);
            if (elect_one()) mma_commit(&kv_empty[j % kStages]);
            __syncwarp();
        }
    } else {
        // softmax warps 2..9: tile = (warp - 2) / 4; TMEM lane quadrant = warp % 4
        // (warps 2,3,4,5 cover quadrants 2,3,0,1 — all four rows blocks of the tile)
        const int t = (int)(warp - 2) >> 2;
        const uint32_t quad = warp & 3;
        const uint32_t row = quad * 32 + lane;
        const uint32_t lane_addr = (quad * 32) << 16;
        const uint32_t s_addr = tmem + lane_addr + t * kBK;
        const uint32_t o_addr = tmem + lane_addr + kColO + t * kD;
        uint8_t* pbuf = sP + t * kPBytes;
        float m = -INFINITY, l = 0.0f;
        for (int j = 0; j < n_kv; ++j) {
            const int valid = Lw - j * kBK;  // keys beyond are masked
            mbar_wait(&s_full[t], j & 1);
            tc_fence_after();
            const bool tail = __any_sync(0xffffffffu, valid < kBK);  // warp-uniform: only the last key tile
            // pass A: row max straight from TMEM (S stays there for pass B; keeps
            // register pressure to 64 S values per thread)
            float mt[8];
#pragma unroll
            for (int t8 = 0; t8 < 8; ++t8) mt[t8] = -INFINITY;
#pragma unroll
            for (int c = 0; c < 4; c += 2) {
                uint32_t r[2][32];
                tmem_ld32(s_addr + c * 32, r[0]);
                tmem_ld32(s_addr + (c + 1) * 32, r[1]);
                tmem_ld_wait();
#pragma unroll
                for (int h2 = 0; h2 < 2; ++h2) {
                    if (tail) {
#pragma unroll
                        for (int u = 0; u < 32; ++u)
                            if ((c + h2) * 32 + u >= valid) r[h2][u] = __float_as_uint(-INFINITY);
                    }
#pragma unroll
                    for (int u = 0; u < 32; u += 16)
#pragma unroll
                        for (int t8 = 0; t8 < 8; ++t8)
                            mt[t8] = max3f(mt[t8], __uint_as_float(r[h2][u + t8]), __uint_as_float(r[h2][u + t8 + 8]));
                }
            }
            float tmax = max3f(max3f(mt[0], mt[1], mt[2]), max3f(mt[3], mt[4], mt[5]), fmaxf(mt[6], mt[7]));
            tmax *= scale_log2;
            // lazy rescale: warp-uniform decision (tcgen05.ld/st are warp-collective)
            const bool need = tmax > m + kRescale;
            if (__any_sync(0xffffffffu, need)) {
                const float mn = fmaxf(m, tmax);
                const float alpha = ex2(m - mn);  // 0 when m = -inf
                l *= alpha;
                m = mn;
                if (j > 0) {
                    mbar_wait(&o_done[t], (j - 1) & 1);  // O holds P(<j)·V, stable
                    tc_fence_after();
#pragma unroll
                    for (int c = 0; c < kD; c += 32) {
                        uint32_t o[32];
                        tmem_ld32(o_addr + c, o);
                        tmem_ld_wait();
#pragma unroll
                        for (int u = 0; u < 32; ++u) o[u] = __float_as_uint(__uint_as_float(o[u]) * alpha);
                        tmem_st32(o_addr + c, o);
                    }
                    tmem_st_wait();
                }
            }
            // P = 2^(c·s − m) <= 2^8, rounded to fp16 and staged for P·V
            if (j > 0) mbar_wait(&o_done[t], (j - 1) & 1);  // P buffer free (PV(j-1) done)
            // packed fp32x2 arguments/sums; 1 pair in 4 via the FMA-pipe polynomial
            const uint64_t cc = pack2(scale_log2, scale_log2), nm = pack2(-m, -m);
            uint64_t acc0 = pack2(0.0f, 0.0f), acc1 = acc0;
            // pass B: re-read S in two 64-column halves
#pragma unroll
            for (int c2 = 0; c2 < 4; c2 += 2) {
                uint32_t r[2][32];
                tmem_ld32(s_addr + c2 * 32, r[0]);
                tmem_ld32(s_addr + (c2 + 1) * 32, r[1]);
                tmem_ld_wait();
                if (tail) {
#pragma unroll
                    for (int h2 = 0; h2 < 2; ++h2)
#pragma unroll
                        for (int u = 0; u < 32; ++u)
                            if ((c2 + h2) * 32 + u >= valid) r[h2][u] = __float_as_uint(-INFINITY);
                }
                uint8_t* panel = pbuf + (c2 >> 1) * (kPBytes / 2);
#pragma unroll
                for (int h2 = 0; h2 < 2; ++h2) {
#pragma unroll
                    for (int u = 0; u < 32; u += 8) {
                        __align__(16) __half2 h[4];
#pragma unroll
                        for (int e = 0; e < 8; e += 2) {
                            const uint64_t a = ffma2(
                                pack2(__uint_as_float(r[h2][u + e]), __uint_as_float(r[h2][u + e + 1])), cc, nm);
                            uint64_t pe;
                            if (e == 6) {
                                pe = ex2_poly2_d3(a);
                            } else {
                                const float2 x = unpack2(a);
                                pe = pack2(ex2(x.x), ex2(x.y));
                            }
                            if (e & 2) acc1 = fadd2(acc1, pe);
                            else acc0 = fadd2(acc0, pe);
                            const float2 pf = unpack2(pe);
                            h[e >> 1] = __floats2half2_rn(pf.x, pf.y);
                        }
                        *reinterpret_cast<uint4*>(panel + sw128_off(row, h2 * 32 + u)) = *reinterpret_cast<uint4*>(h);
                    }
                }
            }
            const float2 rs = unpack2(fadd2(acc0, acc1));
            l += rs.x + rs.y;
            tc_fence_before();
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_empty[t]);  // S fully consumed (both passes)
            if (lane == 0) mbar_arrive(&p_full[t]);
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
