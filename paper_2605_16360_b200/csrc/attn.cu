// attn.cu — the mapper encoder's multi-head self-attention
// (proj/src/mapper.cpp:254-270: softmax(q·kᵀ/√64)·v, non-causal, per window),
// as a flash-style tcgen05 kernel; the N_w×N_w score matrix never leaves the SM.
//
// CTA = (256 queries = two 128-row tiles A/B, head, window); 64-key K/V tiles
// are loaded once by TMA and shared by both query tiles.
//   warp 0      TMA producer + TMEM allocator
//   warps 1, 2  MMA issuers for tile A, B (independent chains)
//   warps 3-6 / 7-10: softmax for tile A / B (one thread per query row)
// TMEM (512 columns): per tile three 64-column S/P buffers and a 64-column O.
// Per key tile j and query tile t, in buffer j % 3:
//   S = Q_t·K_jᵀ; issued two key tiles ahead (as soon as P·V_{j-3} has
//   released the buffer), so the tensor-core latency is off the softmax's path.
//   The softmax warps read S once into registers and evaluate P = 2^(c·s − m)
//   against the running (integer, log2) max m while tracking the tile max;
//   kPolyPairs of the 32 pairs run on the FMA pipe, the rest on MUFU. P is
//   packed to fp16 and written over the first 32 columns of the same buffer
//   (tcgen05.st); O_t += P·V_j takes its A operand straight from TMEM, so P
//   never touches shared memory. If the tile max exceeds m by more than 2^15
//   (fp16 headroom; always on the first tile) the row max is raised, O and the
//   sum are rescaled and P is recomputed from the register copy of S.
// Epilogue: O / l -> ctx hi/lo fp16 planes.
//
// Input: qkv fp16 [rows, 3·D] (q | k | v, head h at columns h·64 of each),
// rows = window·Lw + t. Output: ctx hi/lo fp16 planes [rows, ld_out].
#include <cstdlib>

#include "attn.cuh"
#include "sm100.cuh"

namespace pkv {
namespace {

using namespace sm100;

constexpr int kBQ = 128, kBK = 64, kD = 64;
constexpr int kTiles = 1;  // query tiles per CTA (two CTAs per SM)
constexpr int kBufs = 3;   // S/P buffers per tile
constexpr int kStages = 5;
constexpr int kQBytes = kBQ * kD * 2;   // 16 KB
constexpr int kKVBytes = kBK * kD * 2;  // 8 KB: one K or V tile
constexpr int kThreads = 32 * (1 + kTiles) + 128 * kTiles;
constexpr int kSmem = 1024 + kQBytes * kTiles + 2 * kKVBytes * kStages + 512;
constexpr uint32_t kTmemCols = kTiles == 1 ? 256 : 512;
constexpr uint32_t kColO = kTiles * kBufs * 64;
constexpr float kHeadroom = 15.0f;  // P <= 2^15 < fp16 max

__device__ __forceinline__ uint32_t pack_half2(float a, float b) {
    const __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&h);
}

// 32 scores of one row (registers) -> 16 fp16 pairs of P = 2^(c·s − m)
// stored to TMEM at p_col (16 columns); returns the raw max (or -inf) of the
// chunk and adds Σp to acc. kBase: index of the chunk's first pair within the
// 64-key tile (for the MUFU/FMA interleave and the tail mask).
template <bool kMask, int kMode, int kPolyPairs>
__device__ __forceinline__ float p_chunk(const uint32_t (&r)[32], int kbase, uint32_t p_col, int valid, uint64_t cc,
                                         uint64_t nm, uint64_t mp, uint64_t& acc0, uint64_t& acc1) {
    float mt[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
    uint32_t pk[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        float a = __uint_as_float(r[2 * i]), b = __uint_as_float(r[2 * i + 1]);
        if (kMask) {
            a = kbase + 2 * i < valid ? a : -INFINITY;
            b = kbase + 2 * i + 1 < valid ? b : -INFINITY;
        }
        if (kMode == 1) {  // timing probe: P = fp16(s), no exponentials
            pk[i] = pack_half2(a, b);
        } else {
            mt[i & 3] = max3f(mt[i & 3], a, b);
            const uint64_t s2 = pack2(a, b);
            uint64_t e;
            if (!kMask && ((i + 1) * kPolyPairs) / 16 != (i * kPolyPairs) / 16) {
                e = ex2_poly2_fused(s2, cc, mp);
            } else {
                const float2 x = unpack2(ffma2(s2, cc, nm));
                e = pack2(ex2(x.x), ex2(x.y));
            }
            if (i & 1) acc1 = fadd2(acc1, e);
            else acc0 = fadd2(acc0, e);
            const float2 ef = unpack2(e);
            pk[i] = pack_half2(ef.x, ef.y);
        }
    }
    tmem_st16(p_col, pk);
    return fmaxf(fmaxf(mt[0], mt[1]), fmaxf(mt[2], mt[3]));
}

// P for a whole 64-key tile from its two register chunks.
template <int kMode, int kPolyPairs>
__device__ __forceinline__ float p_tile(const uint32_t (&ra)[32], const uint32_t (&rb)[32], uint32_t p_col, bool tail,
                                        int valid, uint64_t cc, uint64_t nm, uint64_t mp, uint64_t& acc0,
                                        uint64_t& acc1) {
    if (tail) {
        const float h0 = p_chunk<true, kMode, kPolyPairs>(ra, 0, p_col, valid, cc, nm, mp, acc0, acc1);
        return fmaxf(h0, p_chunk<true, kMode, kPolyPairs>(rb, 32, p_col + 16, valid, cc, nm, mp, acc0, acc1));
    }
    const float h0 = p_chunk<false, kMode, kPolyPairs>(ra, 0, p_col, 64, cc, nm, mp, acc0, acc1);
    return fmaxf(h0, p_chunk<false, kMode, kPolyPairs>(rb, 32, p_col + 16, 64, cc, nm, mp, acc0, acc1));
}

template <int kMode, int kPolyPairs>
__global__ void __launch_bounds__(kThreads, 2 / kTiles)
    attn_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tkv, __half* __restrict__ out_h,
                __half* __restrict__ out_l, int64_t ld_out, int Lw, int D, float scale_log2) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = smem;                     // [kTiles] tiles
    uint8_t* sK = sQ + kTiles * kQBytes;    // [kStages]
    uint8_t* sV = sK + kStages * kKVBytes;  // [kStages]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sV + kStages * kKVBytes);
    uint64_t* bar_q = bars;
    uint64_t* kv_full = bars + 1;
    uint64_t* kv_empty = kv_full + kStages;
    uint64_t* s_full = kv_empty + kStages;        // [kTiles][kBufs]
    uint64_t* p_full = s_full + kTiles * kBufs;   // [kTiles][kBufs]
    uint64_t* pv_done = p_full + kTiles * kBufs;  // [kTiles][kBufs]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_done + kTiles * kBufs);

    const uint32_t warp = warp_id(), lane = lane_id();
    const int q0 = blockIdx.x * (kBQ * kTiles), head = blockIdx.y, win = blockIdx.z;
    const int n_kv = (Lw + kBK - 1) / kBK;

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tq);
        tma_prefetch(&tkv);
        mbar_init(bar_q, 1);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&kv_full[s], 1);
            mbar_init(&kv_empty[s], kTiles);
        }
        for (int i = 0; i < kTiles * kBufs; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&p_full[i], 4);
            mbar_init(&pv_done[i], 1);
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
            mbar_arrive_expect_tx(bar_q, kTiles * kQBytes);
            for (int t = 0; t < kTiles; ++t) tma_load_3d(sQ + t * kQBytes, &tq, bar_q, head * kD, q0 + t * kBQ, win);
            for (int j = 0; j < n_kv; ++j) {
                const int st = j % kStages;
                mbar_wait(&kv_empty[st], ((j / kStages) & 1) ^ 1);
                mbar_arrive_expect_tx(&kv_full[st], 2 * kKVBytes);
                tma_load_3d(sK + st * kKVBytes, &tkv, &kv_full[st], D + head * kD, j * kBK, win);
                tma_load_3d(sV + st * kKVBytes, &tkv, &kv_full[st], 2 * D + head * kD, j * kBK, win);
            }
            // drain: observe the last stages' release too (every mbarrier phase
            // the MMA warps complete is waited on before the CTA exits)
            for (int j = n_kv > kStages ? n_kv - kStages : 0; j < n_kv; ++j)
                mbar_wait(&kv_empty[j % kStages], (j / kStages) & 1);
        }
    } else if (warp <= kTiles) {
        // MMA issuer of tile t = warp - 1
        const int t = (int)warp - 1;
        constexpr uint32_t idesc_s = idesc_f16(kBQ, kBK, 0);
        constexpr uint32_t idesc_o = idesc_f16(kBQ, kD, 0, 0, 1);  // B (V) is MN-major
        const uint32_t buf0 = tmem + t * kBufs * 64;
        const uint32_t o_col = tmem + kColO + t * kD;
        uint64_t* sf = s_full + t * kBufs;
        uint64_t* pf = p_full + t * kBufs;
        uint64_t* pd = pv_done + t * kBufs;
        mbar_wait(bar_q, 0);
        auto issue_s = [&](int j) {  // S -> buffer j % 3
            const int st = j % kStages, b = j % kBufs;
            mbar_wait(&kv_full[st], (j / kStages) & 1);
            tc_fence_after();
            if (elect_one()) {
                const uint64_t a = desc_sw128(sQ + t * kQBytes);
                const uint64_t bk = desc_sw128(sK + st * kKVBytes);
#pragma unroll
                for (int kk = 0; kk < kD / 16; ++kk) mma_f16_ss(buf0 + b * 64, a + kk * 2, bk + kk * 2, idesc_s, kk > 0);
                mma_commit(&sf[b]);
            }
            __syncwarp();
        };
        for (int j = 0; j < kBufs && j < n_kv; ++j) issue_s(j);
        for (int j = 0; j < n_kv; ++j) {
            const int b = j % kBufs;
            mbar_wait(&pf[b], (j / kBufs) & 1);
            tc_fence_after();
            if (elect_one()) {
                const uint8_t* v = sV + (j % kStages) * kKVBytes;
                // O_t += P·V_j: A = P (buffer columns [0, 32)) from TMEM, 16 keys per MMA
#pragma unroll
                for (int kk = 0; kk < kBK / 16; ++kk) {
                    const uint64_t bv = desc_sw128_mn(v + kk * 16 * 128, 8192);
                    mma_f16_ts(o_col, buf0 + b * 64 + kk * 8, bv, idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
                }
                mma_commit(&pd[b]);
                mma_commit(&kv_empty[j % kStages]);
            }
            __syncwarp();
            // S_{j+3} reuses this buffer right behind P·V_j: tcgen05.mma from one
            // thread execute in issue order, so P is read before S overwrites it
            if (j + kBufs < n_kv) issue_s(j + kBufs);
        }
        } else {
        // softmax warps (kTiles + 1) ...: tile = (warp - kTiles - 1) / 4; TMEM lane quadrant = warp % 4
        const int t = (int)(warp - kTiles - 1) >> 2;
        const uint32_t quad = warp & 3;
        const uint32_t row = quad * 32 + lane;
        const uint32_t lane_addr = (quad * 32) << 16;
        const uint32_t buf0 = tmem + lane_addr + t * kBufs * 64;
        const uint32_t o_addr = tmem + lane_addr + kColO + t * kD;
        uint64_t* sf = s_full + t * kBufs;
        uint64_t* pf = p_full + t * kBufs;
        uint64_t* pd = pv_done + t * kBufs;
        const uint64_t cc = pack2(scale_log2, scale_log2);
        float m = -INFINITY, l = 0.0f;  // m: integer, log2 domain (-inf before the first tile)
        // P(j) goes to the MMA warp (wait::st + arrive) as soon as it is stored;
        // then the next tile's S (issued three tiles ahead) is read back.
        uint32_t ra[32], rb[32];
        mbar_wait(&sf[0], 0);
        tc_fence_after();
        tmem_ld32(buf0, ra);
        tmem_ld32(buf0 + 32, rb);
        tmem_ld_wait();
        for (int j = 0; j < n_kv; ++j) {
            const int b = j % kBufs;
            const uint32_t s_addr = buf0 + b * 64;
            const int valid = Lw - j * kBK;  // keys beyond are masked
            const bool tail = valid < kBK;   // uniform across the CTA
            uint64_t acc0, acc1;
            for (int attempt = 0;; ++attempt) {
                const uint64_t nm = pack2(-m, -m), mp = pack2(12582912.0f - m, 12582912.0f - m);
                acc0 = pack2(0.0f, 0.0f);
                acc1 = acc0;
                const float h = p_tile<kMode, kPolyPairs>(ra, rb, s_addr, tail, valid, cc, nm, mp, acc0, acc1);
                if (kMode == 1) break;
                const float rmax = h * scale_log2;
                // warp-uniform (tcgen05.ld/st are warp-collective): raise the
                // running max if any row's P would exceed the fp16 headroom
                if (!__any_sync(0xffffffffu, rmax > m + kHeadroom) || attempt > 0) break;
                const float mn = fmaxf(m, ceilf(rmax));
                const float alpha = ex2(m - mn);  // 0 when m = -inf
                l *= alpha;
                m = mn;
                if (j > 0) {
                    tmem_st_wait();  // P(j-1) stored and handed over below? make sure it is
                    mbar_wait(&pd[(j - 1) % kBufs], ((j - 1) / kBufs) & 1);  // O holds P(<j)·V, stable
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
                }
            }
            const float2 rs = unpack2(fadd2(acc0, acc1));
            l += rs.x + rs.y;
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&pf[b]);
            // P(j) is handed over before S(j+1) is waited for and read back, so the
            // hand-over (and S(j+3), issued behind P·V(j)) never waits on S(j+1)
            // (1 % faster than loading S(j+1) first)
            if (j + 1 < n_kv) {
                const int nb = (j + 1) % kBufs;
                mbar_wait(&sf[nb], ((j + 1) / kBufs) & 1);
                tc_fence_after();
                tmem_ld32(buf0 + nb * 64, ra);
                tmem_ld32(buf0 + nb * 64 + 32, rb);
                tmem_ld_wait();
#pragma unroll
                for (int u = 0; u < 32; ++u) asm volatile("" : "+r"(ra[u]), "+r"(rb[u]));  // reads after wait::ld
            }
        }
        mbar_wait(&pd[(n_kv - 1) % kBufs], ((n_kv - 1) / kBufs) & 1);
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
    // kernel table: [mode 0 with kPolyPairs 2 | 4 | 6 of 16, timing probe]
    using KernT = decltype(&attn_kernel<0, 4>);
    static KernT table[4] = {attn_kernel<0, 2>, attn_kernel<0, 4>, attn_kernel<0, 6>, attn_kernel<1, 0>};
    static std::atomic<uint64_t> attr{0};
    static int pick = 1;
    if (first_on_device(attr)) {
        for (KernT k : table) PKV_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
        if (const char* e = getenv("PKV_ATTN_POLY")) pick = atoi(e) <= 2 ? 0 : (atoi(e) <= 4 ? 1 : 2);
        if (const char* e = getenv("PKV_ATTN_MODE")) pick = atoi(e) == 1 ? 3 : pick;  // timing probe, no exponentials
    }
    const CUtensorMap tq = make_tmap_3d(qkv, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, (uint64_t)(3 * D), (uint64_t)Lw,
                                        (uint64_t)nwin, (uint64_t)(3 * D) * 2, (uint64_t)(3 * D) * 2 * Lw, kD, kBQ, 1,
                                        CU_TENSOR_MAP_SWIZZLE_128B);
    const CUtensorMap tkv = make_tmap_3d(qkv, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, (uint64_t)(3 * D), (uint64_t)Lw,
                                         (uint64_t)nwin, (uint64_t)(3 * D) * 2, (uint64_t)(3 * D) * 2 * Lw, kD, kBK, 1,
                                         CU_TENSOR_MAP_SWIZZLE_128B);
    const dim3 grid((unsigned)((Lw + kBQ * kTiles - 1) / (kBQ * kTiles)), (unsigned)heads, (unsigned)nwin);
    const float scale_log2 = 1.4426950408889634f / sqrtf((float)kD);
    table[pick]<<<grid, kThreads, kSmem, st>>>(tq, tkv, out_h, out_l, ld_out, (int)Lw, (int)D, scale_log2);
    check_launch("attn_kernel");
}

}  // namespace pkv
