// prefill.cu — the proxy model's prefill self-attention emitting the row LSE
// that scoring pass 2 consumes (X is a
// by-product of the proxy's prefill). With it the proxy pays for one Q·Kᵀ
// pass it runs anyway, and scoring is a single tensor-core pass (pool pass
// with the supplied LSE, pkv_score(lse_dev = ...)).
//
//   O[l,h,q,:] = softmax(Q[l,h,q]·K[l,h/g,:]ᵀ/√d) · V[l,h/g,:]   (bf16 out)
//   lse[l,h,q] = log Σ_j exp(Q·K_j/√d)                            (fp32, natural log)
// bf16 Q/K/V, fp32 accumulation, optional causal mask (key j visible to query
// q iff j <= q + Nk - Nq), GQA group g = Hq / Hkv, head_dim 64 or 128.
//
// CTA = one 128-query tile of one head (two CTAs per SM at d = 64).
//   warp 0 TMA producer + TMEM allocator; warp 1 MMA issuer; warps 2-5 softmax
//   (one thread per query row).
// TMEM: three 64-key S/P buffers + O (d columns). Per 64-key tile j, buffer
// j % 3: S = Q·K_jᵀ issued three tiles ahead; the softmax warps read S once,
// evaluate P = 2^(c·s − m) against a lazily raised integer running max (redo
// only if the tile max exceeds it by 2^15), pack P to bf16 over the buffer's
// first 32 columns; O += P·V_j takes P straight from TMEM (TS-MMA). This is
// the encoder attention of attn.cu retargeted to bf16, GQA, causal masks and
// an LSE output.
#include <cuda_bf16.h>

#include <cstdlib>

#include "prefill.cuh"
#include "sm100.cuh"

namespace pkv {
namespace {

using namespace sm100;

template <int D>
struct PF {
    static constexpr int kBQ = 128, kBK = 64;
    static constexpr int kBufs = 3;
    static constexpr int kPanels = D / 64;
    static constexpr int kStages = D == 64 ? 5 : 4;
    static constexpr int kQBytes = kBQ * D * 2;
    static constexpr int kKVBytes = kBK * D * 2;  // one K or V tile
    static constexpr int kThreads = 64 + 128;
    static constexpr int kSmem = 1024 + kQBytes + 2 * kKVBytes * kStages + 512;
    static constexpr uint32_t kColO = kBufs * 64;
    static constexpr uint32_t kTmemCols = kColO + D <= 256 ? 256 : 512;
    static constexpr int kCtasPerSm = kTmemCols == 256 ? 2 : 1;
};

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kHeadroom = 15.0f;
constexpr int kPolyPairs = 4;  // of every 16 exponential pairs

__device__ __forceinline__ uint32_t pack_bf162(float a, float b) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&h);
}

// 32 scores of one row -> 16 bf16 pairs of P = 2^(c·s − m) at p_col; returns
// the chunk's raw max and adds Σp to acc. Columns with kbase + i >= valid are
// masked (key tail / causal diagonal).
template <bool kMask>
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
        pk[i] = pack_bf162(ef.x, ef.y);
    }
    tmem_st16(p_col, pk);
    return fmaxf(fmaxf(mt[0], mt[1]), fmaxf(mt[2], mt[3]));
}

template <int D>
__global__ void __launch_bounds__(PF<D>::kThreads, PF<D>::kCtasPerSm)
    prefill_attn_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                        const __grid_constant__ CUtensorMap tv, int Hq, int Hkv, int Nq, int Nk, int causal,
                        float c_log2, __nv_bfloat16* __restrict__ o_out, float* __restrict__ lse_out) {
    using C = PF<D>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = smem;                          // [panels][128 x 128 B]
    uint8_t* sK = sQ + C::kQBytes;               // [stages][panels][64 x 128 B]
    uint8_t* sV = sK + C::kStages * C::kKVBytes;  // [stages][panels][64 x 128 B]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sV + C::kStages * C::kKVBytes);
    uint64_t* bar_q = bars;
    uint64_t* kv_full = bars + 1;
    uint64_t* kv_empty = kv_full + C::kStages;
    uint64_t* s_full = kv_empty + C::kStages;   // [bufs]
    uint64_t* p_full = s_full + C::kBufs;       // [bufs]
    uint64_t* pv_done = p_full + C::kBufs;      // [bufs]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_done + C::kBufs);

    const uint32_t warp = warp_id(), lane = lane_id();
    const int q0 = blockIdx.x * C::kBQ, h = blockIdx.y, l = blockIdx.z;
    const int g = Hq / Hkv;
    const int qslab = l * Hq + h, kslab = l * Hkv + h / g;
    const int off = Nk - Nq;
    int n_kv = (Nk + C::kBK - 1) / C::kBK;
    if (causal) {
        const int last = q0 + C::kBQ - 1 + off;  // last key any query of the tile sees
        const int t = last < 0 ? 0 : last / C::kBK + 1;
        n_kv = t < n_kv ? t : n_kv;
    }

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tq);
        tma_prefetch(&tk);
        tma_prefetch(&tv);
        mbar_init(bar_q, 1);
        for (int s = 0; s < C::kStages; ++s) {
            mbar_init(&kv_full[s], 1);
            mbar_init(&kv_empty[s], 1);
        }
        for (int i = 0; i < C::kBufs; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&p_full[i], 4);
            mbar_init(&pv_done[i], 1);
        }
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc(tmem_slot, C::kTmemCols);
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
                mbar_wait(&kv_empty[st], ((j / C::kStages) & 1) ^ 1);
                mbar_arrive_expect_tx(&kv_full[st], 2 * C::kKVBytes);
                for (int p = 0; p < C::kPanels; ++p) {
                    tma_load_3d(sK + st * C::kKVBytes + p * (C::kBK * 128), &tk, &kv_full[st], p * 64, j * C::kBK,
                                kslab);
                    tma_load_3d(sV + st * C::kKVBytes + p * (C::kBK * 128), &tv, &kv_full[st], p * 64, j * C::kBK,
                                kslab);
                }
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t idesc_s = idesc_f16(C::kBQ, C::kBK, 1);
        constexpr uint32_t idesc_o = idesc_f16(C::kBQ, D, 1, 0, 1);  // B (V) is MN-major
        if (n_kv > 0) mbar_wait(bar_q, 0);
        auto issue_s = [&](int j) {  // S -> buffer j % 3
            const int st = j % C::kStages, b = j % C::kBufs;
            mbar_wait(&kv_full[st], (j / C::kStages) & 1);
            tc_fence_after();
            if (elect_one()) {
#pragma unroll
                for (int p = 0; p < C::kPanels; ++p) {
                    const uint64_t a = desc_sw128(sQ + p * (C::kBQ * 128));
                    const uint64_t bk = desc_sw128(sK + st * C::kKVBytes + p * (C::kBK * 128));
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        mma_f16_ss(tmem + b * 64, a + kk * 2, bk + kk * 2, idesc_s, (p | kk) != 0);
                }
                mma_commit(&s_full[b]);
            }
            __syncwarp();
        };
        for (int j = 0; j < C::kBufs && j < n_kv; ++j) issue_s(j);
        for (int j = 0; j < n_kv; ++j) {
            const int b = j % C::kBufs;
            mbar_wait(&p_full[b], (j / C::kBufs) & 1);
            tc_fence_after();
            if (elect_one()) {
                const uint8_t* v = sV + (j % C::kStages) * C::kKVBytes;
                // O += P·V_j: A = P (buffer columns [0, 32)) from TMEM, 16 keys per MMA;
                // V panels (64 d each) are the MN-major N groups, 8 KB apart
#pragma unroll
                for (int kk = 0; kk < C::kBK / 16; ++kk) {
                    const uint64_t bv = desc_sw128_mn(v + kk * 16 * 128, C::kBK * 128);
                    mma_f16_ts(tmem + C::kColO, tmem + b * 64 + kk * 8, bv, idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
                }
                mma_commit(&pv_done[b]);
                mma_commit(&kv_empty[j % C::kStages]);
            }
            __syncwarp();
            // S_{j+3} reuses this buffer right behind P·V_j (in-order tcgen05.mma)
            if (j + C::kBufs < n_kv) issue_s(j + C::kBufs);
        }
    } else {
        const uint32_t quad = warp & 3;
        const uint32_t row = quad * 32 + lane;
        const int q = q0 + (int)row;
        const uint32_t lane_addr = (quad * 32) << 16;
        const uint32_t o_addr = tmem + lane_addr + C::kColO;
        const int kend = causal ? min(Nk, q + off + 1) : Nk;  // keys [0, kend) visible to this row
        const uint64_t cc = pack2(c_log2, c_log2);
        float m = -INFINITY, lsum = 0.0f;  // m: integer, log2 domain
        uint32_t ra[32], rb[32];
        if (n_kv > 0) {
            mbar_wait(&s_full[0], 0);
            tc_fence_after();
            tmem_ld32(tmem + lane_addr, ra);
            tmem_ld32(tmem + lane_addr + 32, rb);
            tmem_ld_wait();
        }
        for (int j = 0; j < n_kv; ++j) {
            const int b = j % C::kBufs;
            const uint32_t s_addr = tmem + lane_addr + b * 64;
            const int valid = kend - j * C::kBK;
            const bool masked = __any_sync(0xffffffffu, valid < C::kBK);  // warp-uniform
            uint64_t acc0, acc1;
            for (int attempt = 0;; ++attempt) {
                const uint64_t nm = pack2(-m, -m), mp = pack2(12582912.0f - m, 12582912.0f - m);
                acc0 = pack2(0.0f, 0.0f);
                acc1 = acc0;
                float hmax;
                if (masked) {
                    hmax = fmaxf(p_chunk<true>(ra, 0, s_addr, valid, cc, nm, mp, acc0, acc1),
                                 p_chunk<true>(rb, 32, s_addr + 16, valid, cc, nm, mp, acc0, acc1));
                } else {
                    hmax = fmaxf(p_chunk<false>(ra, 0, s_addr, 64, cc, nm, mp, acc0, acc1),
                                 p_chunk<false>(rb, 32, s_addr + 16, 64, cc, nm, mp, acc0, acc1));
                }
                const float rmax = hmax * c_log2;
                if (!__any_sync(0xffffffffu, rmax > m + kHeadroom) || attempt > 0) break;
                const float mn = fmaxf(m, ceilf(rmax));
                const float alpha = ex2(m - mn);  // 0 when m = -inf
                lsum *= alpha;
                m = mn;
                if (j > 0) {
                    mbar_wait(&pv_done[(j - 1) % C::kBufs], ((j - 1) / C::kBufs) & 1);  // O stable
                    tc_fence_after();
#pragma unroll
                    for (int c = 0; c < D; c += 32) {
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
            lsum += rs.x + rs.y;
            if (j + 1 < n_kv) {  // next tile's S into registers (its MMA ran ahead)
                const int nb = (j + 1) % C::kBufs;
                mbar_wait(&s_full[nb], ((j + 1) / C::kBufs) & 1);
                tc_fence_after();
                tmem_ld32(tmem + lane_addr + nb * 64, ra);
                tmem_ld32(tmem + lane_addr + nb * 64 + 32, rb);
            }
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&p_full[b]);
            if (j + 1 < n_kv) {
                tmem_ld_wait();
#pragma unroll
                for (int u = 0; u < 32; ++u) asm volatile("" : "+r"(ra[u]), "+r"(rb[u]));  // reads after wait::ld
            }
        }
        if (n_kv > 0) {
            mbar_wait(&pv_done[(n_kv - 1) % C::kBufs], ((n_kv - 1) / C::kBufs) & 1);
            tc_fence_after();
        }
        const int64_t orow = (int64_t)qslab * Nq + q;
        const float inv = lsum > 0.0f ? 1.0f / lsum : 0.0f;
        if (lse_out && q < Nq) lse_out[orow] = lsum > 0.0f ? (m + __log2f(lsum)) / kLog2e : -INFINITY;
#pragma unroll
        for (int c0 = 0; c0 < D; c0 += 32) {
            uint32_t o[32];
            if (n_kv > 0) {
                tmem_ld32(o_addr + c0, o);
                tmem_ld_wait();
            } else {
#pragma unroll
                for (int u = 0; u < 32; ++u) o[u] = 0u;
            }
            if (o_out && q < Nq) {
#pragma unroll
                for (int c = 0; c < 32; c += 8) {
                    uint4 w;
                    w.x = pack_bf162(__uint_as_float(o[c]) * inv, __uint_as_float(o[c + 1]) * inv);
                    w.y = pack_bf162(__uint_as_float(o[c + 2]) * inv, __uint_as_float(o[c + 3]) * inv);
                    w.z = pack_bf162(__uint_as_float(o[c + 4]) * inv, __uint_as_float(o[c + 5]) * inv);
                    w.w = pack_bf162(__uint_as_float(o[c + 6]) * inv, __uint_as_float(o[c + 7]) * inv);
                    *reinterpret_cast<uint4*>(o_out + orow * D + c0 + c) = w;
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, C::kTmemCols);
    }
}

template <int D>
void run_prefill(const ScoreShape& s, const void* q, const void* k, const void* v, void* o, float* lse,
                 cudaStream_t st) {
    using C = PF<D>;
    static std::atomic<uint64_t> once{0};
    if (first_on_device(once))
        PKV_CUDA(cudaFuncSetAttribute(prefill_attn_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
    const CUtensorMap tq = make_tmap_3d(q, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, D, s.Nq, s.L * s.Hq, D * 2, D * 2 * s.Nq,
                                        64, C::kBQ, 1, CU_TENSOR_MAP_SWIZZLE_128B);
    const CUtensorMap tk = make_tmap_3d(k, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, D, s.Nk, s.L * s.Hkv, D * 2, D * 2 * s.Nk,
                                        64, C::kBK, 1, CU_TENSOR_MAP_SWIZZLE_128B);
    const CUtensorMap tv = make_tmap_3d(v, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, D, s.Nk, s.L * s.Hkv, D * 2, D * 2 * s.Nk,
                                        64, C::kBK, 1, CU_TENSOR_MAP_SWIZZLE_128B);
    const dim3 grid((unsigned)((s.Nq + C::kBQ - 1) / C::kBQ), (unsigned)s.Hq, (unsigned)s.L);
    prefill_attn_kernel<D><<<grid, C::kThreads, C::kSmem, st>>>(tq, tk, tv, (int)s.Hq, (int)s.Hkv, (int)s.Nq,
                                                                (int)s.Nk, s.causal ? 1 : 0, kLog2e / sqrtf((float)D),
                                                                static_cast<__nv_bfloat16*>(o), lse);
    check_launch("prefill_attn_kernel");
}

}  // namespace

void launch_prefill_attention(const ScoreShape& s, const void* q, const void* k, const void* v, void* o, float* lse,
                              cudaStream_t st) {
    if (s.d == 64) run_prefill<64>(s, q, k, v, o, lse, st);
    else run_prefill<128>(s, q, k, v, o, lse, st);
}

}  // namespace pkv

using namespace pkv;

extern "C" pkv_status pkv_proxy_prefill_attention(pkv_ctx ctx, const void* q_dev, const void* k_dev, const void* v_dev,
                                                  int64_t L, int64_t Hq, int64_t Hkv, int64_t Nq, int64_t Nk,
                                                  int64_t d, uint32_t flags, void* o_out_dev, float* lse_out_dev,
                                                  void* stream) {
    return guard([&] {
        require_ctx(ctx);
        ScoreShape s{L, Hq, Hkv, Nq, Nk, d, (flags & PKV_SCORE_CAUSAL) != 0};
        score_validate(s);
        PKV_REQUIRE_VALUE(o_out_dev != nullptr || lse_out_dev != nullptr, "prefill attention: no output requested");
        launch_prefill_attention(s, q_dev, k_dev, v_dev, o_out_dev, lse_out_dev, static_cast<cudaStream_t>(stream));
        count_launch(ctx);
    });
}
