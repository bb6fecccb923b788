// decode.cu — target-side consumption of the packed cache (SURVEY.md §8(f)
// item 2; the target decodes over the pruned KV): one decode
// query per query head attends over its KV head's K retained rows,
//   o[l, h, :] = softmax(q[l, h]·K_packed[l, h/g]ᵀ · scale) · V_packed[l, h/g]
// bf16 q/K/V, fp32 math and output, GQA group g = Hq / Hkv <= 8, head_dim 128
// (or 64).
//
// HBM-bound (every retained K/V byte is read once; the packed cache is ρ of
// the full one, so decode time scales with ρ). Split-K flash decoding:
//   pass 1: CTA = (key split, KV head, layer), 8 warps; a warp handles four
//     keys per step with 8 lanes per key row (16 dims per lane at d = 128:
//     32-byte coalesced loads, 1 KB per warp instruction; 16 lanes and two
//     keys when g = 8, for registers), all g query heads of the
//     group against each row (K/V read once for the group); each 8-lane group
//     keeps its own online (max, sum, o) state, so no per-key cross-group
//     traffic — three shuffle steps finish each dot. States are merged in
//     shared memory and one partial per (split, head) goes to global.
//   pass 2: merge the splits (log-sum-exp weighted) into o.
#include <cuda_bf16.h>

#include <cstdlib>

#include "decode.cuh"
#include "sm100.cuh"

namespace pkv {
namespace {

constexpr int kWarps = 8;
constexpr int kMaxG = 8;
constexpr float kLazy = 8.0f;  // log2 headroom before a group's running max is raised

__device__ __forceinline__ void bf16x8_to_f32(const uint4& u, float (&f)[8]) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        f[2 * i] = __uint_as_float(w[i] << 16);
        f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
}

using sm100::ex2;
using sm100::ffma2;
using sm100::pack2;
using sm100::unpack2;

// Paged cache (vLLM-style): row r of (layer, KV head) slab s lives in page
// table[s·max_blocks + r / page] at row r % page of the [pages, page, D] pools;
// slab s holds lens[s] rows (per-head variable length).
struct Paged {
    const int32_t* table = nullptr;
    const int32_t* lens = nullptr;
    int64_t max_blocks = 0, page = 0;
};

// partial: [L, Hq, splits] x {m (log2 domain), l, o[D]}. G: group-size
// bucket (1, 2, 4, 8); g <= G heads are live (g = 7 for Qwen-2.5-7B).
template <int D, int G, bool kPaged>
__global__ void __launch_bounds__(32 * kWarps, 2)
    decode_split_kernel(const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ kc,
                        const __nv_bfloat16* __restrict__ vc, int Hq, int Hkv, int g, int64_t K, int64_t chunk,
                        float scale_log2, float* __restrict__ part, Paged pg) {
    // lanes per key row: 8 (16 dims each at d = 128), 16 for G = 8 at d = 128 (register budget)
    constexpr int kLPK = (G >= 4 && D == 128) ? 16 : 8;
    constexpr int kKPW = 32 / kLPK;  // keys per warp step
    constexpr int kDL = D / kLPK;    // dims per lane
    const int split = blockIdx.x, kh = blockIdx.y, l = blockIdx.z;
    const int splits = gridDim.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int grp = lane / kLPK, sub = lane % kLPK;  // key group, lane within the group
    const int64_t kslab = (int64_t)l * Hkv + kh;
    const int64_t len = kPaged ? (int64_t)__ldg(pg.lens + kslab) : K;
    const int64_t k_lo = split * chunk, k_hi = min(len, k_lo + chunk);
    const __nv_bfloat16* kbase = kPaged ? kc + sub * kDL : kc + kslab * K * D + sub * kDL;
    const __nv_bfloat16* vbase = kPaged ? vc + sub * kDL : vc + kslab * K * D + sub * kDL;
    const int32_t* ptab = kPaged ? pg.table + kslab * pg.max_blocks : nullptr;

    // this lane's slice of the group's queries (pre-scaled to the log2 domain)
    float qr[G][kDL];
#pragma unroll
    for (int h = 0; h < G; ++h) {
        const __nv_bfloat16* qp = q + ((int64_t)l * Hq + kh * g + (h < g ? h : 0)) * D + sub * kDL;
#pragma unroll
        for (int c = 0; c < kDL; c += 8) {
            float f[8];
            bf16x8_to_f32(*reinterpret_cast<const uint4*>(qp + c), f);
#pragma unroll
            for (int e = 0; e < 8; ++e) qr[h][c + e] = f[e] * scale_log2;
        }
    }
    float m[G], ls[G], o[G][kDL];
#pragma unroll
    for (int h = 0; h < G; ++h) {
        m[h] = -INFINITY;
        ls[h] = 0.0f;
#pragma unroll
        for (int e = 0; e < kDL; ++e) o[h][e] = 0.0f;
    }
    // keys of this CTA: warp w, group r take key k_lo + kKPW*(w + kWarps*i) + r.
    // The loop runs warp-uniformly (the dot reductions shuffle across the
    // warp); a group past the chunk end computes on a clamped row and skips
    // its state update.
    // raw 16-byte row slices of the current and the next key (register double
    // buffer: the next step's loads are in flight during this step's math)
    constexpr int kV = kDL / 8;
    uint4 kraw[kV], vraw[kV], knx[kV], vnx[kV];
    auto load_row = [&](int64_t key0, uint4 (&kr)[kV], uint4 (&vr)[kV]) {
        const int64_t key = key0 + grp;
        int64_t kk = key < k_hi ? key : k_lo;
        if (kPaged) kk = (int64_t)__ldg(ptab + kk / pg.page) * pg.page + kk % pg.page;  // pool row
#pragma unroll
        for (int c = 0; c < kV; ++c) {
            kr[c] = __ldcs(reinterpret_cast<const uint4*>(kbase + kk * D + 8 * c));
            vr[c] = __ldcs(reinterpret_cast<const uint4*>(vbase + kk * D + 8 * c));
        }
    };
    const int64_t kstep = kKPW * kWarps;
    if (k_lo + kKPW * warp < k_hi) load_row(k_lo + kKPW * warp, kraw, vraw);
    for (int64_t key0 = k_lo + kKPW * warp; key0 < k_hi; key0 += kstep) {
        const int64_t key = key0 + grp;
        const bool ok = key < k_hi;
        if (key0 + kstep < k_hi) load_row(key0 + kstep, knx, vnx);
        float kf[kDL], vf[kDL];
#pragma unroll
        for (int c = 0; c < kV; ++c) {
            float f[8];
            bf16x8_to_f32(kraw[c], f);
#pragma unroll
            for (int e = 0; e < 8; ++e) kf[8 * c + e] = f[e];
            bf16x8_to_f32(vraw[c], f);
#pragma unroll
            for (int e = 0; e < 8; ++e) vf[8 * c + e] = f[e];
        }
        // all G dots first, then the G butterfly reductions interleaved step by
        // step (independent shuffle chains), then the online-softmax updates
        float sc[G];
#pragma unroll
        for (int h = 0; h < G; ++h) {
            uint64_t s2 = pack2(0.0f, 0.0f);
#pragma unroll
            for (int e = 0; e < kDL; e += 2) s2 = ffma2(pack2(qr[h][e], qr[h][e + 1]), pack2(kf[e], kf[e + 1]), s2);
            const float2 sp = unpack2(s2);
            sc[h] = sp.x + sp.y;
        }
#pragma unroll
        for (int o2 = 1; o2 < kLPK; o2 <<= 1)
#pragma unroll
            for (int h = 0; h < G; ++h) sc[h] += __shfl_xor_sync(0xffffffffu, sc[h], o2);
        if (ok) {
#pragma unroll
            for (int h = 0; h < G; ++h) {
                if (h >= g) break;  // warp-uniform
                const float s = sc[h];
                // lazy rescale: the reference max moves only when a score
                // exceeds it by more than 2^kLazy (p <= 2^8 is exact in fp32)
                if (s > m[h] + kLazy) {
                    const float a = ex2(m[h] - s);  // 0 on the first key (m = -inf)
                    ls[h] *= a;
                    const uint64_t aa = pack2(a, a);
#pragma unroll
                    for (int e = 0; e < kDL; e += 2) {
                        const float2 r = unpack2(sm100::fmul2(pack2(o[h][e], o[h][e + 1]), aa));
                        o[h][e] = r.x;
                        o[h][e + 1] = r.y;
                    }
                    m[h] = s;
                }
                const float p = ex2(s - m[h]);
                ls[h] += p;
                const uint64_t pp = pack2(p, p);
#pragma unroll
                for (int e = 0; e < kDL; e += 2) {
                    const float2 r = unpack2(ffma2(pp, pack2(vf[e], vf[e + 1]), pack2(o[h][e], o[h][e + 1])));
                    o[h][e] = r.x;
                    o[h][e + 1] = r.y;
                }
            }
        }
#pragma unroll
        for (int c = 0; c < kV; ++c) {
            kraw[c] = knx[c];
            vraw[c] = vnx[c];
        }
    }
    // merge the 32 group states per head through shared memory
    constexpr int kGroupsCta = kWarps * kKPW;
    __shared__ float s_m[kGroupsCta][G], s_l[kGroupsCta][G];
    __shared__ float s_o[G][D];
    const int gid = warp * kKPW + grp;
    if (sub == 0) {
#pragma unroll
        for (int h = 0; h < G; ++h) {
            s_m[gid][h] = m[h];
            s_l[gid][h] = ls[h];
        }
    }
    for (int i = threadIdx.x; i < G * D; i += blockDim.x) s_o[i / D][i % D] = 0.0f;
    __syncthreads();
    float M[G];
#pragma unroll
    for (int h = 0; h < G; ++h) {
        M[h] = -INFINITY;
        for (int r = 0; r < kGroupsCta; ++r) M[h] = fmaxf(M[h], s_m[r][h]);
    }
#pragma unroll
    for (int h = 0; h < G; ++h) {
        const float w = M[h] == -INFINITY ? 0.0f : exp2f(m[h] - M[h]);
#pragma unroll
        for (int e = 0; e < kDL; ++e) atomicAdd(&s_o[h][sub * kDL + e], o[h][e] * w);
    }
    __syncthreads();
    const int64_t pstride = 2 + D;
    for (int i = threadIdx.x; i < g * D; i += blockDim.x) {
        const int h = i / D, e = i % D;
        float* pp = part + (((int64_t)l * Hq + kh * g + h) * splits + split) * pstride;
        pp[2 + e] = s_o[h][e];
        if (e == 0) {
            float L = 0.0f;
            for (int r = 0; r < kGroupsCta; ++r)
                L += s_m[r][h] == -INFINITY ? 0.0f : s_l[r][h] * exp2f(s_m[r][h] - M[h]);
            pp[0] = M[h];
            pp[1] = L;
        }
    }
}

// Tensor-core variant: per warp, 16-key tiles staged by cp.async into a
// private 3-stage shared-memory ring (16-byte chunks XOR-swizzled by row, so
// ldmatrix is conflict-free); S = Q·Kᵀ and O += P·V as mma.sync m16n8k16 with
// the G <= 8 heads of the group as the M rows (rows G..15 are zero padding:
// with M >= 64, tcgen05 would waste 8x more). Scores are scaled in fp32; P is
// split into bf16 hi + lo (two MMAs) so the product keeps fp32-level accuracy
// against the exact bf16 V. Lazy max per head (raised only by > 2^8).
constexpr int kMmaWarps = 4;
constexpr int kMmaStages = 3;
constexpr int kTileKeys = 16;

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t (&r)[4]) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t (&r)[4]) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}
__device__ __forceinline__ void mma_bf16(float (&d)[4], uint32_t a0, uint32_t a2, uint32_t b0, uint32_t b1) {
    // A rows 8..15 (a1, a3) are zero padding
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
        "{%0, %1, %2, %3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}

template <int D>
struct MmaCfg {
    static constexpr int kRowBytes = D * 2;
    static constexpr int kChunks = D / 8;  // 16-byte chunks per row
    static constexpr int kTileBytes = kTileKeys * kRowBytes;
    static constexpr int kStageBytes = 2 * kTileBytes;  // K | V
    static constexpr int kSmem = kMmaWarps * kMmaStages * kStageBytes;
};

template <int D, int G>
__global__ void __launch_bounds__(32 * kMmaWarps)
    decode_mma_kernel(const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ kc,
                      const __nv_bfloat16* __restrict__ vc, int Hq, int Hkv, int g, int64_t K, int64_t chunk,
                      float scale_log2, float* __restrict__ part, Paged pg, bool paged) {
    using C = MmaCfg<D>;
    static_assert(G <= 8, "heads are the MMA rows 0..7");
    extern __shared__ __align__(128) uint8_t dsm[];
    const int split = blockIdx.x, kh = blockIdx.y, l = blockIdx.z;
    const int splits = gridDim.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t kslab = (int64_t)l * Hkv + kh;
    const int64_t len = paged ? (int64_t)__ldg(pg.lens + kslab) : K;
    const int64_t k_lo = split * chunk, k_hi = min(len, k_lo + chunk);
    const int64_t n_tiles = k_hi > k_lo ? (k_hi - k_lo + kTileKeys - 1) / kTileKeys : 0;
    const int32_t* ptab = paged ? pg.table + kslab * pg.max_blocks : nullptr;
    uint8_t* ring = dsm + warp * kMmaStages * C::kStageBytes;
    const uint32_t ring_s = static_cast<uint32_t>(__cvta_generic_to_shared(ring));

    // this warp's tiles: t = warp, warp + kMmaWarps, ...
    auto issue = [&](int64_t t, int stage) {
        const int64_t key0 = k_lo + t * kTileKeys;
        const uint32_t dk = ring_s + stage * C::kStageBytes, dv = dk + C::kTileBytes;
#pragma unroll
        for (int j = 0; j < kTileKeys * C::kChunks / 32; ++j) {
            const int i = lane + 32 * j;
            const int row = i / C::kChunks, c = i % C::kChunks;
            int64_t key = key0 + row;
            key = key < k_hi ? key : k_lo;
            const int64_t grow = paged ? (int64_t)__ldg(ptab + key / pg.page) * pg.page + key % pg.page
                                       : kslab * K + key;
            const uint32_t off = row * C::kRowBytes + ((c ^ (row & 7)) << 4);
            cp_async16(dk + off, kc + grow * D + c * 8);
            cp_async16(dv + off, vc + grow * D + c * 8);
        }
    };

    // Q as the A operand (head rows; rows >= g are zero): 16 dims per k-step
    const int hrow = lane >> 2, qd = (lane & 3) * 2;
    uint32_t qa[D / 16][2];
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
        if (hrow < g) {
            const __nv_bfloat16* qp = q + ((int64_t)l * Hq + kh * g + hrow) * D + kk * 16 + qd;
            qa[kk][0] = *reinterpret_cast<const uint32_t*>(qp);
            qa[kk][1] = *reinterpret_cast<const uint32_t*>(qp + 8);
        } else {
            qa[kk][0] = qa[kk][1] = 0u;
        }
    }
    float o[D / 8][4];
#pragma unroll
    for (int nd = 0; nd < D / 8; ++nd) o[nd][0] = o[nd][1] = o[nd][2] = o[nd][3] = 0.0f;
    float m = -INFINITY, lsum = 0.0f;

    const int64_t my_tiles = n_tiles > warp ? (n_tiles - warp + kMmaWarps - 1) / kMmaWarps : 0;
#pragma unroll
    for (int i = 0; i < kMmaStages - 1; ++i) {
        if (i < my_tiles) issue(warp + (int64_t)i * kMmaWarps, i);
        cp_async_commit();
    }
    for (int64_t i = 0; i < my_tiles; ++i) {
        const int stage = (int)(i % kMmaStages);
        if (i + kMmaStages - 1 < my_tiles) issue(warp + (i + kMmaStages - 1) * kMmaWarps, (int)((i + kMmaStages - 1) % kMmaStages));
        cp_async_commit();
        cp_async_wait<kMmaStages - 1>();
        __syncwarp();
        const uint32_t tk = ring_s + stage * C::kStageBytes, tv = tk + C::kTileBytes;
        const int64_t key0 = k_lo + (warp + i * kMmaWarps) * kTileKeys;
        // S = Q·Kᵀ for two 8-key blocks
        float sacc[2][4];
#pragma unroll
        for (int nb = 0; nb < 2; ++nb) {
            sacc[nb][0] = sacc[nb][1] = sacc[nb][2] = sacc[nb][3] = 0.0f;
#pragma unroll
            for (int kk = 0; kk < D / 16; kk += 2) {
                const int mtx = lane >> 3, r = lane & 7;
                const int key = nb * 8 + r, c = (kk + (mtx >> 1)) * 2 + (mtx & 1);
                uint32_t b[4];
                ldsm_x4(tk + key * C::kRowBytes + ((c ^ (key & 7)) << 4), b);
                mma_bf16(sacc[nb], qa[kk][0], qa[kk][1], b[0], b[1]);
                mma_bf16(sacc[nb], qa[kk + 1][0], qa[kk + 1][1], b[2], b[3]);
            }
        }
        // softmax over this tile's keys for head row hrow (a quad of lanes holds all 16 keys)
        float x[2][2];
        float tmax = -INFINITY;
#pragma unroll
        for (int nb = 0; nb < 2; ++nb)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int64_t key = key0 + nb * 8 + qd + j;
                x[nb][j] = key < k_hi ? sacc[nb][j] * scale_log2 : -INFINITY;
                tmax = fmaxf(tmax, x[nb][j]);
            }
        tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 1));
        tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 2));
        if (tmax > m + kLazy) {  // raise the reference max (first tile always)
            const float a = ex2(m - tmax);
            lsum *= a;
#pragma unroll
            for (int nd = 0; nd < D / 8; ++nd) {
                o[nd][0] *= a;
                o[nd][1] *= a;
            }
            m = tmax;
        }
        float p[2][2];
#pragma unroll
        for (int nb = 0; nb < 2; ++nb)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                p[nb][j] = ex2(x[nb][j] - m);
                lsum += p[nb][j];
            }
        // P as the A operand, split into bf16 hi + lo
        const uint32_t ah0 = pack_bf16(p[0][0], p[0][1]), ah2 = pack_bf16(p[1][0], p[1][1]);
        const __nv_bfloat162 h0 = *reinterpret_cast<const __nv_bfloat162*>(&ah0);
        const __nv_bfloat162 h2 = *reinterpret_cast<const __nv_bfloat162*>(&ah2);
        const uint32_t al0 = pack_bf16(p[0][0] - __low2float(h0), p[0][1] - __high2float(h0));
        const uint32_t al2 = pack_bf16(p[1][0] - __low2float(h2), p[1][1] - __high2float(h2));
        // O += P·V, two 8-dim blocks per ldmatrix.x4.trans
#pragma unroll
        for (int nd = 0; nd < D / 8; nd += 2) {
            const int mtx = lane >> 3, r = lane & 7;
            const int key = (mtx & 1) * 8 + r, c = nd + (mtx >> 1);
            uint32_t b[4];
            ldsm_x4_t(tv + key * C::kRowBytes + ((c ^ (key & 7)) << 4), b);
            mma_bf16(o[nd], ah0, ah2, b[0], b[1]);
            mma_bf16(o[nd], al0, al2, b[0], b[1]);
            mma_bf16(o[nd + 1], ah0, ah2, b[2], b[3]);
            mma_bf16(o[nd + 1], al0, al2, b[2], b[3]);
        }
        __syncwarp();  // the stage is refilled by the next issue
    }
    cp_async_wait<0>();
    lsum += __shfl_xor_sync(0xffffffffu, lsum, 1);
    lsum += __shfl_xor_sync(0xffffffffu, lsum, 2);

    // merge the kMmaWarps warp states per head
    __shared__ float s_m[kMmaWarps][8], s_l[kMmaWarps][8];
    __shared__ float s_o[8][D];
    if ((lane & 3) == 0) {
        s_m[warp][hrow] = m;
        s_l[warp][hrow] = lsum;
    }
    for (int i = threadIdx.x; i < 8 * D; i += blockDim.x) s_o[i / D][i % D] = 0.0f;
    __syncthreads();
    float M = -INFINITY;
    for (int w = 0; w < kMmaWarps; ++w) M = fmaxf(M, s_m[w][hrow]);
    const float wgt = M == -INFINITY ? 0.0f : exp2f(m - M);
    if (hrow < g) {
#pragma unroll
        for (int nd = 0; nd < D / 8; ++nd) {
            atomicAdd(&s_o[hrow][nd * 8 + qd], o[nd][0] * wgt);
            atomicAdd(&s_o[hrow][nd * 8 + qd + 1], o[nd][1] * wgt);
        }
    }
    __syncthreads();
    const int64_t pstride = 2 + D;
    for (int i = threadIdx.x; i < g * D; i += blockDim.x) {
        const int h = i / D, e = i % D;
        float* pp = part + (((int64_t)l * Hq + kh * g + h) * splits + split) * pstride;
        pp[2 + e] = s_o[h][e];
        if (e == 0) {
            float Mh = -INFINITY;
            for (int w = 0; w < kMmaWarps; ++w) Mh = fmaxf(Mh, s_m[w][h]);
            float Ls = 0.0f;
            for (int w = 0; w < kMmaWarps; ++w)
                Ls += s_m[w][h] == -INFINITY ? 0.0f : s_l[w][h] * exp2f(s_m[w][h] - Mh);
            pp[0] = Mh;
            pp[1] = Ls;
        }
    }
}

template <int D>
__global__ void decode_merge_kernel(const float* __restrict__ part, int splits, float* __restrict__ out) {
    const int64_t head = blockIdx.x;  // l * Hq + h
    const float* pp = part + head * splits * (2 + D);
    float M = -INFINITY;
    for (int s = 0; s < splits; ++s) M = fmaxf(M, pp[s * (2 + D)]);
    float L = 0.0f;
    for (int s = 0; s < splits; ++s) {
        const float ms = pp[s * (2 + D)];
        L += ms == -INFINITY ? 0.0f : pp[s * (2 + D) + 1] * exp2f(ms - M);
    }
    for (int e = threadIdx.x; e < D; e += blockDim.x) {
        float acc = 0.0f;
        for (int s = 0; s < splits; ++s) {
            const float ms = pp[s * (2 + D)];
            if (ms != -INFINITY) acc += pp[s * (2 + D) + 2 + e] * exp2f(ms - M);
        }
        out[head * D + e] = L > 0.0f ? acc / L : 0.0f;
    }
}

template <int D, int G>
void run_decode(const DecodeShape& s, const void* q, const void* kc, const void* vc, float* out, DevBuf& ws,
                int sm_count, cudaStream_t st, const Paged& pg) {
    const int64_t heads = s.L * s.Hkv;
    // ~2 waves of CTAs (more splits cost more in per-CTA setup and the merge
    // than a partial last wave), at least 64 keys per split
    int64_t splits = (2 * sm_count + heads - 1) / heads;
    splits = std::max<int64_t>(1, std::min<int64_t>(splits, (s.K + 63) / 64));
    const int64_t chunk = (s.K + splits - 1) / splits;
    splits = (s.K + chunk - 1) / chunk;
    float* part = static_cast<float*>(ws.get(static_cast<size_t>(s.L * s.Hq * splits * (2 + D)) * 4));
    const dim3 grid((unsigned)splits, (unsigned)s.Hkv, (unsigned)s.L);
    static const bool mma_off = getenv("PKV_DECODE_MMA") && atoi(getenv("PKV_DECODE_MMA")) == 0;  // A/B knob
    if (!mma_off) {
        static std::atomic<uint64_t> attr{0};
        if (first_on_device(attr))
            PKV_CUDA(cudaFuncSetAttribute(decode_mma_kernel<D, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          MmaCfg<D>::kSmem));
        decode_mma_kernel<D, G><<<grid, 32 * kMmaWarps, MmaCfg<D>::kSmem, st>>>(
            static_cast<const __nv_bfloat16*>(q), static_cast<const __nv_bfloat16*>(kc),
            static_cast<const __nv_bfloat16*>(vc), (int)s.Hq, (int)s.Hkv, (int)(s.Hq / s.Hkv), s.K, chunk,
            s.scale * 1.4426950408889634f, part, pg, pg.table != nullptr);
    } else {
        auto kern = pg.table ? decode_split_kernel<D, G, true> : decode_split_kernel<D, G, false>;
        kern<<<grid, 32 * kWarps, 0, st>>>(static_cast<const __nv_bfloat16*>(q),
                                           static_cast<const __nv_bfloat16*>(kc),
                                           static_cast<const __nv_bfloat16*>(vc), (int)s.Hq, (int)s.Hkv,
                                           (int)(s.Hq / s.Hkv), s.K, chunk, s.scale * 1.4426950408889634f, part, pg);
    }
    check_launch("decode_split_kernel");
    decode_merge_kernel<D><<<(unsigned)(s.L * s.Hq), D, 0, st>>>(part, (int)splits, out);
    check_launch("decode_merge_kernel");
}

template <int D>
void dispatch_g(const DecodeShape& s, const void* q, const void* kc, const void* vc, float* out, DevBuf& ws, int sm,
                cudaStream_t st, const Paged& pg) {
    const int64_t g = s.Hq / s.Hkv;
    if (g <= 1) return run_decode<D, 1>(s, q, kc, vc, out, ws, sm, st, pg);
    if (g <= 2) return run_decode<D, 2>(s, q, kc, vc, out, ws, sm, st, pg);
    if (g <= 4) return run_decode<D, 4>(s, q, kc, vc, out, ws, sm, st, pg);
    return run_decode<D, 8>(s, q, kc, vc, out, ws, sm, st, pg);
}

}  // namespace

void launch_packed_decode(const DecodeShape& s, const void* q, const void* kc, const void* vc, float* out, DevBuf& ws,
                          int sm_count, cudaStream_t st) {
    if (s.d == 128) dispatch_g<128>(s, q, kc, vc, out, ws, sm_count, st, Paged{});
    else dispatch_g<64>(s, q, kc, vc, out, ws, sm_count, st, Paged{});
}

}  // namespace pkv

using namespace pkv;

extern "C" pkv_status pkv_packed_decode_attention(pkv_ctx ctx, const void* q_dev, const void* k_packed_dev,
                                                  const void* v_packed_dev, int64_t L, int64_t Hq, int64_t Hkv,
                                                  int64_t K, int64_t d, double scale, float* out_dev, void* stream) {
    return guard([&] {
        require_ctx(ctx);
        PKV_REQUIRE_SHAPE(L > 0 && Hq > 0 && Hkv > 0 && K > 0, "packed decode extents must be positive");
        PKV_REQUIRE_SHAPE(Hq % Hkv == 0, "query heads ", Hq, " not a multiple of KV heads ", Hkv);
        PKV_REQUIRE(d == 64 || d == 128, PKV_ECONFIG, "packed decode supports head_dim 64 or 128, got ", d);
        PKV_REQUIRE(Hq / Hkv <= kMaxG, PKV_ECONFIG, "packed decode supports GQA groups up to ", kMaxG);
        PKV_REQUIRE(L * Hkv <= 65535, PKV_ECONFIG, "too many (layer, KV head) pairs for one launch");
        DecodeShape s{L, Hq, Hkv, K, d, static_cast<float>(scale)};
        launch_packed_decode(s, q_dev, k_packed_dev, v_packed_dev, out_dev, ctx->scratch_decode, ctx->sm_count,
                             static_cast<cudaStream_t>(stream));
        count_launch(ctx, 2);
    });
}

extern "C" pkv_status pkv_paged_decode_attention(pkv_ctx ctx, const void* q_dev, const void* k_pool_dev,
                                                 const void* v_pool_dev, const int32_t* block_table_dev,
                                                 const int32_t* seq_lens_dev, int64_t L, int64_t Hq, int64_t Hkv,
                                                 int64_t max_blocks, int64_t page_size, int64_t max_len, int64_t d,
                                                 double scale, float* out_dev, void* stream) {
    return guard([&] {
        require_ctx(ctx);
        PKV_REQUIRE_SHAPE(L > 0 && Hq > 0 && Hkv > 0 && max_len > 0, "paged decode extents must be positive");
        PKV_REQUIRE_SHAPE(Hq % Hkv == 0, "query heads ", Hq, " not a multiple of KV heads ", Hkv);
        PKV_REQUIRE_VALUE(block_table_dev && seq_lens_dev && page_size > 0, "paged decode needs a block table");
        PKV_REQUIRE_VALUE(max_blocks * page_size >= max_len, "block table too short for max_len ", max_len);
        PKV_REQUIRE(d == 64 || d == 128, PKV_ECONFIG, "paged decode supports head_dim 64 or 128, got ", d);
        PKV_REQUIRE(Hq / Hkv <= kMaxG, PKV_ECONFIG, "paged decode supports GQA groups up to ", kMaxG);
        PKV_REQUIRE(L * Hkv <= 65535, PKV_ECONFIG, "too many (layer, KV head) pairs for one launch");
        // splits sized on max_len; slabs shorter than a split's start contribute nothing
        DecodeShape s{L, Hq, Hkv, max_len, d, static_cast<float>(scale)};
        const Paged pg{block_table_dev, seq_lens_dev, max_blocks, page_size};
        auto st = static_cast<cudaStream_t>(stream);
        if (d == 128) dispatch_g<128>(s, q_dev, k_pool_dev, v_pool_dev, out_dev, ctx->scratch_decode, ctx->sm_count, st, pg);
        else dispatch_g<64>(s, q_dev, k_pool_dev, v_pool_dev, out_dev, ctx->scratch_decode, ctx->sm_count, st, pg);
        count_launch(ctx, 2);
    });
}
