// sm100.cuh — thin inline-PTX layer for Blackwell (sm_100a): mbarriers, TMA,
// tcgen05 (TMEM alloc / MMA / commit / ld) and UMMA descriptors.
// Everything here is hand-written PTX; compile with
// -gencode arch=compute_100a,code=sm_100a.
#pragma once

#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace pkv {
namespace sm100 {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t warp_id() { return threadIdx.x >> 5; }
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }

__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "elect.sync _|P, 0xffffffff;\n\t"
        "selp.b32 %0, 1, 0, P;\n\t}"
        : "=r"(pred));
    return pred != 0;
}

// ---------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2, 0x989680;\n\t"
        "selp.b32 %0, 1, 0, P;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}

// --------------------------------------------------------------------- TMA
__device__ __forceinline__ void tma_prefetch(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t c0,
                                            int32_t c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t c0,
                                            int32_t c1, int32_t c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}

// ----------------------------------------------------- clusters (CTA pairs)
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Address of the same smem object in CTA `rank` of the cluster.
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
// Relaxed: used to hand a TMEM accumulator back to the pair's MMA issuer after
// tcgen05.wait::ld + tcgen05.fence::before_thread_sync; a .release arrive would
// make every epilogue warp drain its global stores first (MEMBAR.ALL.GPU).
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// 2-SM TMA: both CTAs of the pair load their half; the bytes complete on the
// leader CTA's barrier (peer bit 24 of the shared::cluster address cleared).
__device__ __forceinline__ void tma_load_2d_2sm(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t c0,
                                                int32_t c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
        "%4}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void tmem_alloc_2sm(uint32_t* smem_dst, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_dst)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_2sm(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
// Pair MMA, issued by the leader CTA: D (M = 256 across both CTAs' TMEM) += A·Bᵀ.
__device__ __forceinline__ void mma_f16_ss_2sm(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                               uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void mma_f8_ss_2sm(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// Commit the pair's MMAs to the same-offset barrier in every CTA of `mask`.
__device__ __forceinline__ void mma_commit_2sm(uint64_t* bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(mask)
        : "memory");
}

// ----------------------------------------------------------------- tcgen05
// TMEM allocation: one full warp executes alloc/dealloc.
__device__ __forceinline__ void tmem_alloc(uint32_t* smem_dst, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_dst)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// D[tmem] (+)= A[smem] * B[smem]^T, kind::f16 (fp16/bf16 in, fp32 accumulate).
__device__ __forceinline__ void mma_f16_ss(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                           uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// D[tmem] (+)= A[tmem] * B[smem]^T, kind::f16: A (M = 128 rows = TMEM lanes,
// K packed two fp16 per 32-bit column) is read from tensor memory.
__device__ __forceinline__ void mma_f16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                           uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// D[tmem] (+)= A[smem] * B[smem]^T, kind::f8f6f4 (e4m3 in with the same
// instruction descriptor bits as kind::f16 / fp16, fp32 accumulate): K = 32 per
// instruction. Accumulates into the same fp32 TMEM tile as kind::f16 MMAs
// (tools/probe_f8mma.cu checks the mixed accumulation).
__device__ __forceinline__ void mma_f8_ss(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// Arrive on an mbarrier once all previously issued tcgen05.mma of this thread
// complete (implicitly fences before_thread_sync).
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

// 32 lanes x 32 columns of 32-bit: thread t of the warp gets TMEM lane
// (base lane + t), columns [col, col + 32).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}

// 32 lanes x 64 columns in one instruction (one MIO op for a 64-column chunk).
__device__ __forceinline__ void tmem_ld64(uint32_t taddr, uint32_t (&a)[32], uint32_t (&b)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x64.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,"
        "%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,"
        "%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
        : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]), "=r"(a[4]), "=r"(a[5]), "=r"(a[6]), "=r"(a[7]),
          "=r"(a[8]), "=r"(a[9]), "=r"(a[10]), "=r"(a[11]), "=r"(a[12]), "=r"(a[13]), "=r"(a[14]), "=r"(a[15]),
          "=r"(a[16]), "=r"(a[17]), "=r"(a[18]), "=r"(a[19]), "=r"(a[20]), "=r"(a[21]), "=r"(a[22]), "=r"(a[23]),
          "=r"(a[24]), "=r"(a[25]), "=r"(a[26]), "=r"(a[27]), "=r"(a[28]), "=r"(a[29]), "=r"(a[30]), "=r"(a[31]),
          "=r"(b[0]), "=r"(b[1]), "=r"(b[2]), "=r"(b[3]), "=r"(b[4]), "=r"(b[5]), "=r"(b[6]), "=r"(b[7]),
          "=r"(b[8]), "=r"(b[9]), "=r"(b[10]), "=r"(b[11]), "=r"(b[12]), "=r"(b[13]), "=r"(b[14]), "=r"(b[15]),
          "=r"(b[16]), "=r"(b[17]), "=r"(b[18]), "=r"(b[19]), "=r"(b[20]), "=r"(b[21]), "=r"(b[22]), "=r"(b[23]),
          "=r"(b[24]), "=r"(b[25]), "=r"(b[26]), "=r"(b[27]), "=r"(b[28]), "=r"(b[29]), "=r"(b[30]), "=r"(b[31])
        : "r"(taddr));
}

__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// registers -> TMEM, same 32x32b.x32 shape as tmem_ld32.
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]),
        "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]),
        "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}

// registers -> TMEM, 32x32b.x16 (16 columns).
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* r) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}

// 32x32b.x8 (8 columns) load / store: small register footprint for rare paths.
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
                 "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}

__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// Packed fp32x2 arithmetic (sm_100: FFMA2 / FADD2 — two lanes' worth of
// fp32 work per instruction slot).
__device__ __forceinline__ uint64_t pack2(float lo, float hi) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ float2 unpack2(uint64_t v) {
    float2 r;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
    return r;
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ uint64_t fsub2(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}

// Broadcast-operand forms: a scalar duplicated into both halves inside the asm
// lets ptxas encode it as a .F32 broadcast register or an immediate, so the
// FFMA2 reads 3-4 32-bit registers instead of 6 (measured: 6-register FFMA2
// issues every 3 cycles per SMSP, 4-register ones every 2; tools/probe_exp.cu).
// a2 * b + c, b and c scalars
__device__ __forceinline__ uint64_t ffma2_ss(uint64_t a, float b, float c) {
    uint64_t d;
    asm("{.reg .b64 bb, cc;\n\tmov.b64 bb, {%2, %2};\n\tmov.b64 cc, {%3, %3};\n\t"
        "fma.rn.f32x2 %0, %1, bb, cc;}"
        : "=l"(d)
        : "l"(a), "f"(b), "f"(c));
    return d;
}
// a2 * b + c2, b scalar
__device__ __forceinline__ uint64_t ffma2_sp(uint64_t a, float b, uint64_t c) {
    uint64_t d;
    asm("{.reg .b64 bb;\n\tmov.b64 bb, {%2, %2};\n\tfma.rn.f32x2 %0, %1, bb, %3;}" : "=l"(d) : "l"(a), "f"(b), "l"(c));
    return d;
}
// a2 * b2 + c, c scalar
__device__ __forceinline__ uint64_t ffma2_ps(uint64_t a, uint64_t b, float c) {
    uint64_t d;
    asm("{.reg .b64 cc;\n\tmov.b64 cc, {%3, %3};\n\tfma.rn.f32x2 %0, %1, %2, cc;}" : "=l"(d) : "l"(a), "l"(b), "f"(c));
    return d;
}
// a - b2, a scalar
__device__ __forceinline__ uint64_t fsub2_s(float a, uint64_t b) {
    uint64_t d;
    asm("{.reg .b64 aa;\n\tmov.b64 aa, {%1, %1};\n\tsub.rn.f32x2 %0, aa, %2;}" : "=l"(d) : "f"(a), "l"(b));
    return d;
}

// ex2_poly2_fused with scalar c (ideally a compile-time constant: an FFMA2
// immediate) and mp = 1.5·2^23 − m: 2^(c·s − m) for both halves of s2.
__device__ __forceinline__ uint64_t ex2_poly2_fused_s(uint64_t s2, float c, float mp) {
    uint64_t t = ffma2_ss(s2, c, mp);
    float2 tf = unpack2(t);
    tf.x = fmaxf(tf.x, 12582912.0f - 125.0f);
    tf.y = fmaxf(tf.y, 12582912.0f - 125.0f);
    t = pack2(tf.x, tf.y);
    const uint64_t f = ffma2_sp(s2, c, fsub2_s(mp, t));
    uint64_t p = ffma2_ss(f, 0.05508868396282196f, 0.24260404706001282f);
    p = ffma2_ps(p, f, 0.6932762265205383f);
    p = ffma2_ps(p, f, 0.9999289512634277f);
    const float2 pf = unpack2(p);
    return pack2(__int_as_float((__float_as_int(tf.x) << 23) + __float_as_int(pf.x)),
                 __int_as_float((__float_as_int(tf.y) << 23) + __float_as_int(pf.y)));
}

// Two 2^x (x <= 0) on the FMA pipe with packed FADD2/FFMA2 (see ex2_poly).
__device__ __forceinline__ uint64_t ex2_poly2(uint64_t x2) {
    float2 x = unpack2(x2);
    x.x = fmaxf(x.x, -125.0f);
    x.y = fmaxf(x.y, -125.0f);
    const uint64_t xv = pack2(x.x, x.y);
    const uint64_t t = fadd2(xv, pack2(12582912.0f, 12582912.0f));
    const uint64_t j = fsub2(t, pack2(12582912.0f, 12582912.0f));
    const uint64_t f = fsub2(xv, j);
    uint64_t p = ffma2(pack2(0.009560510516166687f, 0.009560510516166687f), f,
                       pack2(0.05591703951358795f, 0.05591703951358795f));
    p = ffma2(p, f, pack2(0.24024981260299683f, 0.24024981260299683f));
    p = ffma2(p, f, pack2(0.6931219696998596f, 0.6931219696998596f));
    p = ffma2(p, f, pack2(0.9999991655349731f, 0.9999991655349731f));
    const float2 pf = unpack2(p), tf = unpack2(t);
    return pack2(__int_as_float(__float_as_int(tf.x) * 8388608 + __float_as_int(pf.x)),
                 __int_as_float(__float_as_int(tf.y) * 8388608 + __float_as_int(pf.y)));
}

// Cheaper pair variant for sums that tolerate 8e-5 relative error per term
// (the LSE pass): degree-3 fit of 2^f on [-0.5, 0.5] (max rel err 7.7e-5), and
// the exponent insertion as shift+add (LEA on the ALU pipe, off the FMA pipe).
__device__ __forceinline__ uint64_t ex2_poly2_d3(uint64_t x2) {
    float2 x = unpack2(x2);
    x.x = fmaxf(x.x, -125.0f);
    x.y = fmaxf(x.y, -125.0f);
    const uint64_t xv = pack2(x.x, x.y);
    const uint64_t t = fadd2(xv, pack2(12582912.0f, 12582912.0f));
    const uint64_t j = fsub2(t, pack2(12582912.0f, 12582912.0f));
    const uint64_t f = fsub2(xv, j);
    uint64_t p = ffma2(pack2(0.05508868396282196f, 0.05508868396282196f), f,
                       pack2(0.24260404706001282f, 0.24260404706001282f));
    p = ffma2(p, f, pack2(0.6932762265205383f, 0.6932762265205383f));
    p = ffma2(p, f, pack2(0.9999289512634277f, 0.9999289512634277f));
    const float2 pf = unpack2(p), tf = unpack2(t);
    return pack2(__int_as_float((__float_as_int(tf.x) << 23) + __float_as_int(pf.x)),
                 __int_as_float((__float_as_int(tf.y) << 23) + __float_as_int(pf.y)));
}

// 2^(c·s − m) for a pair, with an INTEGER row offset m folded into the range
// reduction: mp = 1.5·2^23 − m (exact for |m| < 2^22). t = c·s + mp rounds to
// 1.5·2^23 + j (j = rint(c·s − m)); mp − t is exact (Sterbenz), so f = c·s +
// (mp − t) = (c·s − m) − j in one FFMA. 3 packed FP ops replace the scale
// FFMA + 3-op magic-number reduction. j is clamped at −125 (2^f ≥ 0.7 keeps the exponent field ≥ 1; 2^f·2^−125 is
// negligible); inputs must be finite. Degree-3 fit as ex2_poly2_d3.
__device__ __forceinline__ uint64_t ex2_poly2_fused(uint64_t s2, uint64_t c2, uint64_t mp2) {
    uint64_t t = ffma2(s2, c2, mp2);
    float2 tf = unpack2(t);
    tf.x = fmaxf(tf.x, 12582912.0f - 125.0f);
    tf.y = fmaxf(tf.y, 12582912.0f - 125.0f);
    t = pack2(tf.x, tf.y);
    const uint64_t f = ffma2(s2, c2, fsub2(mp2, t));
    uint64_t p = ffma2(pack2(0.05508868396282196f, 0.05508868396282196f), f,
                       pack2(0.24260404706001282f, 0.24260404706001282f));
    p = ffma2(p, f, pack2(0.6932762265205383f, 0.6932762265205383f));
    p = ffma2(p, f, pack2(0.9999289512634277f, 0.9999289512634277f));
    const float2 pf = unpack2(p);
    return pack2(__int_as_float((__float_as_int(tf.x) << 23) + __float_as_int(pf.x)),
                 __int_as_float((__float_as_int(tf.y) << 23) + __float_as_int(pf.y)));
}

// 2^x for x <= 0 on the FMA pipe (FA4-style MUFU offload): x = j + f with
// j = rint(x), f ∈ [-0.5, 0.5]; 2^f by a degree-4 fit (max rel err 2.7e-6);
// the exponent j is added as an integer.
__device__ __forceinline__ float ex2_poly(float x) {
    x = fmaxf(x, -125.0f);
    const float t = x + 12582912.0f;  // 1.5·2^23: low mantissa bits = rint(x)
    const float j = t - 12582912.0f;
    const float f = x - j;
    float p = fmaf(0.009560510516166687f, f, 0.05591703951358795f);
    p = fmaf(p, f, 0.24024981260299683f);
    p = fmaf(p, f, 0.6931219696998596f);
    p = fmaf(p, f, 0.9999991655349731f);
    return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

// Generic-proxy smem writes -> visible to the async proxy (tcgen05.mma / TMA).
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Exact-erf GELU, 0.5·x·(1 + erf(x/√2)) (ops.cpp:225-234), branch-free:
// erfc(z) = t·P5(t)·e^(−z²), t = 1/(1 + p·z) (Abramowitz–Stegun 7.1.26, |Δerf|
// ≤ 1.5e-7); GELU = x − x·erfc/2 for x ≥ 0, x·erfc/2 otherwise. Max abs error
// 5.3e-7 on [−8, 8] in fp32 (the fp32 erff form: 6.8e-7), 2 MUFU + ~14 FMA-pipe
// ops instead of erff's two-range polynomial.
__device__ __forceinline__ float gelu_fast(float x) {
    const float z = fabsf(x) * 0.70710678118654752f;
    const float t = rcp_approx(fmaf(0.3275911f, z, 1.0f));
    float p = fmaf(1.061405429f, t, -1.453152027f);
    p = fmaf(p, t, 1.421413741f);
    p = fmaf(p, t, -0.284496736f);
    p = fmaf(p, t, 0.254829592f);
    const float e = ex2((z * -1.4426950408889634f) * z);
    const float h = (0.5f * x) * ((p * t) * e);
    return x >= 0.0f ? x - h : h;
}

// Three-input max (sm_100+).
__device__ __forceinline__ float max3f(float a, float b, float c) {
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}

__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ------------------------------------------------------------ descriptors
// Shared-memory matrix descriptor, K-major operand in the canonical
// 128-byte-swizzle layout TMA (CU_TENSOR_MAP_SWIZZLE_128B) writes: rows of
// 128 B, 8-row core groups 1024 B apart (SBO), tile base 1024-B aligned.
__device__ __forceinline__ uint64_t desc_sw128(const void* smem_tile) {
    const uint64_t addr = smem_u32(smem_tile);
    uint64_t d = 0;
    d |= (addr >> 4) & 0x3FFFull;          // start address  [0,14)
    d |= 1ull << 16;                        // LBO (ignored for swizzled K-major) [16,30)
    d |= (uint64_t)(1024 >> 4) << 32;       // SBO = 1024 B   [32,46)
    d |= 1ull << 46;                        // version = 1 (sm100)
    d |= 2ull << 61;                        // SWIZZLE_128B
    return d;
}

// K-major e4m3 operand in the 64-byte-swizzle layout TMA
// (CU_TENSOR_MAP_SWIZZLE_64B) writes for 64-element K blocks: rows of 64 B,
// 8-row core groups 512 B apart (SBO), tile base 512-B aligned. The second
// K = 32 half of a row is +32 B (+2 in the address field), as with SW128.
__device__ __forceinline__ uint64_t desc_sw64(const void* smem_tile) {
    const uint64_t addr = smem_u32(smem_tile);
    uint64_t d = 0;
    d |= (addr >> 4) & 0x3FFFull;
    d |= 1ull << 16;
    d |= (uint64_t)(512 >> 4) << 32;  // SBO = 512 B
    d |= 1ull << 46;
    d |= 4ull << 61;  // SWIZZLE_64B
    return d;
}

// MN-major operand (e.g. V[keys][d] as B of P·V), 128-B swizzle: 64 elements
// of N contiguous per 128-B row, K rows 128 B apart, 8-row groups 1024 B
// apart (SBO); LBO = byte distance between 64-element N groups.
__device__ __forceinline__ uint64_t desc_sw128_mn(const void* smem_tile, uint32_t lbo_bytes) {
    const uint64_t addr = smem_u32(smem_tile);
    uint64_t d = 0;
    d |= (addr >> 4) & 0x3FFFull;
    d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= 1ull << 46;
    d |= 2ull << 61;
    return d;
}

// Instruction descriptor for kind::f16: fp16 A/B (fmt 0) or bf16 (fmt 1),
// fp32 accumulate, M = 128, N = n; a_mn/b_mn select MN-major operands.
__host__ __device__ constexpr uint32_t idesc_f16(uint32_t m, uint32_t n, uint32_t ab_fmt, uint32_t a_mn = 0,
                                                 uint32_t b_mn = 0) {
    return (1u << 4)               // D = f32
           | (ab_fmt << 7)         // A format
           | (ab_fmt << 10)        // B format
           | (a_mn << 15)          // A major
           | (b_mn << 16)          // B major
           | ((n >> 3) << 17)      // N / 8
           | ((m >> 4) << 24);     // M / 16
}

}  // namespace sm100
}  // namespace pkv
