// test_hooks.cpp — unit-test entry points (include/pkv_test_hooks.h).
#include "../../include/pkv_test_hooks.h"

#include "attn.cuh"
#include "gemm.cuh"
#include "util.cuh"

using namespace pkv;

extern "C" pkv_status pkv_test_gemm(pkv_ctx ctx, const float* a_dev, int64_t M, int64_t K, const float* b_dev,
                                    int64_t N, int na, int nb, int bn, int epi, const float* bias_dev,
                                    const float* pe_dev, int64_t lw, float* out_dev, void* stream) {
    return guard([&] {
        require_ctx(ctx);
        PKV_REQUIRE_VALUE(K % 8 == 0, "K must be a multiple of 8 (16-byte TMA rows)");
        auto st = static_cast<cudaStream_t>(stream);
        DevBuf buf;
        const size_t a_el = (size_t)(M * K), b_el = (size_t)(N * K), o_el = (size_t)(M * N);
        auto* base = static_cast<__half*>(buf.get((2 * a_el + 2 * b_el + 2 * o_el) * sizeof(__half)));
        __half *ah = base, *al = ah + a_el, *bh = al + a_el, *bl = bh + b_el, *oh = bl + b_el, *ol = oh + o_el;
        launch_split_f16(a_dev, (int64_t)a_el, ah, na > 1 ? al : nullptr, st);
        launch_split_f16(b_dev, (int64_t)b_el, bh, nb > 1 ? bl : nullptr, st);
        GemmArgs g;
        g.bn = bn == 512 ? 256 : bn;  // 512 selects the CTA-pair 256x256 kernel
        g.pair = bn == 512;
        g.epi = static_cast<GemmEpi>(epi);
        gemm_set_a(g, 0, ah, M, K, K);
        g.a[1] = g.a[0];
        if (na > 1) gemm_set_a(g, 1, al, M, K, K);
        gemm_set_b(g, 0, bh, N, K, K);
        g.b[1] = g.b[0];
        if (nb > 1) gemm_set_b(g, 1, bl, N, K, K);
        g.p.bias = bias_dev;
        g.p.pe = pe_dev;
        g.p.lw = lw > 0 ? lw : 1;
        g.p.ldo = N;
        const bool planes = (epi == EPI_F16X || epi == EPI_GELU_F16X);
        if (planes) {
            g.p.out_h = oh;
            g.p.out_l = ol;
        } else {
            g.p.out_f32 = out_dev;
        }
        gemm_run(g, ctx->sm_count, st);
        if (planes) launch_combine_f16(oh, ol, (int64_t)o_el, out_dev, st);
        PKV_CUDA(cudaStreamSynchronize(st));
        count_launch(ctx, 3);
    });
}

extern "C" pkv_status pkv_test_attention(pkv_ctx ctx, const float* qkv_dev, int64_t nwin, int64_t Lw, int64_t D,
                                         int64_t heads, float* out_dev, void* stream) {
    return guard([&] {
        require_ctx(ctx);
        auto st = static_cast<cudaStream_t>(stream);
        DevBuf buf;
        const size_t in_el = (size_t)(nwin * Lw * 3 * D), o_el = (size_t)(nwin * Lw * D);
        auto* base = static_cast<__half*>(buf.get((in_el + 2 * o_el) * sizeof(__half)));
        __half *q = base, *oh = q + in_el, *ol = oh + o_el;
        launch_split_f16(qkv_dev, (int64_t)in_el, q, nullptr, st);
        launch_encoder_attention(q, nwin, Lw, D, heads, oh, ol, D, st);
        launch_combine_f16(oh, ol, (int64_t)o_el, out_dev, st);
        PKV_CUDA(cudaStreamSynchronize(st));
        count_launch(ctx, 3);
    });
}
