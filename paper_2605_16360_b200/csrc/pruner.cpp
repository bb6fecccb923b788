// pruner.cpp — the whole hot path for one context shape, stream-ordered on
// the caller's stream: score (proxy Q·Kᵀ, pooled) -> HybridAxialMapper
// forward_full -> per-(layer, head) Top-K select (ascending indices) -> packed
// KV gather. No host synchronisation inside pkv_pruner_run; the host-buffer
// form adds the H2D / D2H copies and synchronises once at the end.
#include <cmath>
#include <map>

#include "mapper.h"
#include "score.cuh"

using namespace pkv;

struct pkv_pruner_s {
    pkv_ctx ctx = nullptr;
    Mapper* mapper = nullptr;
    ScoreShape score;
    bool reduce_max = true;
    int64_t dt = 0, N = 0, K = 0, Ll = 0, Hl = 0;
    std::vector<int64_t> unit_off;
    std::vector<int> out_unit;
    DevBuf lam, x, y, idx;
    DevBuf host_in, host_out;  // device copies for the host-buffer form
};

extern "C" {

pkv_status pkv_pruner_create(pkv_ctx ctx, pkv_mapper m, int64_t Hq, int64_t dp, int64_t dt, int64_t N, double rho,
                             uint32_t score_flags, pkv_pruner* out) {
    return guard([&] {
        require_ctx(ctx);
        PKV_REQUIRE_VALUE(m != nullptr, "null pkv_mapper");
        Mapper& mp = *m->m;
        PKV_REQUIRE_VALUE(rho > 0.0 && rho <= 1.0, "retention ratio must be in (0, 1], got ", rho);
        PKV_REQUIRE_VALUE(N > 0 && dt > 0, "context length and target head_dim must be positive");
        auto* p = new pkv_pruner_s();
        p->ctx = ctx;
        p->mapper = &mp;
        p->score = ScoreShape{mp.geom.proxy_layers, Hq, mp.geom.proxy_heads, N, N, dp,
                              (score_flags & PKV_SCORE_CAUSAL) != 0};
        try {
            score_validate(p->score);
        } catch (...) {
            delete p;
            throw;
        }
        p->reduce_max = (score_flags & PKV_SCORE_REDUCE_SUM) == 0;
        p->dt = dt;
        p->N = N;
        p->K = static_cast<int64_t>(std::ceil(rho * static_cast<double>(N)));  // pruning.cpp:17
        p->Ll = mp.geom.target_layers;
        p->Hl = mp.geom.target_heads;
        std::map<int64_t, int> unit_of;
        for (int64_t ll = 1; ll <= p->Ll; ++ll) {
            const int64_t ls = layer_pair(ll, mp.geom);
            auto it = unit_of.find(ls);
            if (it == unit_of.end()) {
                it = unit_of.emplace(ls, static_cast<int>(p->unit_off.size())).first;
                p->unit_off.push_back((ls - 1) * mp.geom.proxy_heads * N);
            }
            p->out_unit.push_back(it->second);
        }
        *out = p;
    });
}

void pkv_pruner_destroy(pkv_pruner p) { delete p; }

int64_t pkv_pruner_k(pkv_pruner p) { return p ? p->K : 0; }

pkv_status pkv_pruner_run(pkv_pruner p, const void* q, const void* kp, const void* kt, const void* vt, void* k_out,
                          void* v_out, int32_t* idx_out, float* scores_out, void* stream) {
    return guard([&] {
        PKV_REQUIRE_VALUE(p != nullptr, "null pkv_pruner");
        auto st = static_cast<cudaStream_t>(stream);
        const ScoreShape& s = p->score;
        auto* lam = static_cast<__nv_bfloat16*>(p->lam.get(static_cast<size_t>(s.L * s.Hq * s.Nq) * 16));
        auto* x = static_cast<float*>(p->x.get(static_cast<size_t>(s.L * s.Hkv * s.Nk) * 4));
        float* y = scores_out ? scores_out
                              : static_cast<float*>(p->y.get(static_cast<size_t>(p->Ll * p->Hl * p->N) * 4));
        int32_t* idx = idx_out ? idx_out : static_cast<int32_t*>(p->idx.get(static_cast<size_t>(p->Ll * p->Hl * p->K) * 4));
        // (1) proxy scoring: X [1, L_s, H_s, N]
        launch_score_lse(s, q, kp, nullptr, lam, st);
        launch_score_pool(s, q, kp, lam, p->reduce_max, x, st);
        count_launch(p->ctx, 2);
        // (2) mapper: Ŷ [1, L_l, H_l, N]
        p->mapper->run(x, p->unit_off, p->N, p->out_unit, y, st);
        // (3) Top-K per (target layer, head): ascending retained indices
        launch_topk_select(y, p->Ll * p->Hl, p->N, p->K, nullptr, idx, st);
        // (4) packed KV gather
        launch_compact_kv(kt, vt, idx, p->Ll * p->Hl, p->N, p->K, p->dt * 2, k_out, v_out, p->ctx->sm_count, st);
        count_launch(p->ctx, 2);
    });
}

pkv_status pkv_pruner_run_host(pkv_pruner p, const void* q_h, const void* kp_h, const void* kt_h, const void* vt_h,
                               void* k_out_h, void* v_out_h, int32_t* idx_out_h, void* stream) {
    return guard([&] {
        PKV_REQUIRE_VALUE(p != nullptr, "null pkv_pruner");
        auto st = static_cast<cudaStream_t>(stream);
        const ScoreShape& s = p->score;
        const size_t qb = static_cast<size_t>(s.L * s.Hq * s.Nq * s.d) * 2;
        const size_t kpb = static_cast<size_t>(s.L * s.Hkv * s.Nk * s.d) * 2;
        const size_t kvb = static_cast<size_t>(p->Ll * p->Hl * p->N * p->dt) * 2;
        const size_t ob = static_cast<size_t>(p->Ll * p->Hl * p->K * p->dt) * 2;
        const size_t ib = static_cast<size_t>(p->Ll * p->Hl * p->K) * 4;
        auto* in = static_cast<uint8_t*>(p->host_in.get(qb + kpb + 2 * kvb));
        auto* outb = static_cast<uint8_t*>(p->host_out.get(2 * ob + ib));
        PKV_CUDA(cudaMemcpyAsync(in, q_h, qb, cudaMemcpyHostToDevice, st));
        PKV_CUDA(cudaMemcpyAsync(in + qb, kp_h, kpb, cudaMemcpyHostToDevice, st));
        PKV_CUDA(cudaMemcpyAsync(in + qb + kpb, kt_h, kvb, cudaMemcpyHostToDevice, st));
        PKV_CUDA(cudaMemcpyAsync(in + qb + kpb + kvb, vt_h, kvb, cudaMemcpyHostToDevice, st));
        const pkv_status rc = pkv_pruner_run(p, in, in + qb, in + qb + kpb, in + qb + kpb + kvb, outb, outb + ob,
                                             reinterpret_cast<int32_t*>(outb + 2 * ob), nullptr, stream);
        if (rc != PKV_OK) throw Error{rc, pkv_last_error()};
        PKV_CUDA(cudaMemcpyAsync(k_out_h, outb, ob, cudaMemcpyDeviceToHost, st));
        PKV_CUDA(cudaMemcpyAsync(v_out_h, outb + ob, ob, cudaMemcpyDeviceToHost, st));
        if (idx_out_h) PKV_CUDA(cudaMemcpyAsync(idx_out_h, outb + 2 * ob, ib, cudaMemcpyDeviceToHost, st));
        PKV_CUDA(cudaStreamSynchronize(st));
    });
}

}  // extern "C"
