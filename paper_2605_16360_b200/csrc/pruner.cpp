// pruner.cpp — the whole hot path for one context shape, stream-ordered on
// the caller's stream: score (proxy Q·Kᵀ, pooled) -> HybridAxialMapper
// forward_full -> per-(layer, head) Top-K select (ascending indices) -> packed
// KV gather. No host synchronisation inside pkv_pruner_run; the host-buffer
// form adds the H2D / D2H copies and synchronises once at the end. A sharded
// pruner (shard.cpp) runs the same steps on its part of one context.
#include <algorithm>
#include <cmath>
#include <map>
#include <memory>

#include "mapper.h"
#include "score.cuh"
#include "shard.h"

using namespace pkv;

struct pkv_pruner_s {
    pkv_ctx ctx = nullptr;
    Mapper* mapper = nullptr;
    ScoreShape score;  // proxy layers [plan.p_lo, plan.p_hi) of the full proxy tensors
    bool reduce_max = true;
    int64_t dt = 0, N = 0, K = 0, Ll = 0, Hl = 0, Hq = 0, dp = 0;
    ShardPlan plan;  // world 1, layer mode = the whole context on one GPU
    pkv_comm comm = nullptr;
    std::vector<int64_t> unit_off;  // mapper units (unique proxy layers of target layers [a, b))
    std::vector<int> out_unit;      // target layer a + i -> unit
    DevBuf lam, x, y, y_local, idx;
    DevBuf score_aux;  // fixed-reference pass 1 scratch
    DevBuf y_remote;  // two-device mode: Ŷ on the target device (allocated there)
    cudaEvent_t ev_remote = nullptr;
    DevBuf host_in, host_out;  // device copies for the host-buffer form
    cudaEvent_t ev = nullptr;
    // host-buffer form: copy stream + events (proxy layer chunks, target KV)
    cudaStream_t copy_st = nullptr;
    static constexpr int kChunks = 16;  // proxy-layer chunks of the H2D
    static constexpr int kGroups = 8;   // target-layer groups of the map -> select -> compact -> D2H tail
    static constexpr int kSub = 4;      // KV-head groups of the first chunk (its copy is the exposed one)
    cudaEvent_t ev_in[kChunks + 2] = {};
    cudaEvent_t ev_sub[kSub] = {};
    cudaEvent_t ev_grp[kGroups + 1] = {};
    // stage profiling (pkv_pruner_profile): kProfEv events per run at the stage boundaries
    // (LSE pass | pooled pass | map | select | compaction), recorded on the launching streams
    static constexpr int kProfEv = 6;
    std::vector<cudaEvent_t> prof_ev;
    int64_t prof_max = 0, prof_next = 0;
    cudaEvent_t prof(int i) const { return prof_ev[static_cast<size_t>(prof_next * kProfEv + i)]; }
    ~pkv_pruner_s() {
        if (ev) cudaEventDestroy(ev);
        if (ev_remote) cudaEventDestroy(ev_remote);
        for (cudaEvent_t e : ev_in)
            if (e) cudaEventDestroy(e);
        for (cudaEvent_t e : ev_grp)
            if (e) cudaEventDestroy(e);
        for (cudaEvent_t e : ev_sub)
            if (e) cudaEventDestroy(e);
        for (cudaEvent_t e : prof_ev) cudaEventDestroy(e);
        if (copy_st) cudaStreamDestroy(copy_st);
    }
    int64_t slices() const { return (plan.t_hi - plan.t_lo) * (plan.h_hi - plan.h_lo); }
};

namespace {

// Inputs arriving from the host (pkv_pruner_run_host): scoring of proxy-layer
// chunk c waits for ev_chunk[c]; select + compaction wait for ev_kv.
struct HostArrival {
    int chunks = 0;
    int64_t chunk_layers = 0;
    const cudaEvent_t* ev_chunk = nullptr;
    // chunk 0 (one proxy layer) split into `sub` KV-head groups, each scored as
    // soon as its own copy lands (ev_sub[s]): only the first group's copy is
    // exposed before the GPU starts
    int sub = 1;
    const cudaEvent_t* ev_sub = nullptr;
    cudaEvent_t ev_kv = nullptr;
    // outputs leaving for the host: when set (layer mode), the tail runs per
    // target-layer group and each group's packed K/V + indices are copied out
    // on `copy` while the next group is mapped
    void* k_out_h = nullptr;
    void* v_out_h = nullptr;
    int32_t* idx_out_h = nullptr;
    cudaStream_t copy = nullptr;
    const cudaEvent_t* ev_grp = nullptr;  // kGroups + 1
};

// map -> select -> compact per group of target layers (contiguous unit
// blocks, so no unit is mapped twice), each group's outputs D2H on arr.copy
// while the next group is mapped; `ps` finally waits for the last copy.
void grouped_tail(pkv_pruner p, const float* x, const void* kt, const void* vt, void* k_out, void* v_out,
                  int32_t* idx, float* y, cudaStream_t ps, const HostArrival& arr) {
    const int64_t units = static_cast<int64_t>(p->unit_off.size());
    const int64_t nt = static_cast<int64_t>(p->out_unit.size());
    const int G = static_cast<int>(std::min<int64_t>(pkv_pruner_s::kGroups, units));
    const size_t row_kv = static_cast<size_t>(p->N * p->dt) * 2, row_out = static_cast<size_t>(p->K * p->dt) * 2;
    int64_t t0 = 0;
    for (int g = 0; g < G; ++g) {
        const int64_t u0 = units * g / G, u1 = units * (g + 1) / G;
        int64_t t1 = t0;
        while (t1 < nt && p->out_unit[t1] < u1) ++t1;
        if (t1 == t0) continue;
        std::vector<int64_t> uo(p->unit_off.begin() + u0, p->unit_off.begin() + u1);
        std::vector<int> ou(p->out_unit.begin() + t0, p->out_unit.begin() + t1);
        for (int& v : ou) v -= static_cast<int>(u0);
        p->mapper->run(x, uo, p->N, ou, y + t0 * p->Hl * p->N, ps);
        if (g == 0) PKV_CUDA(cudaStreamWaitEvent(ps, arr.ev_kv, 0));
        const int64_t s0 = t0 * p->Hl, ns = (t1 - t0) * p->Hl;
        launch_topk_select(y + s0 * p->N, ns, p->N, p->K, nullptr, idx + s0 * p->K, ps);
        launch_compact_kv(static_cast<const uint8_t*>(kt) + s0 * row_kv, static_cast<const uint8_t*>(vt) + s0 * row_kv,
                          idx + s0 * p->K, ns, p->N, p->K, p->dt * 2, static_cast<uint8_t*>(k_out) + s0 * row_out,
                          static_cast<uint8_t*>(v_out) + s0 * row_out, p->ctx->sm_count, ps);
        count_launch(p->ctx, 2);
        PKV_CUDA(cudaEventRecord(arr.ev_grp[g], ps));
        PKV_CUDA(cudaStreamWaitEvent(arr.copy, arr.ev_grp[g], 0));
        PKV_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(arr.k_out_h) + s0 * row_out,
                                 static_cast<uint8_t*>(k_out) + s0 * row_out, ns * row_out, cudaMemcpyDeviceToHost,
                                 arr.copy));
        PKV_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(arr.v_out_h) + s0 * row_out,
                                 static_cast<uint8_t*>(v_out) + s0 * row_out, ns * row_out, cudaMemcpyDeviceToHost,
                                 arr.copy));
        if (arr.idx_out_h)
            PKV_CUDA(cudaMemcpyAsync(arr.idx_out_h + s0 * p->K, idx + s0 * p->K, ns * p->K * 4,
                                     cudaMemcpyDeviceToHost, arr.copy));
        t0 = t1;
    }
    PKV_CUDA(cudaEventRecord(arr.ev_grp[pkv_pruner_s::kGroups], arr.copy));
    PKV_CUDA(cudaStreamWaitEvent(ps, arr.ev_grp[pkv_pruner_s::kGroups], 0));
}

pkv_pruner make_pruner(pkv_ctx ctx, pkv_mapper m, int64_t Hq, int64_t dp, int64_t dt, int64_t N, double rho,
                       uint32_t score_flags, uint32_t mode, int world, int rank, pkv_comm comm) {
    require_ctx(ctx);
    PKV_REQUIRE_VALUE(m != nullptr, "null pkv_mapper");
    Mapper& mp = *m->m;
    PKV_REQUIRE_VALUE(rho > 0.0 && rho <= 1.0, "retention ratio must be in (0, 1], got ", rho);
    PKV_REQUIRE_VALUE(N > 0 && dt > 0, "context length and target head_dim must be positive");
    ShardPlan plan = make_shard_plan(mp.geom, world, rank, mode);
    PKV_REQUIRE_VALUE(mode != PKV_SHARD_HEAD || comm != nullptr, "head-group sharding needs a pkv_comm");
    PKV_REQUIRE_VALUE(comm == nullptr || (comm->world == world && comm->rank == rank),
                      "pkv_comm (world ", comm ? comm->world : 0, ", rank ", comm ? comm->rank : 0,
                      ") does not match the shard (world ", world, ", rank ", rank, ")");
    ScoreShape sc{plan.p_hi - plan.p_lo, Hq, mp.geom.proxy_heads, N, N, dp, (score_flags & PKV_SCORE_CAUSAL) != 0};
    if (sc.L > 0) score_validate(sc);
    auto p = std::make_unique<pkv_pruner_s>();
    p->ctx = ctx;
    p->mapper = &mp;
    p->score = sc;
    p->reduce_max = (score_flags & PKV_SCORE_REDUCE_SUM) == 0;
    p->dt = dt;
    p->N = N;
    p->Hq = Hq;
    p->dp = dp;
    p->K = static_cast<int64_t>(std::ceil(rho * static_cast<double>(N)));  // pruning.cpp:17
    p->Ll = mp.geom.target_layers;
    p->Hl = mp.geom.target_heads;
    p->plan = std::move(plan);
    p->comm = comm;
    std::map<int64_t, int> unit_of;
    for (int64_t t = p->plan.a; t < p->plan.b; ++t) {
        const int64_t ls = layer_pair(t + 1, mp.geom) - 1;
        auto it = unit_of.find(ls);
        if (it == unit_of.end()) {
            it = unit_of.emplace(ls, static_cast<int>(p->unit_off.size())).first;
            p->unit_off.push_back((ls - p->plan.p_lo) * mp.geom.proxy_heads * N);
        }
        p->out_unit.push_back(it->second);
    }
    return p.release();
}

// score -> map (-> exchange) on `ps`; select -> compact on `ts` (gated by an
// event when the streams differ).
void run_pruner(pkv_pruner p, const void* q, const void* kp, const void* kt, const void* vt, void* k_out,
                void* v_out, int32_t* idx_out, float* scores_out, cudaStream_t ps, cudaStream_t ts,
                const HostArrival* arr = nullptr, const float* lse_in = nullptr) {
    const ScoreShape& s = p->score;
    const ShardPlan& pl = p->plan;
    const int64_t slices = p->slices();
    const int64_t n_map = pl.b - pl.a;
    float* y_sel = scores_out ? scores_out : static_cast<float*>(p->y.get(static_cast<size_t>(slices * p->N) * 4));
    float* y_map = pl.mode == PKV_SHARD_HEAD
                       ? static_cast<float*>(p->y_local.get(static_cast<size_t>(std::max<int64_t>(n_map, 1) * p->Hl * p->N) * 4))
                       : y_sel;
    int32_t* idx = idx_out ? idx_out : static_cast<int32_t*>(p->idx.get(static_cast<size_t>(slices * p->K) * 4));
    // profiled run (device-resident, single-stream form only): boundary events
    const bool prof = p->prof_next < p->prof_max && !arr && !lse_in && ps == ts && n_map > 0 && slices > 0 &&
                      pl.mode != PKV_SHARD_HEAD;
    if (prof) PKV_CUDA(cudaEventRecord(p->prof(0), ps));
    if (n_map > 0) {
        // (1) proxy scoring of this rank's proxy layers: X [L, H_s, N]
        const size_t q_off = static_cast<size_t>(pl.p_lo * p->Hq * p->N * p->dp) * 2;
        const size_t k_off = static_cast<size_t>(pl.p_lo * s.Hkv * p->N * p->dp) * 2;
        const auto* qp = static_cast<const uint8_t*>(q) + q_off;
        const auto* kpp = static_cast<const uint8_t*>(kp) + k_off;
        auto* lam = static_cast<__nv_bfloat16*>(p->lam.get(static_cast<size_t>(s.L * s.Hq * s.Nq) * 16));
        auto* x = static_cast<float*>(p->x.get(static_cast<size_t>(s.L * s.Hkv * s.Nk) * 4));
        {
        StageRange r_score("pkv.score");
        if (lse_in) {  // LSE from the proxy's prefill attention: the pooled pass only
            launch_lam_from_lse(lse_in + static_cast<size_t>(pl.p_lo * p->Hq * p->N), s.L * s.Hq * s.Nq, s.d, lam,
                                ps);
            launch_score_pool(s, qp, kpp, lam, p->reduce_max, x, ps);
            count_launch(p->ctx, 2);
        } else if (!arr) {
            launch_score_lse(s, qp, kpp, nullptr, lam, ps, &p->score_aux);
            if (prof) PKV_CUDA(cudaEventRecord(p->prof(1), ps));
            launch_score_pool(s, qp, kpp, lam, p->reduce_max, x, ps);
            if (prof) PKV_CUDA(cudaEventRecord(p->prof(2), ps));
            count_launch(p->ctx, 2);
        } else {  // proxy layers scored chunk by chunk as their H2D copies land
            for (int c = 0; c < arr->chunks; ++c) {
                const int64_t l0 = c * arr->chunk_layers, l1 = std::min<int64_t>(s.L, l0 + arr->chunk_layers);
                if (l0 >= l1) break;
                if (c == 0 && arr->sub > 1 && l1 - l0 == 1) {  // the first layer, per KV-head group
                    const int64_t g = s.Hq / s.Hkv, hk = s.Hkv / arr->sub;
                    for (int sg = 0; sg < arr->sub; ++sg) {
                        const int64_t k0 = sg * hk;
                        ScoreShape sc = s;
                        sc.L = 1;
                        sc.Hq = hk * g;
                        sc.Hkv = hk;
                        PKV_CUDA(cudaStreamWaitEvent(ps, arr->ev_sub[sg], 0));
                        const auto* qc = qp + static_cast<size_t>(k0 * g * p->N * p->dp) * 2;
                        const auto* kc = kpp + static_cast<size_t>(k0 * p->N * p->dp) * 2;
                        __nv_bfloat16* lc = lam + static_cast<size_t>(k0 * g * s.Nq) * 8;
                        launch_score_lse(sc, qc, kc, nullptr, lc, ps, &p->score_aux);
                        launch_score_pool(sc, qc, kc, lc, p->reduce_max, x + static_cast<size_t>(k0 * s.Nk), ps);
                        count_launch(p->ctx, 2);
                    }
                    continue;
                }
                ScoreShape sc = s;
                sc.L = l1 - l0;
                PKV_CUDA(cudaStreamWaitEvent(ps, arr->ev_chunk[c], 0));
                const auto* qc = qp + static_cast<size_t>(l0 * p->Hq * p->N * p->dp) * 2;
                const auto* kc = kpp + static_cast<size_t>(l0 * s.Hkv * p->N * p->dp) * 2;
                __nv_bfloat16* lc = lam + static_cast<size_t>(l0 * s.Hq * s.Nq) * 8;
                launch_score_lse(sc, qc, kc, nullptr, lc, ps, &p->score_aux);
                launch_score_pool(sc, qc, kc, lc, p->reduce_max, x + static_cast<size_t>(l0 * s.Hkv * s.Nk), ps);
                count_launch(p->ctx, 2);
            }
        }
        }  // pkv.score
        // (2)-(4) per target-layer group with the outputs leaving for the host
        if (arr && arr->k_out_h && pl.mode != PKV_SHARD_HEAD && ts == ps && slices > 0 &&
            n_map * p->Hl == slices) {
            grouped_tail(p, x, kt, vt, k_out, v_out, idx, y_sel, ps, *arr);
            return;
        }
        // (2) mapper: Ŷ for target layers [a, b), all heads
        StageRange r_map("pkv.map");
        p->mapper->run(x, p->unit_off, p->N, p->out_unit, y_map, ps);
        if (prof) PKV_CUDA(cudaEventRecord(p->prof(3), ps));
    }
    // (2b) head-group sharding: every mapped row to the owner of its head
    if (pl.mode == PKV_SHARD_HEAD) {
        StageRange r_x("pkv.exchange");
        exchange_scores(p->comm, pl, p->Hl, p->N, y_map, y_sel, ps);
    }
    if (ts != ps) {
        if (!p->ev) PKV_CUDA(cudaEventCreateWithFlags(&p->ev, cudaEventDisableTiming));
        PKV_CUDA(cudaEventRecord(p->ev, ps));
        PKV_CUDA(cudaStreamWaitEvent(ts, p->ev, 0));
    }
    if (slices == 0) return;
    if (arr) PKV_CUDA(cudaStreamWaitEvent(ts, arr->ev_kv, 0));
    // (3) Top-K per (target layer, head): ascending retained indices
    {
        StageRange r_sel("pkv.select");
        launch_topk_select(y_sel, slices, p->N, p->K, nullptr, idx, ts);
        if (prof) PKV_CUDA(cudaEventRecord(p->prof(4), ts));
    }
    // (4) packed KV gather
    StageRange r_cmp("pkv.compact");
    launch_compact_kv(kt, vt, idx, slices, p->N, p->K, p->dt * 2, k_out, v_out, p->ctx->sm_count, ts);
    count_launch(p->ctx, 2);
    if (prof) {
        PKV_CUDA(cudaEventRecord(p->prof(5), ts));
        ++p->prof_next;
    }
}

}  // namespace

extern "C" {

pkv_status pkv_pruner_create(pkv_ctx ctx, pkv_mapper m, int64_t Hq, int64_t dp, int64_t dt, int64_t N, double rho,
                             uint32_t score_flags, pkv_pruner* out) {
    return guard([&] { *out = make_pruner(ctx, m, Hq, dp, dt, N, rho, score_flags, PKV_SHARD_LAYER, 1, 0, nullptr); });
}

pkv_status pkv_pruner_create_sharded(pkv_ctx ctx, pkv_mapper m, int64_t Hq, int64_t dp, int64_t dt, int64_t N,
                                     double rho, uint32_t score_flags, uint32_t shard_mode, int world, int rank,
                                     pkv_comm comm, pkv_pruner* out) {
    return guard(
        [&] { *out = make_pruner(ctx, m, Hq, dp, dt, N, rho, score_flags, shard_mode, world, rank, comm); });
}

void pkv_pruner_destroy(pkv_pruner p) { delete p; }

int64_t pkv_pruner_k(pkv_pruner p) { return p ? p->K : 0; }

pkv_status pkv_pruner_run(pkv_pruner p, const void* q, const void* kp, const void* kt, const void* vt, void* k_out,
                          void* v_out, int32_t* idx_out, float* scores_out, void* stream) {
    return guard([&] {
        PKV_REQUIRE_VALUE(p != nullptr, "null pkv_pruner");
        auto st = static_cast<cudaStream_t>(stream);
        run_pruner(p, q, kp, kt, vt, k_out, v_out, idx_out, scores_out, st, st);
    });
}

pkv_status pkv_pruner_profile(pkv_pruner p, int64_t runs) {
    return guard([&] {
        PKV_REQUIRE_VALUE(p && runs >= 0, "pkv_pruner_profile: runs must be >= 0");
        const size_t need = static_cast<size_t>(runs * pkv_pruner_s::kProfEv);
        while (p->prof_ev.size() < need) {
            cudaEvent_t e = nullptr;
            PKV_CUDA(cudaEventCreate(&e));
            p->prof_ev.push_back(e);
        }
        p->prof_max = runs;
        p->prof_next = 0;
    });
}

pkv_status pkv_pruner_profile_read(pkv_pruner p, double* ms_out, int64_t cap_runs, int64_t* runs_out) {
    return guard([&] {
        PKV_REQUIRE_VALUE(p, "null pruner");
        const int64_t n = std::min(p->prof_next, cap_runs);
        for (int64_t r = 0; r < n; ++r) {
            const size_t b = static_cast<size_t>(r * pkv_pruner_s::kProfEv);
            PKV_CUDA(cudaEventSynchronize(p->prof_ev[b + pkv_pruner_s::kProfEv - 1]));
            for (int i = 0; i + 1 < pkv_pruner_s::kProfEv; ++i) {
                float ms = 0.0f;
                PKV_CUDA(cudaEventElapsedTime(&ms, p->prof_ev[b + i], p->prof_ev[b + i + 1]));
                ms_out[r * (pkv_pruner_s::kProfEv - 1) + i] = ms;
            }
        }
        *runs_out = n;
    });
}

pkv_status pkv_pruner_exchange(pkv_pruner p, const float* y_local_dev, float* y_recv_dev, void* stream) {
    return guard([&] {
        PKV_REQUIRE_VALUE(p != nullptr, "null pkv_pruner");
        PKV_REQUIRE_VALUE(p->plan.mode == PKV_SHARD_HEAD && p->comm != nullptr,
                          "pkv_pruner_exchange needs a head-group sharded pruner");
        exchange_scores(p->comm, p->plan, p->Hl, p->N, y_local_dev, y_recv_dev, static_cast<cudaStream_t>(stream));
    });
}

pkv_status pkv_pruner_run_lse(pkv_pruner p, const void* q, const void* kp, const float* lse, const void* kt,
                              const void* vt, void* k_out, void* v_out, int32_t* idx_out, float* scores_out,
                              void* stream) {
    return guard([&] {
        PKV_REQUIRE_VALUE(p != nullptr, "null pkv_pruner");
        PKV_REQUIRE_VALUE(lse != nullptr, "pkv_pruner_run_lse needs the proxy prefill's LSE");
        auto st = static_cast<cudaStream_t>(stream);
        run_pruner(p, q, kp, kt, vt, k_out, v_out, idx_out, scores_out, st, st, nullptr, lse);
    });
}

pkv_status pkv_pruner_run_dual(pkv_pruner p, const void* q, const void* kp, const void* kt, const void* vt,
                               void* k_out, void* v_out, int32_t* idx_out, float* scores_out, void* proxy_stream,
                               void* target_stream) {
    return guard([&] {
        PKV_REQUIRE_VALUE(p != nullptr, "null pkv_pruner");
        run_pruner(p, q, kp, kt, vt, k_out, v_out, idx_out, scores_out, static_cast<cudaStream_t>(proxy_stream),
                   static_cast<cudaStream_t>(target_stream));
    });
}

// Paper regime: the proxy device scores
// and maps; Ŷ crosses to the target device with one peer copy on the proxy
// stream, and the target stream (on the target device) waits for it before
// select + compaction. Outputs are identical to pkv_pruner_run.
pkv_status pkv_pruner_run_two_device(pkv_pruner p, pkv_ctx target_ctx, const void* q_dev, const void* kp_dev,
                                     const void* kt_target_dev, const void* vt_target_dev, void* k_out_target_dev,
                                     void* v_out_target_dev, int32_t* idx_out_target_dev, float* scores_target_dev,
                                     void* proxy_stream, void* target_stream) {
    return guard([&] {
        PKV_REQUIRE_VALUE(p != nullptr, "null pkv_pruner");
        require_ctx(target_ctx);
        PKV_REQUIRE_VALUE(p->plan.world == 1, "two-device mode runs one whole context (world 1)");
        auto ps = static_cast<cudaStream_t>(proxy_stream);
        auto ts = static_cast<cudaStream_t>(target_stream);
        const int dev_p = p->ctx->device, dev_t = target_ctx->device;
        const int64_t slices = p->slices();
        const size_t ybytes = static_cast<size_t>(slices * p->N) * 4;
        PKV_CUDA(cudaSetDevice(dev_p));
        // score -> map on the proxy device into p->y (no select: slices handled below)
        float* y_p = static_cast<float*>(p->y.get(ybytes));
        {
            const ScoreShape& s = p->score;
            auto* lam = static_cast<__nv_bfloat16*>(p->lam.get(static_cast<size_t>(s.L * s.Hq * s.Nq) * 16));
            auto* x = static_cast<float*>(p->x.get(static_cast<size_t>(s.L * s.Hkv * s.Nk) * 4));
            launch_score_lse(s, q_dev, kp_dev, nullptr, lam, ps, &p->score_aux);
            launch_score_pool(s, q_dev, kp_dev, lam, p->reduce_max, x, ps);
            count_launch(p->ctx, 2);
            p->mapper->run(x, p->unit_off, p->N, p->out_unit, y_p, ps);
        }
        // Ŷ -> target device
        PKV_CUDA(cudaSetDevice(dev_t));
        float* y_t = scores_target_dev ? scores_target_dev : static_cast<float*>(p->y_remote.get(ybytes));
        PKV_CUDA(cudaSetDevice(dev_p));
        PKV_CUDA(cudaMemcpyPeerAsync(y_t, dev_t, y_p, dev_p, ybytes, ps));
        if (!p->ev_remote) PKV_CUDA(cudaEventCreateWithFlags(&p->ev_remote, cudaEventDisableTiming));
        PKV_CUDA(cudaEventRecord(p->ev_remote, ps));
        // select + compaction on the target device
        PKV_CUDA(cudaSetDevice(dev_t));
        PKV_CUDA(cudaStreamWaitEvent(ts, p->ev_remote, 0));
        int32_t* idx = idx_out_target_dev ? idx_out_target_dev
                                          : static_cast<int32_t*>(target_ctx->scratch_select.get(
                                                static_cast<size_t>(slices * p->K) * 4));
        launch_topk_select(y_t, slices, p->N, p->K, nullptr, idx, ts);
        launch_compact_kv(kt_target_dev, vt_target_dev, idx, slices, p->N, p->K, p->dt * 2, k_out_target_dev,
                          v_out_target_dev, target_ctx->sm_count, ts);
        count_launch(target_ctx, 2);
        PKV_CUDA(cudaSetDevice(dev_p));
    });
}

pkv_status pkv_pruner_run_host(pkv_pruner p, const void* q_h, const void* kp_h, const void* kt_h, const void* vt_h,
                               void* k_out_h, void* v_out_h, int32_t* idx_out_h, void* stream) {
    return guard([&] {
        PKV_REQUIRE_VALUE(p != nullptr, "null pkv_pruner");
        auto st = static_cast<cudaStream_t>(stream);
        const ShardPlan& pl = p->plan;
        const int64_t Ls = p->mapper->geom.proxy_layers, Hs = p->mapper->geom.proxy_heads;
        const size_t q_layer = static_cast<size_t>(p->Hq * p->N * p->dp) * 2;
        const size_t kp_layer = static_cast<size_t>(Hs * p->N * p->dp) * 2;
        const size_t qb = Ls * q_layer, kpb = Ls * kp_layer;
        const size_t kvb = static_cast<size_t>(p->slices() * p->N * p->dt) * 2;
        const size_t ob = static_cast<size_t>(p->slices() * p->K * p->dt) * 2;
        const size_t ib = static_cast<size_t>(p->slices() * p->K) * 4;
        auto* in = static_cast<uint8_t*>(p->host_in.get(qb + kpb + 2 * kvb));
        auto* outb = static_cast<uint8_t*>(p->host_out.get(2 * ob + ib));
        if (!p->copy_st) {
            PKV_CUDA(cudaStreamCreateWithFlags(&p->copy_st, cudaStreamNonBlocking));
            for (cudaEvent_t& e : p->ev_in) PKV_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            for (cudaEvent_t& e : p->ev_grp) PKV_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            for (cudaEvent_t& e : p->ev_sub) PKV_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        }
        cudaStream_t cs = p->copy_st;
        constexpr int kC = pkv_pruner_s::kChunks;
        // the copies may overwrite the input buffers only after earlier work on `st`
        PKV_CUDA(cudaEventRecord(p->ev_in[kC + 1], st));
        PKV_CUDA(cudaStreamWaitEvent(cs, p->ev_in[kC + 1], 0));
        // H2D overlapped with compute: the proxy layers this pruner scores, in
        // kC chunks (scoring of chunk c starts when it lands), then the target
        // KV (needed only by select + compaction, after the mapper)
        HostArrival arr;
        const int64_t nl = pl.b > pl.a ? pl.p_hi - pl.p_lo : 0;
        arr.chunk_layers = std::max<int64_t>(1, (nl + kC - 1) / kC);
        arr.chunks = kC;
        arr.ev_chunk = p->ev_in;
        constexpr int kS = pkv_pruner_s::kSub;
        if (arr.chunk_layers == 1 && nl > 0 && Hs % kS == 0) {
            arr.sub = kS;
            arr.ev_sub = p->ev_sub;
        }
        for (int c = 0; c < kC; ++c) {
            const int64_t l0 = pl.p_lo + c * arr.chunk_layers;
            const int64_t l1 = std::min<int64_t>(pl.p_lo + nl, l0 + arr.chunk_layers);
            if (c == 0 && arr.sub > 1 && l0 < l1) {  // first layer per KV-head group (Q heads of the group + its K head)
                const size_t qg = q_layer / kS, kg = kp_layer / kS;
                for (int sg = 0; sg < kS; ++sg) {
                    PKV_CUDA(cudaMemcpyAsync(in + l0 * q_layer + sg * qg,
                                             static_cast<const uint8_t*>(q_h) + l0 * q_layer + sg * qg, qg,
                                             cudaMemcpyHostToDevice, cs));
                    PKV_CUDA(cudaMemcpyAsync(in + qb + l0 * kp_layer + sg * kg,
                                             static_cast<const uint8_t*>(kp_h) + l0 * kp_layer + sg * kg, kg,
                                             cudaMemcpyHostToDevice, cs));
                    PKV_CUDA(cudaEventRecord(p->ev_sub[sg], cs));
                }
            } else if (l0 < l1) {
                PKV_CUDA(cudaMemcpyAsync(in + l0 * q_layer, static_cast<const uint8_t*>(q_h) + l0 * q_layer,
                                         (l1 - l0) * q_layer, cudaMemcpyHostToDevice, cs));
                PKV_CUDA(cudaMemcpyAsync(in + qb + l0 * kp_layer, static_cast<const uint8_t*>(kp_h) + l0 * kp_layer,
                                         (l1 - l0) * kp_layer, cudaMemcpyHostToDevice, cs));
            }
            PKV_CUDA(cudaEventRecord(p->ev_in[c], cs));
        }
        PKV_CUDA(cudaMemcpyAsync(in + qb + kpb, kt_h, kvb, cudaMemcpyHostToDevice, cs));
        PKV_CUDA(cudaMemcpyAsync(in + qb + kpb + kvb, vt_h, kvb, cudaMemcpyHostToDevice, cs));
        PKV_CUDA(cudaEventRecord(p->ev_in[kC], cs));
        arr.ev_kv = p->ev_in[kC];
        // layer mode: the outputs leave per target-layer group (grouped_tail)
        const bool grouped = pl.mode != PKV_SHARD_HEAD && pl.b > pl.a && p->slices() > 0 &&
                             (pl.b - pl.a) * p->Hl == p->slices();
        if (grouped) {
            arr.k_out_h = k_out_h;
            arr.v_out_h = v_out_h;
            arr.idx_out_h = idx_out_h;
            arr.copy = cs;
            arr.ev_grp = p->ev_grp;
        }
        run_pruner(p, in, in + qb, in + qb + kpb, in + qb + kpb + kvb, outb, outb + ob,
                   reinterpret_cast<int32_t*>(outb + 2 * ob), nullptr, st, st, &arr);
        if (!grouped) {
            PKV_CUDA(cudaMemcpyAsync(k_out_h, outb, ob, cudaMemcpyDeviceToHost, st));
            PKV_CUDA(cudaMemcpyAsync(v_out_h, outb + ob, ob, cudaMemcpyDeviceToHost, st));
            if (idx_out_h) PKV_CUDA(cudaMemcpyAsync(idx_out_h, outb + 2 * ob, ib, cudaMemcpyDeviceToHost, st));
        }
        PKV_CUDA(cudaStreamSynchronize(st));
    });
}

}  // extern "C"
