// shard.cpp — multi-GPU partition of the pruning path and the
// NCCL plumbing for its one exchange step.
//
// Two plans, both with bit-identical per-slice results to the 1-GPU path
// (same per-unit kernels, no cross-unit reductions):
//  - PKV_SHARD_LAYER (BASELINE configs[2], "layer-sharded"): rank r owns a
//    contiguous block of target layers with all their KV heads. layer_pair is
//    monotone (reference test_mapper.cpp:53-60), so the block needs a
//    contiguous range of proxy layers, which the rank scores and maps itself
//    (boundary proxy layers are computed by both neighbours): no collective.
//  - PKV_SHARD_HEAD (configs[3], "head-group sharded", the tensor-parallel
//    target): rank r owns a contiguous group of target KV heads across all
//    layers. The proxy work is split by unique paired proxy layer; each rank
//    maps its proxy layers for all heads, then one NCCL all-to-all (grouped
//    send/recv, one message per (target layer, peer)) moves every mapped-score
//    row to the owner of its head — the "scores broadcast over NVLink" step.
#include "shard.h"

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <set>

namespace pkv {

namespace {

inline int64_t blk(int64_t i, int64_t n, int64_t w) { return i * n / w; }

// libnccl.so.2 resolved at first use (torch's bundled copy when it is already
// loaded in the process, else the system one).
struct Nccl {
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) comm_init_rank = nullptr;
    decltype(&ncclCommDestroy) comm_destroy = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclGroupStart) group_start = nullptr;
    decltype(&ncclGroupEnd) group_end = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
};

const Nccl& nccl() {
    static Nccl n;
    static std::string err;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            err = dlerror() ? dlerror() : "dlopen failed";
            return;
        }
        n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        n.comm_init_rank = reinterpret_cast<decltype(n.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        n.send = reinterpret_cast<decltype(n.send)>(dlsym(h, "ncclSend"));
        n.recv = reinterpret_cast<decltype(n.recv)>(dlsym(h, "ncclRecv"));
        n.group_start = reinterpret_cast<decltype(n.group_start)>(dlsym(h, "ncclGroupStart"));
        n.group_end = reinterpret_cast<decltype(n.group_end)>(dlsym(h, "ncclGroupEnd"));
        n.error_string = reinterpret_cast<decltype(n.error_string)>(dlsym(h, "ncclGetErrorString"));
    });
    PKV_REQUIRE(n.send && n.recv && n.comm_init_rank && n.get_unique_id, PKV_ENCCL, "NCCL unavailable: ", err);
    return n;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) {
        const char* s = nccl().error_string ? nccl().error_string(r) : "?";
        throw Error{PKV_ENCCL, cat(what, " failed: ", s)};
    }
}

}  // namespace

ShardPlan make_shard_plan(const Geometry& g, int world, int rank, uint32_t mode) {
    g.validate();
    PKV_REQUIRE_VALUE(world >= 1 && rank >= 0 && rank < world, "rank ", rank, " out of range for world ", world);
    PKV_REQUIRE(mode == PKV_SHARD_LAYER || mode == PKV_SHARD_HEAD, PKV_ECONFIG, "unknown shard mode ", mode);
    ShardPlan p;
    p.mode = mode;
    p.world = world;
    p.rank = rank;
    const int64_t Ll = g.target_layers, Hl = g.target_heads;
    if (mode == PKV_SHARD_LAYER) {
        PKV_REQUIRE(world <= Ll, PKV_ECONFIG, "layer sharding needs world <= target layers (", Ll, "), got ", world);
        p.t_lo = blk(rank, Ll, world);
        p.t_hi = blk(rank + 1, Ll, world);
        p.h_lo = 0;
        p.h_hi = Hl;
        p.a = p.t_lo;
        p.b = p.t_hi;
        p.p_lo = layer_pair(p.t_lo + 1, g) - 1;  // monotone pairing: a contiguous proxy block
        p.p_hi = layer_pair(p.t_hi, g);
        return p;
    }
    PKV_REQUIRE(world <= Hl, PKV_ECONFIG, "head-group sharding needs world <= target KV heads (", Hl, "), got ", world);
    for (int r = 0; r <= world; ++r) p.h_begin.push_back(blk(r, Hl, world));
    p.h_lo = p.h_begin[rank];
    p.h_hi = p.h_begin[rank + 1];
    p.t_lo = 0;
    p.t_hi = Ll;
    // unique paired proxy layers (ascending), split into contiguous blocks
    std::vector<int64_t> pair(Ll);
    std::set<int64_t> uniq;
    for (int64_t t = 0; t < Ll; ++t) uniq.insert(pair[t] = layer_pair(t + 1, g) - 1);
    const std::vector<int64_t> U(uniq.begin(), uniq.end());
    const int64_t nu = static_cast<int64_t>(U.size());
    auto owner = [&](int64_t ls) {
        for (int r = 0; r < world; ++r) {
            const int64_t lo = blk(r, nu, world), hi = blk(r + 1, nu, world);
            if (lo < hi && ls >= U[lo] && ls <= U[hi - 1]) return r;
        }
        return -1;
    };
    p.producer.resize(Ll);
    for (int64_t t = 0; t < Ll; ++t) p.producer[t] = owner(pair[t]);
    const int64_t ulo = blk(rank, nu, world), uhi = blk(rank + 1, nu, world);
    if (ulo < uhi) {
        p.p_lo = U[ulo];
        p.p_hi = U[uhi - 1] + 1;
        p.a = Ll;
        p.b = 0;
        for (int64_t t = 0; t < Ll; ++t) {
            if (p.producer[t] == rank) {
                p.a = std::min(p.a, t);
                p.b = std::max(p.b, t + 1);
            }
        }
    }
    return p;
}

std::vector<XOp> exchange_schedule(const ShardPlan& plan, int64_t Hl, int64_t N) {
    std::vector<XOp> ops;
    if (plan.mode != PKV_SHARD_HEAD) return ops;
    const int64_t nh = plan.h_hi - plan.h_lo;
    for (int64_t t = plan.a; t < plan.b; ++t) {
        for (int g = 0; g < plan.world; ++g) {
            const int64_t hg = plan.h_begin[g], ng = plan.h_begin[g + 1] - hg;
            if (ng == 0) continue;
            ops.push_back({0, g, ((t - plan.a) * Hl + hg) * N, ng * N, t});
        }
    }
    if (nh > 0) {
        for (int64_t t = 0; t < static_cast<int64_t>(plan.producer.size()); ++t)
            ops.push_back({1, plan.producer[t], t * nh * N, nh * N, t});
    }
    return ops;
}

void exchange_scores(pkv_comm comm, const ShardPlan& plan, int64_t Hl, int64_t N, const float* y_local,
                     float* y_recv, cudaStream_t st) {
    const Nccl& n = nccl();
    auto c = static_cast<ncclComm_t>(comm->nccl);
    nccl_check(n.group_start(), "ncclGroupStart");
    for (const XOp& op : exchange_schedule(plan, Hl, N)) {
        if (op.kind == 0)
            nccl_check(n.send(y_local + op.off, static_cast<size_t>(op.count), ncclFloat, op.peer, c, st), "ncclSend");
        else
            nccl_check(n.recv(y_recv + op.off, static_cast<size_t>(op.count), ncclFloat, op.peer, c, st), "ncclRecv");
    }
    nccl_check(n.group_end(), "ncclGroupEnd");
}

}  // namespace pkv

using namespace pkv;

extern "C" {

pkv_status pkv_shard_plan(const int64_t* geom5, int world, int rank, uint32_t mode, int64_t* out8) {
    return guard([&] {
        const ShardPlan p = make_shard_plan(Geometry::from5(geom5), world, rank, mode);
        const int64_t v[8] = {p.t_lo, p.t_hi, p.h_lo, p.h_hi, p.p_lo, p.p_hi, p.a, p.b};
        for (int i = 0; i < 8; ++i) out8[i] = v[i];
    });
}

pkv_status pkv_shard_exchange_schedule(const int64_t* geom5, int world, int rank, int64_t N, int64_t* ops_out,
                                       int64_t cap, int64_t* count_out) {
    return guard([&] {
        PKV_REQUIRE_VALUE(N > 0, "context length must be positive");
        const Geometry g = Geometry::from5(geom5);
        const auto ops = exchange_schedule(make_shard_plan(g, world, rank, PKV_SHARD_HEAD), g.target_heads, N);
        *count_out = static_cast<int64_t>(ops.size());
        for (int64_t i = 0; i < cap && i < *count_out; ++i) {
            const XOp& o = ops[i];
            const int64_t v[5] = {o.kind, o.peer, o.off, o.count, o.tag};
            for (int j = 0; j < 5; ++j) ops_out[i * 5 + j] = v[j];
        }
    });
}

pkv_status pkv_comm_unique_id(uint8_t* id_out) {
    return guard([&] {
        ncclUniqueId id;
        nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
        static_assert(sizeof(id) == PKV_COMM_ID_BYTES, "ncclUniqueId size");
        std::memcpy(id_out, &id, sizeof(id));
    });
}

pkv_status pkv_comm_create(pkv_ctx ctx, int world, int rank, const uint8_t* id, pkv_comm* out) {
    return guard([&] {
        require_ctx(ctx);
        PKV_REQUIRE_VALUE(world >= 1 && rank >= 0 && rank < world, "rank ", rank, " out of range for world ", world);
        PKV_CUDA(cudaSetDevice(ctx->device));
        ncclUniqueId uid;
        std::memcpy(&uid, id, sizeof(uid));
        ncclComm_t c = nullptr;
        nccl_check(nccl().comm_init_rank(&c, world, uid, rank), "ncclCommInitRank");
        auto* h = new pkv_comm_s();
        h->nccl = c;
        h->world = world;
        h->rank = rank;
        *out = h;
    });
}

void pkv_comm_destroy(pkv_comm c) {
    if (!c) return;
    if (c->nccl && nccl().comm_destroy) nccl().comm_destroy(static_cast<ncclComm_t>(c->nccl));
    delete c;
}

}  // extern "C"
