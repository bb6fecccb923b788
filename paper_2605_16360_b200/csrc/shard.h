// shard.h — one context pruned by G ranks: the sharding plan
// (host logic) and the NCCL communicator (libnccl loaded at run time, so the
// single-GPU library has no NCCL dependency).
#pragma once

#include <cstdint>
#include <vector>

#include "internal.h"
#include "mapper.h"

struct pkv_comm_s {
    void* nccl = nullptr;  // ncclComm_t
    int world = 1, rank = 0;
};

namespace pkv {

// What rank `rank` of `world` owns for one context (all ranges 0-based, half-open).
struct ShardPlan {
    uint32_t mode = PKV_SHARD_LAYER;
    int world = 1, rank = 0;
    int64_t t_lo = 0, t_hi = 0;  // target layers whose slices this rank selects + compacts
    int64_t h_lo = 0, h_hi = 0;  // target KV heads of those slices
    int64_t p_lo = 0, p_hi = 0;  // proxy layers this rank scores and maps
    int64_t a = 0, b = 0;        // target layers whose mapped scores this rank produces (all heads)
    std::vector<int> producer;   // [L_l] rank producing each target layer (head mode)
    std::vector<int64_t> h_begin;  // [world + 1] head group boundaries (head mode)
};

ShardPlan make_shard_plan(const Geometry& g, int world, int rank, uint32_t mode);

// One point-to-point operation of the head-group exchange.
struct XOp {
    int kind;      // 0 send (from y_local), 1 recv (into y_recv)
    int peer;
    int64_t off;   // element offset into y_local / y_recv
    int64_t count; // elements
    int64_t tag;   // target layer
};
// The exchange as ops, in issue order (sends, then recvs).
std::vector<XOp> exchange_schedule(const ShardPlan& plan, int64_t Hl, int64_t N);

// NCCL point-to-point exchange of mapped scores (head mode): rank r sends
// y_local[t - a, heads of g, :] to every g for its produced layers t, and
// receives y_recv[t, :, :] (its own head group) from producer(t) for all t.
void exchange_scores(pkv_comm comm, const ShardPlan& plan, int64_t Hl, int64_t N, const float* y_local,
                     float* y_recv, cudaStream_t st);

}  // namespace pkv
