"""Multi-GPU partition of one context (shard.cpp), on CPU.

* pkv_shard_plan (host logic of libpkv_b200.so, no device needed) covers every
  (target layer, head) slice exactly once, every rank scores/maps the proxy
  layers its produced target layers pair with (layer_pair, mapper.cpp:44-49),
  and the produced target layers partition [0, L_l) — at the BASELINE configs'
  geometries and world sizes 1..8.
* A world_size-2 gloo run of the head-group plan's exchange (the same
  per-(target layer, peer) messages pkv_pruner sends with NCCL; self messages
  are local copies) delivers each rank exactly its head group's rows, and the
  select the ranks then run (the oracle's topk_select) reproduces the 1-rank
  selection bit for bit. Layer sharding needs no exchange: the same check on
  its per-rank slices.
Mapped scores are synthetic (a deterministic function of target layer, head
and token) — the exchange and the partition are what is under test."""
import os
import socket

import numpy as np
import pytest

from oracle import pkv_oracle as O

GEOMS = {  # (L_l, H_l, L_s, H_s, d_t): BASELINE configs
    "tiny": (4, 8, 2, 4, 64),
    "llama": (32, 8, 16, 8, 128),
    "qwen25": (28, 4, 24, 2, 128),
    "qwen3": (64, 8, 28, 8, 128),
}


def _geom(name):
    import paper_2605_16360_b200 as P
    return P.ModelGeometry(*GEOMS[name])


def _pair(t, g):  # 0-based target layer -> 0-based proxy layer (mapper.cpp:44-49)
    return (t + 1) * g.proxy_layers // g.target_layers + (1 if ((t + 1) * g.proxy_layers) % g.target_layers else 0) - 1


@pytest.mark.parametrize("name", sorted(GEOMS))
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_layer_plan_partitions_slices(name, world):
    import paper_2605_16360_b200 as P
    g = _geom(name)
    if world > g.target_layers:
        with pytest.raises(P.ConfigError):
            P.shard_plan(g, world, 0, P.SHARD_LAYER)
        return
    owned = np.zeros((g.target_layers, g.target_heads), int)
    for r in range(world):
        p = P.shard_plan(g, world, r, P.SHARD_LAYER)
        assert (p.h_lo, p.h_hi) == (0, g.target_heads) and (p.a, p.b) == (p.t_lo, p.t_hi)
        owned[p.t_lo:p.t_hi] += 1
        for t in range(p.t_lo, p.t_hi):
            assert P.layer_pair(t + 1, g) - 1 == _pair(t, g)
            assert p.p_lo <= _pair(t, g) < p.p_hi
        assert p.p_hi - p.p_lo <= (g.proxy_layers + world - 1) // world + 1  # at most one shared boundary layer
    assert (owned == 1).all()


@pytest.mark.parametrize("name", sorted(GEOMS))
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_head_plan_partitions_heads_and_producers(name, world):
    import paper_2605_16360_b200 as P
    g = _geom(name)
    if world > g.target_heads:
        with pytest.raises(P.ConfigError):
            P.shard_plan(g, world, 0, P.SHARD_HEAD)
        return
    heads = np.zeros(g.target_heads, int)
    produced = np.zeros(g.target_layers, int)
    proxy = np.zeros(g.proxy_layers, int)
    for r in range(world):
        p = P.shard_plan(g, world, r, P.SHARD_HEAD)
        assert (p.t_lo, p.t_hi) == (0, g.target_layers)
        heads[p.h_lo:p.h_hi] += 1
        produced[p.a:p.b] += 1
        proxy[p.p_lo:p.p_hi] += 1
        for t in range(p.a, p.b):
            assert p.p_lo <= _pair(t, g) < p.p_hi
    assert (heads == 1).all() and (produced == 1).all()
    assert (proxy <= 1).all()  # proxy work is split, never duplicated


def test_plan_rejects_bad_rank():
    import paper_2605_16360_b200 as P
    with pytest.raises(P.PkvValueError):
        P.shard_plan(_geom("llama"), 2, 2, P.SHARD_LAYER)
    with pytest.raises(P.ConfigError):
        P.shard_plan(_geom("llama"), 2, 0, 7)


# ---------------------------------------------------------------- gloo run --
def _yhat(t, g, N):
    """Synthetic mapped scores of target layer t, all heads: ties included."""
    r = np.random.RandomState(1000 + t)
    return (np.floor(r.rand(g.target_heads, N) * 64) / 64).astype(np.float32)


def _worker(rank, world, port, name, N, rho, mode, q):
    import torch
    import torch.distributed as dist
    import paper_2605_16360_b200 as P
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        g = _geom(name)
        plans = [P.shard_plan(g, world, r, mode) for r in range(world)]
        p = plans[rank]
        k = O.retention_count(rho, N)
        # this rank's mapper output: target layers [a, b), all heads
        y_local = {t: _yhat(t, g, N) for t in range(p.a, p.b)}
        if mode == P.SHARD_HEAD:
            # the library's own exchange schedule (pkv_shard_exchange_schedule:
            # the ops the NCCL exchange issues), executed over gloo
            nh = p.h_hi - p.h_lo
            y_sel = np.zeros((g.target_layers, nh, N), np.float32)
            flat_local = (np.concatenate([y_local[t] for t in range(p.a, p.b)]).reshape(-1)
                          if p.b > p.a else np.zeros(0, np.float32))
            flat_sel = y_sel.reshape(-1)
            ops = P.shard_exchange_schedule(g, world, rank, N)
            reqs, bufs, self_sends = [], [], {}
            for kind, peer, off, cnt, tag in ops.tolist():
                if kind == 0:
                    rows = flat_local[off:off + cnt]
                    if peer == rank:
                        self_sends[tag] = rows
                    else:
                        reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(rows)), peer, tag=tag))
                else:
                    if peer == rank:
                        flat_sel[off:off + cnt] = self_sends.pop(tag)
                    else:
                        b = torch.empty(cnt)
                        reqs.append(dist.irecv(b, peer, tag=tag))
                        bufs.append((off, cnt, b))
            assert not self_sends
            for r_ in reqs:
                r_.wait()
            for off, cnt, b in bufs:
                flat_sel[off:off + cnt] = b.numpy()
            slices = y_sel.reshape(-1, N)
        else:
            slices = np.concatenate([y_local[t] for t in range(p.t_lo, p.t_hi)]).reshape(-1, N)
        _, idx = O.topk_select(slices, k)
        q.put((rank, p, idx))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("mode_name,name,world", [("head", "tiny", 2), ("layer", "tiny", 2), ("head", "llama", 2),
                                                 ("layer", "llama", 2), ("head", "qwen3", 4), ("head", "qwen25", 3)])
def test_gloo_sharded_select_matches_single_rank(mode_name, name, world):
    import torch.multiprocessing as mp
    import paper_2605_16360_b200 as P
    mode = P.SHARD_HEAD if mode_name == "head" else P.SHARD_LAYER
    N, rho = 512, 0.2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, N, rho, mode, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = {}
    for _ in range(world):
        rank, plan, idx = q.get(timeout=120)
        res[rank] = (plan, idx)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    g = _geom(name)
    k = O.retention_count(rho, N)
    full = np.stack([_yhat(t, g, N) for t in range(g.target_layers)])  # [L_l, H_l, N]
    _, ref = O.topk_select(full.reshape(-1, N), k)
    ref = ref.reshape(g.target_layers, g.target_heads, k)
    for rank, (plan, idx) in res.items():
        got = idx.reshape(plan.t_hi - plan.t_lo, plan.h_hi - plan.h_lo, k)
        np.testing.assert_array_equal(got, ref[plan.t_lo:plan.t_hi, plan.h_lo:plan.h_hi])


@pytest.mark.parametrize("name", sorted(GEOMS))
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_exchange_schedule_matches_across_ranks(name, world):
    """pkv_shard_exchange_schedule over all ranks: every recv has exactly one
    send with the same (peer pair, tag, count); the recvs of a rank tile its
    y_recv [L_l, nh, N] exactly once; each send reads inside y_local."""
    import paper_2605_16360_b200 as P
    g = _geom(name)
    if world > g.target_heads:
        return
    N = 100
    plans = [P.shard_plan(g, world, r, P.SHARD_HEAD) for r in range(world)]
    ops = [P.shard_exchange_schedule(g, world, r, N) for r in range(world)]
    sends = {}
    for r in range(world):
        p = plans[r]
        cover = np.zeros(g.target_layers * (p.h_hi - p.h_lo) * N, int)
        for kind, peer, off, cnt, tag in ops[r].tolist():
            if kind == 0:
                assert p.a <= tag < p.b and 0 <= off and off + cnt <= (p.b - p.a) * g.target_heads * N
                key = (r, peer, tag)
                assert key not in sends
                sends[key] = cnt
            else:
                cover[off:off + cnt] += 1
        assert (cover == 1).all()
    n_recv = 0
    for r in range(world):
        for kind, peer, off, cnt, tag in ops[r].tolist():
            if kind == 1:
                assert sends.pop((peer, r, tag)) == cnt
                n_recv += 1
    assert not sends and n_recv == g.target_layers * sum(1 for p in plans if p.h_hi > p.h_lo)
