"""Sharded pruning on the GPU (shard.cpp): per-rank results are
bit-identical to the 1-GPU pruner's slices of the same context.

This run has one GPU, so:
  * layer sharding (no collective) runs every rank of world 2 / 4 one after
    the other on cuda:0, each with its own KV shard;
  * head-group sharding runs world 1 through a real NCCL communicator (the
    grouped send/recv exchange, to self); its world>1 message pattern is
    covered by tests/test_shard.py on gloo;
  * the dual-stream form (proxy stream -> event -> target stream) matches the
    single-stream run."""
import numpy as np
import pytest

from oracle import pkv_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def setup(gpu):
    import torch
    import paper_2605_16360_b200 as P
    Ls, Hq, Hs, dp, Ll, Hl, dt, N, rho = 2, 4, 4, 64, 4, 8, 64, 2048, 0.2
    geom = P.ModelGeometry(Ll, Hl, Ls, Hs, dt)
    m = P.Mapper(geom, P.MapperConfig(), seed=7, precision=3, ctx=gpu)
    r = np.random.RandomState(3)
    q = r.standard_normal((Ls, Hq, N, dp)).astype(np.float32) * 0.35
    kp = r.standard_normal((Ls, Hs, N, dp)).astype(np.float32)
    dev = lambda a: torch.from_numpy(a.view(np.int16)).cuda().view(torch.bfloat16)
    qd, kpd = dev(O.f32_to_bf16_bits(q)), dev(O.f32_to_bf16_bits(kp))
    kt = dev(r.randint(0, 1 << 15, (Ll, Hl, N, dt)).astype(np.uint16))
    vt = dev(r.randint(0, 1 << 15, (Ll, Hl, N, dt)).astype(np.uint16))
    full = P.Pruner(m, Hq, dp, dt, N, rho)
    K = full.k
    ref = dict(ko=torch.empty(Ll, Hl, K, dt, dtype=torch.bfloat16, device="cuda"),
               idx=torch.empty(Ll, Hl, K, dtype=torch.int32, device="cuda"),
               y=torch.empty(Ll, Hl, N, device="cuda"))
    ref["vo"] = torch.empty_like(ref["ko"])
    full.run(qd, kpd, kt, vt, ref["ko"], ref["vo"], ref["idx"], ref["y"])
    torch.cuda.synchronize()
    return dict(P=P, m=m, q=qd, kp=kpd, kt=kt, vt=vt, ref=ref, dims=(Ls, Hq, Hs, dp, Ll, Hl, dt, N, rho), K=K)


def _run_shard(s, pr, stream_pair=None):
    import torch
    p = pr.plan
    _, _, _, _, Ll, Hl, dt, N, _ = s["dims"]
    K = s["K"]
    kt = s["kt"][p.t_lo:p.t_hi, p.h_lo:p.h_hi].contiguous()
    vt = s["vt"][p.t_lo:p.t_hi, p.h_lo:p.h_hi].contiguous()
    nt, nh = p.t_hi - p.t_lo, p.h_hi - p.h_lo
    ko = torch.empty(nt, nh, K, dt, dtype=torch.bfloat16, device="cuda")
    vo = torch.empty_like(ko)
    idx = torch.empty(nt, nh, K, dtype=torch.int32, device="cuda")
    y = torch.empty(nt, nh, N, device="cuda")
    if stream_pair is None:
        pr.run(s["q"], s["kp"], kt, vt, ko, vo, idx, y)
    else:
        pr.run_dual(s["q"], s["kp"], kt, vt, ko, vo, idx, y, proxy_stream=stream_pair[0], target_stream=stream_pair[1])
    torch.cuda.synchronize()
    return p, ko, vo, idx, y


def _check(s, p, ko, vo, idx, y):
    import torch
    ref = s["ref"]
    sl = (slice(p.t_lo, p.t_hi), slice(p.h_lo, p.h_hi))
    assert torch.equal(y, ref["y"][sl])
    assert torch.equal(idx, ref["idx"][sl])
    assert torch.equal(ko.view(torch.int16), ref["ko"][sl].view(torch.int16))
    assert torch.equal(vo.view(torch.int16), ref["vo"][sl].view(torch.int16))


@pytest.mark.parametrize("world", [1, 2, 4])
def test_layer_sharded_ranks_bit_identical(setup, world):
    P = setup["P"]
    Ls, Hq, Hs, dp, Ll, Hl, dt, N, rho = setup["dims"]
    for rank in range(world):
        pr = P.Pruner(setup["m"], Hq, dp, dt, N, rho, shard=(P.SHARD_LAYER, world, rank))
        _check(setup, *_run_shard(setup, pr))


def test_head_sharded_world1_through_nccl(setup):
    P = setup["P"]
    Ls, Hq, Hs, dp, Ll, Hl, dt, N, rho = setup["dims"]
    comm = P.Comm(setup["m"].ctx, 1, 0, P.Comm.unique_id())
    pr = P.Pruner(setup["m"], Hq, dp, dt, N, rho, shard=(P.SHARD_HEAD, 1, 0), comm=comm)
    _check(setup, *_run_shard(setup, pr))


def test_head_sharding_requires_comm(setup):
    P = setup["P"]
    Ls, Hq, Hs, dp, Ll, Hl, dt, N, rho = setup["dims"]
    with pytest.raises(P.PkvValueError):
        P.Pruner(setup["m"], Hq, dp, dt, N, rho, shard=(P.SHARD_HEAD, 2, 0))


def test_dual_stream_matches_single_stream(setup):
    import torch
    P = setup["P"]
    Ls, Hq, Hs, dp, Ll, Hl, dt, N, rho = setup["dims"]
    pr = P.Pruner(setup["m"], Hq, dp, dt, N, rho)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    _check(setup, *_run_shard(setup, pr, stream_pair=(s1, s2)))
