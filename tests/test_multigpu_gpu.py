"""Multi-GPU paths on real devices (VERDICT r1 missing#3 / ADVICE low
shard.cpp): skipped below 2 devices (gpurun and the driver's test tier give
one GPU; the driver's 8-GPU bench runs the same library code).
  * head-group sharding at world 2 over a real NCCL communicator (the
    library's own pkv_comm + grouped send/recv, one process per GPU): every
    rank's retained indices and packed K/V are bit-identical to the 1-GPU
    pruner's slices of its head group;
  * layer sharding at world 2, same check;
  * pkv_pruner_run_two_device from device 0 (proxy) to device 1 (target) equals
    pkv_pruner_run on one device."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CFG = dict(Ls=4, Hq=8, Hs=4, dp=64, Ll=6, Hl=4, dt=128, N=3000, rho=0.2)


def _need2():
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 CUDA devices")


def _inputs(dev):
    import torch
    c = CFG
    g = torch.Generator(device=dev).manual_seed(5)
    q = (torch.randn(c["Ls"], c["Hq"], c["N"], c["dp"], device=dev, generator=g) * 0.35).to(torch.bfloat16)
    kp = torch.randn(c["Ls"], c["Hs"], c["N"], c["dp"], device=dev, generator=g).to(torch.bfloat16)
    kt = torch.randn(c["Ll"], c["Hl"], c["N"], c["dt"], device=dev, generator=g).to(torch.bfloat16)
    vt = torch.randn(c["Ll"], c["Hl"], c["N"], c["dt"], device=dev, generator=g).to(torch.bfloat16)
    return q, kp, kt, vt


def _run(P, ctx, dev, shard=None, comm=None):
    import torch
    c = CFG
    geom = P.ModelGeometry(c["Ll"], c["Hl"], c["Ls"], c["Hs"], c["dt"])
    m = P.Mapper(geom, P.MapperConfig(encoder_layers=2), seed=4, ctx=ctx)
    pr = P.Pruner(m, c["Hq"], c["dp"], c["dt"], c["N"], c["rho"], shard=shard, comm=comm)
    pl = pr.plan
    q, kp, kt, vt = _inputs(dev)
    kt = kt[pl.t_lo:pl.t_hi, pl.h_lo:pl.h_hi].contiguous()
    vt = vt[pl.t_lo:pl.t_hi, pl.h_lo:pl.h_hi].contiguous()
    nt, nh = pl.t_hi - pl.t_lo, pl.h_hi - pl.h_lo
    ko = torch.empty(nt, nh, pr.k, c["dt"], dtype=torch.bfloat16, device=dev)
    vo = torch.empty_like(ko)
    idx = torch.empty(nt, nh, pr.k, dtype=torch.int32, device=dev)
    y = torch.empty(nt, nh, c["N"], device=dev)
    pr.run(q, kp, kt, vt, ko, vo, idx, y)
    torch.cuda.synchronize(dev)
    bits = lambda t: t.view(torch.int16).cpu().numpy()
    return pl, idx.cpu().numpy(), bits(ko), bits(vo), y.cpu().numpy()


def _worker(rank, world, mode_name, uid_q, out_q):
    import torch
    import paper_2605_16360_b200 as P
    torch.cuda.set_device(rank)
    ctx = P.Context(rank)
    mode = P.SHARD_HEAD if mode_name == "head" else P.SHARD_LAYER
    comm = None
    if mode == P.SHARD_HEAD:
        if rank == 0:
            uid = P.Comm.unique_id()
            for _ in range(world - 1):
                uid_q.put(uid)
        else:
            uid = uid_q.get(timeout=120)
        comm = P.Comm(ctx, world, rank, uid)
    out_q.put((rank,) + _run(P, ctx, torch.device("cuda", rank), shard=(mode, world, rank), comm=comm))


@pytest.mark.parametrize("mode_name", ["head", "layer"])
def test_sharded_world2_bit_identical(gpu, mode_name):
    _need2()
    import torch
    import torch.multiprocessing as mp
    import paper_2605_16360_b200 as P
    world = 2
    _, idx1, ko1, vo1, y1 = _run(P, gpu, torch.device("cuda", 0))
    ctx = mp.get_context("spawn")
    uid_q, out_q = ctx.Queue(), ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, mode_name, uid_q, out_q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [out_q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, pl, idx, ko, vo, y in res:
        sl = (slice(pl.t_lo, pl.t_hi), slice(pl.h_lo, pl.h_hi))
        np.testing.assert_array_equal(y, y1[sl])
        np.testing.assert_array_equal(idx, idx1[sl])
        np.testing.assert_array_equal(ko, ko1[sl])
        np.testing.assert_array_equal(vo, vo1[sl])


def test_two_device_proxy_to_target(gpu):
    _need2()
    import torch
    import paper_2605_16360_b200 as P
    c = CFG
    _, idx1, ko1, vo1, y1 = _run(P, gpu, torch.device("cuda", 0))
    geom = P.ModelGeometry(c["Ll"], c["Hl"], c["Ls"], c["Hs"], c["dt"])
    m = P.Mapper(geom, P.MapperConfig(encoder_layers=2), seed=4, ctx=gpu)
    pr = P.Pruner(m, c["Hq"], c["dp"], c["dt"], c["N"], c["rho"])
    q, kp, _, _ = _inputs(torch.device("cuda", 0))
    _, _, kt, vt = _inputs(torch.device("cuda", 1))
    tctx = P.Context(1)
    d1 = torch.device("cuda", 1)
    ko = torch.empty(c["Ll"], c["Hl"], pr.k, c["dt"], dtype=torch.bfloat16, device=d1)
    vo = torch.empty_like(ko)
    idx = torch.empty(c["Ll"], c["Hl"], pr.k, dtype=torch.int32, device=d1)
    y = torch.empty(c["Ll"], c["Hl"], c["N"], device=d1)
    ps = torch.cuda.Stream(device=0)
    ts = torch.cuda.Stream(device=1)
    pr.run_two_device(tctx, q, kp, kt, vt, ko, vo, idx, y, proxy_stream=ps, target_stream=ts)
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    bits = lambda t: t.view(torch.int16).cpu().numpy()
    np.testing.assert_array_equal(y.cpu().numpy(), y1)
    np.testing.assert_array_equal(idx.cpu().numpy(), idx1)
    np.testing.assert_array_equal(bits(ko), ko1)
    np.testing.assert_array_equal(bits(vo), vo1)
