#!/usr/bin/env python
"""bench.py — ProxyKV pruning hot path on B200: score -> map -> select -> compact.

Metric (BASELINE.json): proxy-scored+pruned tokens/s and prune latency at
Llama-3.2-1B (proxy) -> Llama-3.1-8B (target) shapes, 32k context, 1 GPU
(configs[1]); Top-K overlap is measured by the parity tests.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config llama32k|qwen25_128k|qwen25_170k|qwen3_64k|tiny]
                    [--shard auto|none|layer|head]

A "step" = one full prune of one context: inputs (proxy Q, proxy K, target K/V)
resident in HBM, outputs = packed K/V + retained indices. At N = 1 `value` =
tokens/s of one context on one GPU. Under torchrun (N > 1) the default
(--shard auto) is STRONG scaling of the same context: the context is split
across the N GPUs by target layer (configs[2]'s partition; no collective,
DESIGN.md §7), `value` = N_ctx / (max over ranks of the step time). The N > 1
line also carries `sharded_configs` (BASELINE configs[2]: Qwen-2.5 170k
layer-sharded; configs[3]: Qwen-3 64k head-group sharded with the NCCL
exchange of mapped scores, its time reported) and `weak_scaling` (one
independent context per GPU). `e2e` = the same metric through the C-ABI
host-buffer call (pkv_pruner_run_host: H2D of inputs and D2H of outputs inside
the timed region), all ranks concurrently, max over ranks. `--impl reference`
times the reference CPU implementation (oracle/_ref, the unmodified reference
sources) on the host's cores on a bounded sample of the same workload and
extrapolates to one context.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: proxy (L_s, Hq, H_s, dp), target (L_l, H_l, dt), N, rho
    "llama32k": dict(Ls=16, Hq=32, Hs=8, dp=64, Ll=32, Hl=8, dt=128, N=32768, rho=0.2,
                     desc="Llama-3.2-1B (16L,32Q/8KV,d64) proxy -> Llama-3.1-8B (32L,8KV,d128) target, 32k ctx"),
    "tiny": dict(Ls=2, Hq=4, Hs=4, dp=64, Ll=4, Hl=8, dt=64, N=2048, rho=0.2,
                 desc="tiny synthetic proxy(2L,4H,d64) -> target(4L,8H,d64), N=2048"),
    "qwen25_128k": dict(Ls=24, Hq=14, Hs=2, dp=64, Ll=28, Hl=4, dt=128, N=131072, rho=0.2,
                        desc="Qwen-2.5-0.5B (24L,14Q/2KV,d64) -> Qwen-2.5-7B (28L,4KV,d128), 128k ctx"),
    "qwen25_170k": dict(Ls=24, Hq=14, Hs=2, dp=64, Ll=28, Hl=4, dt=128, N=170000, rho=0.2,
                        desc="Qwen-2.5-0.5B (24L,14Q/2KV,d64) -> Qwen-2.5-7B (28L,4KV,d128), 170k ctx "
                             "(166 windows, right-aligned tail at 167952)"),
    "qwen3_64k": dict(Ls=28, Hq=16, Hs=8, dp=128, Ll=64, Hl=8, dt=128, N=65536, rho=0.2,
                      desc="Qwen-3-0.6B (28L,16Q/8KV,d128) -> Qwen-3-32B (64L,8KV,d128), 64k ctx"),
}
METRIC = "proxy-scored+pruned tokens/s & prune latency (8B shapes, 32k ctx); Top-K overlap"
UNIT = "tokens/s"


# ------------------------------------------------------------ workload math --
def windows(n, crop=2048, stride=1024):
    if n <= crop:
        return 1
    w = (n - crop) // stride + 1
    return w + (1 if (w - 1) * stride + crop < n else 0)


def unique_pairs(Ll, Ls):
    return len({(l * Ls + Ll - 1) // Ll for l in range(1, Ll + 1)})


def flops_score_pass(c):
    """2·d·Nq·Nk·Hq·L_s per pass (non-causal)."""
    return 2 * c["dp"] * c["N"] * c["N"] * c["Hq"] * c["Ls"]


def flops_mapper(c, D=512, enc=6, Dh=64):
    """per-window algorithmic FLOPs of the reference mapper x U·W."""
    nw = min(c["N"], 2048)
    syn = c["Hs"]
    per = (2 * nw * 256 * c["Hs"] * 3 + 2 * nw * 512 * 768 + enc * (24 * nw * D * D + 4 * nw * nw * D)
           + 4 * nw * D * syn * Dh + 4 * nw * c["Hl"] * syn * Dh + 2 * nw * c["Hl"] * Dh)
    return unique_pairs(c["Ll"], c["Ls"]) * windows(c["N"]) * per


def mma_flops_mapper(c, planes=3, D=512, enc=6, Dh=64):
    """Tensor-core work the mapper issues in a split-precision mode: its GEMM-shaped
    products (conv stem, QKV / Wo / FFN, stage-3 projections) run as `planes` MMAs
    each (3 in FP16X3, mode 3), the encoder attention's QK^T and PV as one."""
    nw = min(c["N"], 2048)
    syn = c["Hs"]
    gemm = (2 * nw * 256 * c["Hs"] * 3 + 2 * nw * 512 * 768 + enc * 24 * nw * D * D + 4 * nw * D * syn * Dh)
    rest = enc * 4 * nw * nw * D + 4 * nw * c["Hl"] * syn * Dh + 2 * nw * c["Hl"] * Dh
    return unique_pairs(c["Ll"], c["Ls"]) * windows(c["N"]) * (planes * gemm + rest)


def k_of(c):
    return math.ceil(c["rho"] * c["N"])


def bytes_select(c):
    s = c["Ll"] * c["Hl"]
    return s * c["N"] * 4 + s * k_of(c) * 4


def bytes_compact(c):
    s = c["Ll"] * c["Hl"]
    return 2 * s * k_of(c) * c["dt"] * 2 * 2 + s * k_of(c) * 4


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d["hbm_gbs"], d["bf16_tflops"], d.get("bf16_tflops_sustained", d["bf16_tflops"]), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


# ------------------------------------------------------------------ clocks --
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------- our arm --
def make_inputs(c, device, seed):
    import torch
    g = torch.Generator(device=device).manual_seed(seed)
    Ls, Hq, Hs, dp, N = c["Ls"], c["Hq"], c["Hs"], c["dp"], c["N"]
    q = torch.randn(Ls, Hq, N, dp, device=device, generator=g) * 0.35
    kp = torch.randn(Ls, Hs, N, dp, device=device, generator=g)
    u = torch.randn(dp, device=device, generator=g)
    u = u / u.norm()
    kp[:, :, : max(1, N // 50)] += 3.0 * u  # attention-sink structure
    q += 0.8 * u
    q, kp = q.to(torch.bfloat16), kp.to(torch.bfloat16)
    kt = torch.randn(c["Ll"], c["Hl"], N, c["dt"], device=device, generator=g).to(torch.bfloat16)
    vt = torch.randn(c["Ll"], c["Hl"], N, c["dt"], device=device, generator=g).to(torch.bfloat16)
    return q, kp, kt, vt


def time_loop(fn, iters, stream):
    """Device time per call of `fn` (launches onto `stream`), CUDA events on the
    launching stream. The launches are queued behind a spin kernel first, so
    back-to-back kernels are timed, not the host's ctypes / launch overhead
    (short kernels such as select would otherwise be host-bound)."""
    import torch
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        torch.cuda._sleep(int(2e5 * iters))  # ~0.1 ms per queued call at ~2 GHz
    a.record(stream)
    for _ in range(iters):
        fn()
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


def max_over_ranks(v, world, dev):
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], device=dev if dist.get_backend() == "nccl" else "cpu", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()


def gather_obj(world, obj):
    if world == 1:
        return [obj]
    import torch.distributed as dist
    out = [None] * world
    dist.all_gather_object(out, obj)
    return out


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def rank_work(c, plan):
    """Algorithmic work of one rank's part of the context."""
    pl = plan
    n_proxy = pl.p_hi - pl.p_lo if pl.b > pl.a else 0
    score = 2 * flops_score_pass(dict(c, Ls=n_proxy))
    units = len({(t + 1) * c["Ls"] // c["Ll"] + (1 if ((t + 1) * c["Ls"]) % c["Ll"] else 0) for t in range(pl.a, pl.b)})
    per_unit = flops_mapper(dict(c, Ll=1, Ls=1))  # one unit's windows
    slices = (pl.t_hi - pl.t_lo) * (pl.h_hi - pl.h_lo)
    sel = slices * c["N"] * 4 + slices * k_of(c) * 4
    cmp = 2 * slices * k_of(c) * c["dt"] * 2 * 2 + slices * k_of(c) * 4
    return {"proxy_layers": n_proxy, "mapper_units": units, "slices": slices, "score_flop": score,
            "map_flop": units * per_unit, "select_compact_bytes": sel + cmp}


class Arm:
    """One pruner (sharded or not) for config `c` with its resident inputs."""

    def __init__(self, P, ctx, c, dev, shard, world, rank, precision, seed):
        import torch
        self.c = c
        geom = P.ModelGeometry(c["Ll"], c["Hl"], c["Ls"], c["Hs"], c["dt"])
        self.mapper = P.Mapper(geom, P.MapperConfig(), seed=7, precision=precision, ctx=ctx)
        self.comm = None
        if shard == "none":
            self.pr = P.Pruner(self.mapper, c["Hq"], c["dp"], c["dt"], c["N"], c["rho"])
        else:
            mode = P.SHARD_HEAD if shard == "head" else P.SHARD_LAYER
            if mode == P.SHARD_HEAD:
                uid = [P.Comm.unique_id() if rank == 0 else None]
                if world > 1:
                    import torch.distributed as dist
                    dist.broadcast_object_list(uid, src=0)
                self.comm = P.Comm(ctx, world, rank, uid[0])
            self.pr = P.Pruner(self.mapper, c["Hq"], c["dp"], c["dt"], c["N"], c["rho"], shard=(mode, world, rank),
                               comm=self.comm)
        self.K = K = self.pr.k
        pl = self.plan = self.pr.plan
        q, kp, kt, vt = make_inputs(c, dev, seed=seed)
        self.q, self.kp = q, kp
        self.kt = kt[pl.t_lo:pl.t_hi, pl.h_lo:pl.h_hi].contiguous()
        self.vt = vt[pl.t_lo:pl.t_hi, pl.h_lo:pl.h_hi].contiguous()
        del kt, vt
        nt, nh = pl.t_hi - pl.t_lo, pl.h_hi - pl.h_lo
        self.ko = torch.empty(nt, nh, K, c["dt"], dtype=torch.bfloat16, device=dev)
        self.vo = torch.empty_like(self.ko)
        self.idx = torch.empty(nt, nh, K, dtype=torch.int32, device=dev)

    def step(self, stream):
        self.pr.run(self.q, self.kp, self.kt, self.vt, self.ko, self.vo, self.idx, stream=stream)

    def timed(self, steps, warmup, stream, world, dev):
        """max over ranks of the per-step device time (barrier + sync around)."""
        import torch
        for _ in range(warmup):
            self.step(stream)
        torch.cuda.synchronize()
        barrier(world)
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(steps):
            self.step(stream)
        b.record(stream)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / steps
        barrier(world)
        return ms, max_over_ranks(ms, world, dev)


def run_ours(args, c, rank, world, local_rank):
    import torch
    import paper_2605_16360_b200 as P

    # test-only knobs (functional runs of the N > 1 path on a one-GPU box):
    # PKV_BENCH_ONE_DEVICE=1 puts every rank on cuda:0, PKV_BENCH_BACKEND=gloo
    # replaces NCCL for the timing collectives (layer sharding has no data-path collective)
    dev_index = 0 if os.environ.get("PKV_BENCH_ONE_DEVICE") == "1" else local_rank
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("PKV_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    ctx = P.Context(dev_index)
    stream = torch.cuda.current_stream(dev)
    shard = args.shard if args.shard != "auto" else ("layer" if world > 1 else "none")
    # weak scaling replicas: an independent context per rank; sharded: every
    # rank holds its part of the same context
    arm = Arm(P, ctx, c, dev, shard, world, rank, args.precision, 1234 + (rank if shard == "none" else 0))

    for _ in range(args.warmup):
        arm.step(stream)
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    l0 = ctx.launches()
    arm.pr.profile(args.steps)  # stage-boundary events inside the timed steps (pkv_pruner_profile)
    with ClockSampler(dev_index) as clk:
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.steps):
            arm.step(stream)
        b.record(stream)
        torch.cuda.synchronize()
    ms_rank = a.elapsed_time(b) / args.steps
    launches = ctx.launches() - l0
    live = arm.pr.profile_read()
    arm.pr.profile(0)
    barrier(world)
    ms = max_over_ranks(ms_rank, world, dev)

    result = {"ms": ms, "K": arm.K, "launches": launches, "clocks": clk.summary(), "shard": shard}
    if live:
        names = ("score_lse", "score_pool", "map", "select", "compact")
        result["stages_live"] = {n: statistics.mean(r[i] for r in live) for i, n in enumerate(names)}
    work = rank_work(c, arm.plan)
    per_rank = {"rank": rank, "ms": ms_rank, **work,
                "score_map_TFLOP/s": (work["score_flop"] + work["map_flop"]) / (ms_rank * 1e-3) / 1e12}
    if world > 1:
        result["per_rank"] = gather_obj(world, per_rank)
    if rank == 0 and world == 1:
        result["stages"] = stage_breakdown(P, ctx, arm, c, stream, args)
    if not args.no_e2e:
        e = e2e(P, arm, c, args, world, dev)
        if rank == 0:
            result["e2e"] = e
    del arm
    torch.cuda.empty_cache()
    if (world > 1 and not args.no_extras) or args.extras:
        # the extra legs never cost the main line: a leg that raises is reported, not fatal, and a
        # watchdog emits the line without them if they have not finished within EXTRAS_BUDGET_S
        partial = dict(result)
        dog = threading.Timer(EXTRAS_BUDGET_S, extras_timeout, args=(partial, args, c, world, rank))
        dog.daemon = True
        dog.start()
        for key, leg in (("weak_scaling", lambda: weak_scaling(P, ctx, c, dev, world, rank, args, stream)),
                         ("sharded_configs", lambda: sharded_configs(P, ctx, dev, world, rank, args, stream))):
            try:
                result[key] = leg()
            except Exception as exc:  # noqa: BLE001
                result[key] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
                torch.cuda.synchronize()
        dog.cancel()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return result


EXTRAS_BUDGET_S = float(os.environ.get("PKV_BENCH_EXTRAS_BUDGET_S", "420"))


def extras_timeout(partial, args, c, world, rank):
    """The extra legs overran (e.g. a communicator that never forms): rank 0 emits the
    main line with the legs marked, and every rank exits."""
    if rank == 0:
        for key in ("weak_scaling", "sharded_configs"):
            partial.setdefault(key, {"error": f"not finished within {EXTRAS_BUDGET_S:.0f} s"})
        try:
            emit(build_line(partial, args, c, world))
        finally:
            os._exit(0)
    os._exit(0)


def weak_scaling(P, ctx, c, dev, world, rank, args, stream):
    import torch
    arm = Arm(P, ctx, c, dev, "none", world, rank, args.precision, 1234 + rank)
    _, ms = arm.timed(max(2, min(args.steps, 5)), 3, stream, world, dev)
    del arm
    torch.cuda.empty_cache()
    return {"value": world * c["N"] / (ms * 1e-3), "unit": UNIT, "ms_per_step": ms,
            "note": f"{world} independent {c['N']}-token contexts, one per GPU, no collective"}


def sharded_configs(P, ctx, dev, world, rank, args, stream):
    """BASELINE configs[2] (Qwen-2.5 170k, layer-sharded) and configs[3]
    (Qwen-3 64k, head-group sharded: NCCL all-to-all of mapped scores) as
    strong scaling of one context over the `world` GPUs."""
    import torch
    out = {}
    for name, mode in (("qwen25_170k", "layer"), ("qwen3_64k", "head")):
        cc = CONFIGS[name]
        if (mode == "layer" and world > cc["Ll"]) or (mode == "head" and world > cc["Hl"]):
            continue
        arm = Arm(P, ctx, cc, dev, mode, world, rank, args.precision, 1234)
        ms_rank, ms = arm.timed(max(2, min(args.steps, 3)), 3, stream, world, dev)
        rec = {"shard": mode, "N": cc["N"], "ms_per_context": ms, "tokens_per_s": cc["N"] / (ms * 1e-3),
               "desc": cc["desc"]}
        work = rank_work(cc, arm.plan)
        rec["per_rank"] = gather_obj(world, {"rank": rank, "ms": ms_rank, **work,
                                             "score_map_TFLOP/s": (work["score_flop"] + work["map_flop"]) /
                                                                  (ms_rank * 1e-3) / 1e12})
        if mode == "head":
            pl = arm.plan
            y_local = torch.zeros(max(pl.b - pl.a, 1), cc["Hl"], cc["N"], device=dev)
            y_recv = torch.zeros(cc["Ll"], pl.h_hi - pl.h_lo, cc["N"], device=dev)
            barrier(world)
            x_ms = time_loop(lambda: arm.pr.exchange(y_local, y_recv, stream=stream), 5, stream)
            rec["exchange_ms"] = max_over_ranks(x_ms, world, dev)
            rec["exchange_bytes_total"] = cc["Ll"] * cc["Hl"] * cc["N"] * 4
        del arm
        torch.cuda.empty_cache()
        out[name] = rec
    return out


def stage_breakdown(P, ctx, arm, c, stream, args):
    """Each stage alone through the C ABI with preallocated outputs, timed as
    back-to-back launches (time_loop)."""
    import torch
    L = P.lib()
    q, kp, kt, vt, ko, vo, K = arm.q, arm.kp, arm.kt, arm.vt, arm.ko, arm.vo, arm.K
    sp = stream.cuda_stream
    it = max(3, min(args.steps, 5))
    dev = q.device
    lse = torch.empty(c["Ls"], c["Hq"], c["N"], device=dev)
    x = torch.empty(c["Ls"], c["Hs"], c["N"], device=dev)
    y = torch.empty(1, c["Ll"], c["Hl"], c["N"], device=dev)
    S = c["Ll"] * c["Hl"]
    idx = torch.empty(S, K, dtype=torch.int32, device=dev)
    dims = (c["Ls"], c["Hq"], c["Hs"], c["N"], c["N"], c["dp"])
    lse_call = lambda: P.check(L.pkv_score_lse(ctx.h, q.data_ptr(), kp.data_ptr(), *dims, 0, lse.data_ptr(), sp))
    pool_call = lambda: P.check(L.pkv_score(ctx.h, q.data_ptr(), kp.data_ptr(), *dims, P.SCORE_REDUCE_MAX,
                                            lse.data_ptr(), x.data_ptr(), sp))
    map_call = lambda: P.check(L.pkv_mapper_forward_full(arm.mapper.h, x.data_ptr(), 1, c["N"], y.data_ptr(), sp))
    sel_call = lambda: P.check(L.pkv_topk_select(ctx.h, y.data_ptr(), S, c["N"], K, None, idx.data_ptr(), sp))
    cmp_call = lambda: P.check(L.pkv_compact_kv(ctx.h, kt.data_ptr(), vt.data_ptr(), idx.data_ptr(), S, c["N"], K,
                                                c["dt"], 2, ko.data_ptr(), vo.data_ptr(), sp))
    for f in (lse_call, pool_call, map_call, sel_call, cmp_call):
        f()
    out = {}
    out["score_lse_ms"] = time_loop(lse_call, it, stream)
    out["score_pool_ms"] = time_loop(pool_call, it, stream)
    out["map_ms"] = time_loop(map_call, it, stream)
    # the short stages: an untimed loop first and long timed loops — the first few ms of
    # back-to-back launches after the long stages run ~45 % slow for select
    # (tools/probe_select_bench.py: 56.8 then 37.0 us on the same data; ncu: 39 us per launch):
    # the power-capped clock after the long stages; an idle gap lets it recover before these
    # latency-bound kernels are timed alone (their in-step cost is stages_live_ms)
    torch.cuda.synchronize()
    time.sleep(0.5)
    time_loop(sel_call, 100, stream)
    out["select_ms"] = time_loop(sel_call, 200, stream)
    time_loop(cmp_call, 20, stream)
    out["compact_ms"] = time_loop(cmp_call, 40, stream)
    # causal scoring with the LSE emitted by the proxy's own prefill
    # attention (its O is the proxy model's output anyway): one scoring pass
    vp = torch.randn_like(kp)
    _, plse = P.proxy_prefill_attention(q, kp, vp, causal=True, want_out=True, ctx=ctx)
    out["x_prefill_attn_causal_ms"] = time_loop(
        lambda: P.proxy_prefill_attention(q, kp, vp, causal=True, want_out=True, ctx=ctx, stream=stream), it, stream)
    out["x_score_pool_causal_ms"] = time_loop(
        lambda: P.score(q, kp, lse=plse, causal=True, ctx=ctx, stream=stream, out=x), it, stream)
    # the whole prune in that regime: causal pruner fed the prefill LSE (pkv_pruner_run_lse)
    prc = P.Pruner(arm.mapper, c["Hq"], c["dp"], c["dt"], c["N"], c["rho"], causal=True)
    prc.run_lse(q, kp, plse, kt, vt, ko, vo, stream=stream)
    out["x_prune_with_prefill_lse_ms"] = time_loop(lambda: prc.run_lse(q, kp, plse, kt, vt, ko, vo, stream=stream),
                                                   it, stream)
    return out


def e2e(P, arm, c, args, world, dev):
    """The public host-buffer call on every rank at once (pinned host inputs in,
    packed K/V + indices out, copies inside the timed region); max over ranks."""
    import torch
    pl = arm.plan
    q, kp, kt, vt = make_inputs(c, dev, seed=99)
    kt = kt[pl.t_lo:pl.t_hi, pl.h_lo:pl.h_hi]
    vt = vt[pl.t_lo:pl.t_hi, pl.h_lo:pl.h_hi]
    q, kp, kt, vt = (t.contiguous().cpu().pin_memory() for t in (q, kp, kt, vt))
    nt, nh = pl.t_hi - pl.t_lo, pl.h_hi - pl.h_lo
    K = arm.K
    ko = torch.empty(nt, nh, K, c["dt"], dtype=torch.bfloat16).pin_memory()
    vo = torch.empty_like(ko).pin_memory()
    idx = torch.empty(nt, nh, K, dtype=torch.int32).pin_memory()
    stream = torch.cuda.current_stream()
    step = lambda: arm.pr.run_host(q, kp, kt, vt, ko, vo, idx, stream=stream)
    for _ in range(max(1, min(args.warmup, 2))):
        step()
    n = max(2, min(args.steps, 5))
    torch.cuda.synchronize()
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(n):
        step()  # synchronises on the stream at the end of every call
    ms = (time.perf_counter() - t0) * 1e3 / n
    ms = max_over_ranks(ms, world, dev)
    # bytes this rank moves: the proxy layers its pruner reads + its KV shard in, its outputs back
    Ls = c["Ls"]
    read_layers = (pl.p_hi - pl.p_lo) if pl.b > pl.a else 0
    h2d = (q.numel() * 2 + kp.numel() * 2) * read_layers // Ls + (kt.numel() + vt.numel()) * 2
    d2h = sum(t.numel() * t.element_size() for t in (ko, vo, idx))
    return {"ms": ms, "h2d": h2d, "d2h": d2h}


# ---------------------------------------------------------- reference arm --
def cpu_reference_sample(c, threads, include_mapper=True):
    """Times the reference CPU implementation on a bounded sample of one context
    and extrapolates to the full context (seconds per context, per stage).
      select+indices: reference topk_mask + apply_mask on one full target layer
                      (H_l slices of N), x L_l layers;
      compaction:     (no reference code) C restatement gather of one layer, x L_l;
      mapper:         reference forward_pair on one 2048-window per thread, run
                      concurrently on `threads` cores, x ceil(U·W / threads);
      scoring:        (SPEC-only, no reference code) fp64 C restatement on one
                      (layer, KV head) with 256 queries per thread, scaled by
                      the full query count, heads and layers."""
    import numpy as np
    from concurrent.futures import ThreadPoolExecutor
    from oracle import pkv_oracle as O

    ref = O.RefLib()
    N, Ll, Hl, dt = c["N"], c["Ll"], c["Hl"], c["dt"]
    r = np.random.RandomState(0)
    out = {}
    # select + apply_mask, one target layer
    s = r.rand(1, 1, Hl, N)
    t0 = time.perf_counter()
    bits, k = ref.topk_mask(s, c["rho"])
    ref.apply_mask(bits, k, dt)
    out["select"] = (time.perf_counter() - t0) * Ll
    # compaction, one target layer (C restatement; the reference has no gather)
    kb = r.randint(0, 1 << 15, (Hl, N, dt)).astype(np.uint16)
    _, idx = O.topk_select(s.reshape(Hl, N).astype(np.float32), k)
    t0 = time.perf_counter()
    O.compact_kv(kb, kb, idx)
    out["compact"] = (time.perf_counter() - t0) * Ll
    # scoring: `threads` concurrent (layer, kv-head) samples of 256 queries of one head group
    g = c["Hq"] // c["Hs"]
    nq = 256
    qb = O.f32_to_bf16_bits(r.standard_normal((1, g, nq, c["dp"])).astype(np.float32))
    kk = O.f32_to_bf16_bits(r.standard_normal((1, 1, N, c["dp"])).astype(np.float32))

    def one_score(_):
        O.score(qb, kk, reduce="max")

    t0 = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(one_score, range(threads)))
    ts = time.perf_counter() - t0
    units = (N / nq) * c["Ls"] * c["Hs"]  # (layer, kv head, 256-query block) units per context
    out["score"] = ts * units / threads
    if include_mapper:
        geo = O.Geometry(Ll, Hl, c["Ls"], c["Hs"], dt)
        m = ref.mapper(geo, O.MapperConfig(), 7)
        x = r.uniform(0, 2, (1, c["Hs"], min(N, 2048)))
        t0 = time.perf_counter()
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(lambda _: m.forward_pair(x), range(threads)))
        tm = time.perf_counter() - t0
        n_win = unique_pairs(Ll, c["Ls"]) * windows(N)
        out["map"] = tm * math.ceil(n_win / threads)
    return out


def cpu_sample_desc(c, threads):
    return (f"reference topk_mask+apply_mask on 1 of {c['Ll']} target layers (x{c['Ll']}); reference forward_pair on "
            f"{threads} concurrent 2048-windows (x ceil({unique_pairs(c['Ll'], c['Ls'])}*{windows(c['N'])}/{threads})); "
            f"fp64 C-restatement scoring of {threads} (layer,kv-head,256-query) blocks and gather of 1 layer "
            f"(no reference code for those), extrapolated to one {c['N']}-token context")


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def cpu_legs(c, st, threads):
    """Which stage times are the reference's own code and which are the C
    restatement (no reference code), and how each was extrapolated."""
    U, W = unique_pairs(c["Ll"], c["Ls"]), windows(c["N"])
    return {
        "select": {"s": st["select"], "code": "reference (topk_mask + apply_mask, pruning.cpp)",
                   "extrapolated": f"1 of {c['Ll']} target layers timed, x{c['Ll']}"},
        "map": {"s": st["map"], "code": "reference (forward_pair, mapper.cpp)",
                "extrapolated": f"{threads} windows timed concurrently on {threads} cores, x ceil({U}*{W}/{threads})"},
        "score": {"s": st["score"], "code": "C restatement (SPEC-only scoring, no reference code)",
                  "extrapolated": f"{threads} (layer, kv-head, 256-query) blocks, x N/256*L_s*H_s/{threads}"},
        "compact": {"s": st["compact"], "code": "C restatement (the reference has no gather)",
                    "extrapolated": f"1 of {c['Ll']} target layers, x{c['Ll']}"},
    }


def run_reference(args, c):
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):  # warm-up: the cheap stages only
        cpu_reference_sample(c, threads, include_mapper=False)
    totals = []
    t_wall = time.perf_counter()
    for _ in range(args.steps):
        st = cpu_reference_sample(c, threads)
        totals.append(sum(st.values()))
    t_wall = time.perf_counter() - t_wall
    sec = statistics.mean(totals)
    value = c["N"] / sec
    return {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.config, "desc": c["desc"], "rho": c["rho"], "N": c["N"]},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "cpu_model": cpu_model(),
                         "kind": "reference", "sample": cpu_sample_desc(c, threads), "extrapolated": True,
                         "timed_wall_s_per_step": t_wall / max(args.steps, 1),
                         "stage_s": {k: round(v, 3) for k, v in st.items()}, "legs": cpu_legs(c, st, threads)},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


# -------------------------------------------------------------------- main --
_OUT_FD = 1  # the real stdout (main() routes fd 1 to stderr for native output)


def emit(obj):
    os.write(_OUT_FD, (json.dumps(obj) + "\n").encode())


def cpu_baseline_entry(c):
    """The reference's CPU path on the host cores, a bounded sample (world 1 only)."""
    try:
        threads = os.cpu_count() or 1
        stc = cpu_reference_sample(c, threads)
        sec = sum(stc.values())
        return {"cpu_baseline": {"value": c["N"] / sec, "unit": UNIT, "cores": threads, "cpu_model": cpu_model(),
                                 "kind": "reference", "sample": cpu_sample_desc(c, threads), "extrapolated": True,
                                 "stage_s": {k: round(v, 3) for k, v in stc.items()},
                                 "legs": cpu_legs(c, stc, threads)}}
    except Exception as e:  # noqa: BLE001
        return {"cpu_baseline": {"value": None, "unavailable": f"{type(e).__name__}: {e}"}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="llama32k")
    ap.add_argument("--precision", type=int, default=3, help="mapper precision mode (1 fp16, 2 act split, 3 act+wt split)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="N > 1: skip weak_scaling and sharded_configs")
    ap.add_argument("--extras", action="store_true", help="run weak_scaling and sharded_configs even at N = 1 "
                                                          "(exercises the sharded code paths on one GPU)")
    ap.add_argument("--shard", choices=["auto", "none", "layer", "head"], default="auto",
                    help="auto: none at N = 1, layer at N > 1 (strong scaling of one context); none: weak scaling "
                         "(one independent context per GPU); head: head-group sharding with the NCCL exchange")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    c = CONFIGS[args.config]
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator / NVLS setup, to stderr (below)
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    # stdout carries exactly one JSON line: everything native code prints (NCCL's
    # version banner and INFO log, CUDA libraries) goes to stderr, the line to the
    # saved stdout descriptor
    sys.stdout.flush()
    global _OUT_FD
    _OUT_FD = os.dup(1)
    os.dup2(2, 1)

    if args.impl == "reference":
        if rank == 0:
            try:
                emit(run_reference(args, c))
            except Exception as e:  # noqa: BLE001
                emit({"impl": "reference", "unavailable": f"{type(e).__name__}: {e}"})
        return

    r = run_ours(args, c, rank, world, local_rank)
    if rank != 0:
        return
    line = build_line(r, args, c, world)
    if not args.no_cpu_baseline and world == 1:
        line.update(cpu_baseline_entry(c))
    emit(line)


def build_line(r, args, c, world):
    """The JSON line (without the CPU baseline) from run_ours' result."""
    hbm, tf_burst, tf_sus, src = peaks()
    ms = r["ms"]
    sharded = r["shard"] != "none"
    n_ctx = 1 if sharded else world
    line = {
        "metric": METRIC, "value": c["N"] * n_ctx / (ms * 1e-3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": args.config, "desc": c["desc"], "rho": c["rho"], "N": c["N"], "K": r["K"],
                   "mapper_precision": args.precision, "score_reduce": "max", "score_passes": 2,
                   "l2": "inputs (>= 7 GB) > L2 (126 MB); no explicit flush",
                   "parallelism": (f"{r['shard']}-sharded: one context over {world} GPUs" if sharded
                                   else f"weak: {world} independent contexts, one per GPU")},
        "prune_latency_ms": ms,
    }
    if "stages" in r:
        st = r["stages"]
        # roofline of the dominant KERNEL: the single-kernel stages (map is ~47 launches)
        single = {"score_lse_ms": ("tensor", flops_score_pass(c)), "score_pool_ms": ("tensor", flops_score_pass(c)),
                  "select_ms": ("hbm", bytes_select(c)), "compact_ms": ("hbm", bytes_compact(c))}
        dom = max(single, key=lambda k: st[k])
        bound, work = single[dom]
        live = r.get("stages_live")
        if bound == "tensor":
            ach_alone = work / (st[dom] * 1e-3) / 1e12
            if live:  # the kernel's duration inside the timed steps (pkv_pruner_profile events on its stream)
                ach = work / (live[dom[:-3]] * 1e-3) / 1e12
                roof = {"kernel": dom[:-3], "bound": "tensor", "achieved": ach, "peak": tf_sus, "unit": "TFLOP/s",
                        "frac": ach / tf_sus, "traffic": None,
                        "peak_source": f"{src} bf16 sustained (kernel timed inside the timed steps: CUDA events "
                                       f"on its stream at the stage boundaries, mean over the steps)"}
            else:
                roof = {"kernel": dom[:-3], "bound": "tensor", "achieved": ach_alone, "peak": tf_burst,
                        "unit": "TFLOP/s", "frac": ach_alone / tf_burst, "traffic": None,
                        "peak_source": f"{src} bf16 burst (kernel timed alone)"}
            roof["note"] = ("algorithmic FLOPs (2*d*Nq*Nk*Hq*L_s per pass); the pass is bounded by MUFU exp2 "
                            "throughput (16/clk/SM), not the tensor pipe (DESIGN.md section 5)")
            # the same kernel timed alone (stages_ms) against the burst peak, for comparison
            roof["alone"] = {"ms": st[dom], "achieved": ach_alone, "frac_of_burst": ach_alone / tf_burst}
        else:
            ach = work / (st[dom] * 1e-3) / 1e9
            roof = {"kernel": dom[:-3], "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s",
                    "frac": ach / hbm, "traffic": None, "peak_source": f"{src} hbm"}
        prof = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(prof):
            roof["traffic"] = json.load(open(prof)).get(roof["kernel"])
        if roof["kernel"] == "score_lse" and r.get("clocks", {}).get("sm_mhz"):
            # the pass's real bound: exponentials on the MUFU (16 ex2/clk/SM) with
            # kPolyPairs of every 32 pairs on the FMA pipe, at the measured SM clock
            import torch
            poly = int(os.environ.get("PKV_POLY_PAIRS", "10"))
            exps = c["N"] * c["N"] * c["Hq"] * c["Ls"]
            on_mufu = exps * (32 - poly) / 32
            sms = torch.cuda.get_device_properties(0).multi_processor_count
            peak_exp = 16 * sms * r["clocks"]["sm_mhz"] * 1e6
            ach_exp = on_mufu / ((live["score_lse"] if live else st["score_lse_ms"]) * 1e-3)
            roof["exp_pipe"] = {"exponentials": exps, "on_mufu": on_mufu, "achieved_mufu_ex2_per_s": ach_exp,
                                "peak_ex2_per_s_at_measured_clock": peak_exp, "frac": ach_exp / peak_exp,
                                "note": f"{poly} of 32 pairs use the FMA-pipe polynomial; peak = 16/clk/SM x "
                                        f"{sms} SMs x median SM clock under load"}
        sc_b = bytes_select(c) + bytes_compact(c)
        sc_ms = st["select_ms"] + st["compact_ms"]
        line["stages_ms"] = {k[:-3]: v for k, v in st.items() if not k.startswith("x_")}
        if live:
            line["stages_live_ms"] = live
            line["stages_live_note"] = ("mean over the timed steps of each stage's time inside the step: CUDA events "
                                        "recorded on the launching stream at the stage boundaries "
                                        "(pkv_pruner_profile); the LSE pass includes its max|k| / flag setup")
        line["stages_note"] = ("each stage alone through the C ABI with preallocated outputs, back-to-back launches "
                               "queued behind a spin kernel (device time, not host launch overhead); select and "
                               "compact after a 0.5 s idle gap so the power-capped clock has recovered")
        fc = 2 * c["dp"] * (c["N"] * (c["N"] + 1) // 2) * c["Hq"] * c["Ls"]  # causal pairs
        line["scoring_single_pass"] = {
            "note": "causal scoring with the LSE from the proxy's prefill attention (pkv_proxy_prefill_attention, "
                    "SURVEY 8(f)-1): one tensor-core pass; the prefill attention itself is proxy-model work",
            "proxy_prefill_attn_ms": st["x_prefill_attn_causal_ms"], "score_pool_ms": st["x_score_pool_causal_ms"],
            "TFLOP/s": fc / st["x_score_pool_causal_ms"] / 1e9,
            "frac_of_burst": fc / st["x_score_pool_causal_ms"] / 1e9 / tf_burst,
            "prune_latency_ms": st["x_prune_with_prefill_lse_ms"],
            "prune_note": "pkv_pruner_run_lse: causal pooled pass + map + select + compact, the prefill LSE given"}
        line["stage_roofline"] = {
            "score_lse": {"TFLOP/s": flops_score_pass(c) / st["score_lse_ms"] / 1e9},
            "score_pool": {"TFLOP/s": flops_score_pass(c) / st["score_pool_ms"] / 1e9},
            "map": {"TFLOP/s": flops_mapper(c) / st["map_ms"] / 1e9,
                    **({"mma_issued_TFLOP/s": mma_flops_mapper(c) / st["map_ms"] / 1e9,
                        "mma_issued_frac_of_burst": mma_flops_mapper(c) / st["map_ms"] / 1e9 / tf_burst,
                        "note": "FP16X3: each GEMM-shaped product issued as 3 fp16 MMAs (hi/lo planes), the "
                                "attention as 1; TFLOP/s above is the reference mapper's algorithmic work"}
                       if args.precision == 3 else {})},
            "select": {"GB/s": bytes_select(c) / st["select_ms"] / 1e6,
                       "frac_hbm": bytes_select(c) / st["select_ms"] / 1e6 / hbm},
            "compact": {"GB/s": bytes_compact(c) / st["compact_ms"] / 1e6,
                        "frac_hbm": bytes_compact(c) / st["compact_ms"] / 1e6 / hbm},
            "select+compact": {"GB/s": sc_b / sc_ms / 1e6, "frac_hbm": sc_b / sc_ms / 1e6 / hbm},
        }
        line["roofline"] = roof
    for key in ("per_rank", "weak_scaling", "sharded_configs"):
        if key in r:
            line[key] = r[key]
    line["clocks"] = r["clocks"]
    line["gpu_launches"] = r["launches"]
    if "e2e" in r:
        e = r["e2e"]
        line["e2e"] = {"value": c["N"] * n_ctx / (e["ms"] * 1e-3), "unit": UNIT,
                       "h2d_bytes_per_step": e["h2d"], "d2h_bytes_per_step": e["d2h"], "ms_per_step": e["ms"],
                       "note": "pkv_pruner_run_host on every rank at once (wall clock, synchronised per call, max over "
                               "ranks); bytes are rank 0's"}
    return line



if __name__ == "__main__":
    main()
