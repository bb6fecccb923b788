"""Scoring pass 1 (pkv_score_lse) timed in different contexts, to explain why it
runs slower inside the bench step than alone: back to back, right after a
mapper forward_full, right after a compaction, and after an idle pause. CUDA
events around the pass only."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_16360_b200 as P  # noqa: E402

c = bench.CONFIGS["llama32k"]
dev = torch.device("cuda", 0)
ctx = P.Context(0)
arm = bench.Arm(P, ctx, c, dev, "none", 1, 0, 3, 1234)
st = torch.cuda.current_stream()
L = P.lib()
dims = (c["Ls"], c["Hq"], c["Hs"], c["N"], c["N"], c["dp"])
lse = torch.empty(c["Ls"], c["Hq"], c["N"], device=dev)
x = P.score(arm.q, arm.kp, ctx=ctx)
y = torch.empty(1, c["Ll"], c["Hl"], c["N"], device=dev)
lse_call = lambda: P.check(L.pkv_score_lse(ctx.h, arm.q.data_ptr(), arm.kp.data_ptr(), *dims, 0, lse.data_ptr(),
                                           st.cuda_stream))
map_call = lambda: arm.mapper.forward_full(x[None], stream=st, out=y)
step_call = lambda: arm.step(st)
for _ in range(2):
    lse_call()
    map_call()
torch.cuda.synchronize()


def timed_lse(before, reps=5, pause=0.0):
    ts = []
    for _ in range(reps):
        if pause:
            torch.cuda.synchronize()
            time.sleep(pause)
        if before:
            before()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        lse_call()
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sum(ts) / len(ts)


print(f"back to back:            {timed_lse(None):.1f} ms", flush=True)
print(f"after mapper forward:    {timed_lse(map_call):.1f} ms", flush=True)
print(f"after a whole prune step: {timed_lse(step_call):.1f} ms", flush=True)
print(f"after a 300 ms idle:     {timed_lse(None, pause=0.3):.1f} ms", flush=True)
print(f"back to back again:      {timed_lse(None):.1f} ms", flush=True)
