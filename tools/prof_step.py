"""Runs the llama32k prune step a few times (for ncu launch lists / captures)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_16360_b200 as P  # noqa: E402

cfg = os.environ.get("PKV_CONFIG", "llama32k")
steps = int(os.environ.get("PKV_STEPS", "2"))
c = bench.CONFIGS[cfg]
ctx = P.Context(0)
m = P.Mapper(P.ModelGeometry(c["Ll"], c["Hl"], c["Ls"], c["Hs"], c["dt"]), P.MapperConfig(), seed=7,
             precision=int(os.environ.get("PKV_PREC", "3")), ctx=ctx)
pr = P.Pruner(m, c["Hq"], c["dp"], c["dt"], c["N"], c["rho"])
q, kp, kt, vt = bench.make_inputs(c, torch.device("cuda"), 1)
ko = torch.empty(c["Ll"], c["Hl"], pr.k, c["dt"], dtype=torch.bfloat16, device="cuda")
vo = torch.empty_like(ko)
idx = torch.empty(c["Ll"], c["Hl"], pr.k, dtype=torch.int32, device="cuda")
for _ in range(steps):
    pr.run(q, kp, kt, vt, ko, vo, idx)
torch.cuda.synchronize()
print("done", ctx.launches())
