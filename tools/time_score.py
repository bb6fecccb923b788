"""Time the two scoring passes alone at a bench config (tuning aid; prints one
line per pass). LSE accuracy is checked on a sampled set of rows against a
float64 torch evaluation of the same bf16 inputs.

    PKV_POLY_PAIRS=14 python tools/time_score.py [--config llama32k]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_16360_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="llama32k")
ap.add_argument("--iters", type=int, default=3)
a = ap.parse_args()
c = bench.CONFIGS[a.config]
dev = torch.device("cuda", 0)
ctx = P.Context(0)
q, kp, _, _ = bench.make_inputs(c, dev, seed=1234)
st = torch.cuda.current_stream()
lse = P.score_lse(q, kp, ctx=ctx)
x = torch.empty(c["Ls"], c["Hs"], c["N"], device=dev)
P.score(q, kp, lse=lse, ctx=ctx, out=x)
t1 = bench.time_loop(lambda: P.score_lse(q, kp, ctx=ctx, stream=st), a.iters, st)
t2 = bench.time_loop(lambda: P.score(q, kp, lse=lse, ctx=ctx, stream=st, out=x), a.iters, st)
f = bench.flops_score_pass(c)
# sampled LSE check (fp64 over all keys for 64 rows of a few heads)
g = torch.Generator().manual_seed(0)
err = 0.0
d = c["dp"]
for l, h in [(0, 0), (c["Ls"] - 1, c["Hq"] - 1), (c["Ls"] // 2, 3)]:
    rows = torch.randint(0, c["N"], (64,), generator=g)
    qs = q[l, h, rows].double()
    ks = kp[l, h // (c["Hq"] // c["Hs"])].double()
    ref = torch.logsumexp(qs @ ks.T / d ** 0.5, dim=1)
    err = max(err, (lse[l, h, rows].double() - ref).abs().max().item())
print(f"poly={os.environ.get('PKV_POLY_PAIRS', 'default')} lse {t1:.2f} ms ({f / t1 / 1e9:.0f} TF/s)  "
      f"pool {t2:.2f} ms ({f / t2 / 1e9:.0f} TF/s)  max|dlse| {err:.2e}")
