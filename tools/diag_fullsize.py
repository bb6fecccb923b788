"""Diagnostic: where does the full-size mapper error come from (per window /
position)? Runs the GPU mapper on the GPU's own llama32k scores for one proxy
layer and the numpy oracle on the same X."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_16360_b200 as P  # noqa: E402
from oracle import pkv_oracle as O  # noqa: E402

c = bench.CONFIGS["llama32k"]
ctx = P.Context(0)
q, kp, kt, vt = bench.make_inputs(c, torch.device("cuda"), 1234)
x = P.score(q, kp, ctx=ctx)[0:1].contiguous()  # proxy layer 1: [1, H_s, N]
geom = P.ModelGeometry(2, c["Hl"], 1, c["Hs"], c["dt"])
og = O.Geometry(2, c["Hl"], 1, c["Hs"], c["dt"])
mp = O.MapperParams.init(og, O.MapperConfig(), 7)
xn = x.cpu().numpy().astype(np.float64)
print("X stats: min %.3e max %.3e mean %.3e" % (xn.min(), xn.max(), xn.mean()))
N = int(os.environ.get("DIAG_N", "6144"))
want = O.sliding_forward(xn[:, :, :N], mp)[0]
for prec in (3, 2):
    m = P.Mapper(geom, P.MapperConfig(), seed=7, precision=prec, ctx=ctx)
    y = m.sliding_forward(x[:, :, :N].contiguous()).cpu().numpy()[0]
    d = np.abs(y - want)
    print(f"prec {prec}: norm-rel {np.linalg.norm(y - want) / np.linalg.norm(want):.2e}; ref rms {np.sqrt((want**2).mean()):.3e} std {want.std():.3e}")
    for b in range(0, N, 1024):
        print(f"   tokens {b:6d}-{b + 1023:6d}: max|d| {d[:, b:b + 1024].max():.3e} mean|d| {d[:, b:b + 1024].mean():.3e}")
