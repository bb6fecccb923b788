"""Mapper precision modes at the bench's full size (llama32k): the GPU's own
scores X for 2 proxy layers through the GPU mapper in each mode vs the numpy
fp64 oracle mapper: norm-wise rel error and Top-K (rho 0.2) index overlap
(mean / min over the 4 paired target layers x 8 heads), plus mapper time.

    python tools/prec_overlap.py [modes...]      (default: 3 5)
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_16360_b200 as P  # noqa: E402
from oracle import pkv_oracle as O  # noqa: E402

modes = [int(a) for a in sys.argv[1:]] or [3, 5]
c = bench.CONFIGS["llama32k"]
ctx = P.Context(0)
q, kp, _, _ = bench.make_inputs(c, torch.device("cuda"), 1234)
x = P.score(q, kp, ctx=ctx)
geom = P.ModelGeometry(c["Ll"], c["Hl"], c["Ls"], c["Hs"], c["dt"])
og = O.Geometry(c["Ll"], c["Hl"], c["Ls"], c["Hs"], c["dt"])
mp = O.MapperParams.init(og, O.MapperConfig(), 7)
xn = x.cpu().numpy().astype(np.float64)
K = P.retention_count(c["rho"], c["N"])
want = {ls: O.sliding_forward(xn[ls - 1][None], mp)[0] for ls in (1, 9)}
st = torch.cuda.current_stream()
for prec in modes:
    m = P.Mapper(geom, P.MapperConfig(), seed=7, precision=prec, ctx=ctx)
    y = torch.empty(1, c["Ll"], c["Hl"], c["N"], device="cuda")
    m.forward_full(x[None], out=y)
    ms = bench.time_loop(lambda: m.forward_full(x[None], stream=st, out=y), 3, st)
    yy = y[0].cpu().numpy()
    worst, ovs = 0.0, []
    for ls in (1, 9):
        w = want[ls]
        for ll in (2 * ls - 1, 2 * ls):
            got = yy[ll - 1]
            worst = max(worst, (np.linalg.norm(got - w, axis=1) / np.linalg.norm(w, axis=1)).max())
            om, _ = O.topk_select(w.astype(np.float32), K)
            gm, _ = O.topk_select(got, K)
            ovs.append(O.topk_overlap_per_slice(gm, om, K))
    ov = np.concatenate(ovs)
    print(f"precision {prec}: mapper {ms:.1f} ms  norm-rel {worst:.2e}  Top-K overlap mean {ov.mean():.5f} "
          f"min {ov.min():.5f}", flush=True)
