"""Mapper forward_full at the bench's full size (Llama/32k scores X, one
context) in the given precision modes: device time per call (CUDA events,
3 iterations after a warm-up) — run under an ncu launch list to split it per
kernel.

    python tools/time_mapper_modes.py [modes...]      (default: 3 6)
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_16360_b200 as P  # noqa: E402

modes = [int(a) for a in sys.argv[1:]] or [3, 6]
c = bench.CONFIGS["llama32k"]
ctx = P.Context(0)
q, kp, _, _ = bench.make_inputs(c, torch.device("cuda"), 1234)
x = P.score(q, kp, ctx=ctx)
geom = P.ModelGeometry(c["Ll"], c["Hl"], c["Ls"], c["Hs"], c["dt"])
st = torch.cuda.current_stream()
for prec in modes:
    m = P.Mapper(geom, P.MapperConfig(), seed=7, precision=prec, ctx=ctx)
    y = torch.empty(1, c["Ll"], c["Hl"], c["N"], device="cuda")
    m.forward_full(x[None], out=y)
    ms = bench.time_loop(lambda: m.forward_full(x[None], stream=st, out=y), 3, st)
    print(f"precision {prec}: mapper {ms:.1f} ms", flush=True)
