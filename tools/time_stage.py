"""Time one stage of the llama32k step in isolation (CUDA events), e.g.
   python tools/time_stage.py score_lse|score_pool|map|attn"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_16360_b200 as P  # noqa: E402

c = bench.CONFIGS[os.environ.get("PKV_CONFIG", "llama32k")]
ctx = P.Context(0)
q, kp, kt, vt = bench.make_inputs(c, torch.device("cuda"), 1)
stream = torch.cuda.current_stream()
for stage in sys.argv[1:]:
    if stage == "score_lse":
        f = lambda: P.score_lse(q, kp, ctx=ctx)
    elif stage == "score_pool":
        lse = P.score_lse(q, kp, ctx=ctx)
        f = lambda: P.score(q, kp, lse=lse, ctx=ctx)
    elif stage == "map":
        m = P.Mapper(P.ModelGeometry(c["Ll"], c["Hl"], c["Ls"], c["Hs"], c["dt"]), P.MapperConfig(), seed=7,
                     precision=int(os.environ.get("PKV_PREC", "3")), ctx=ctx)
        x = torch.rand(1, c["Ls"], c["Hs"], c["N"], device="cuda")
        f = lambda: m.forward_full(x)
    f()
    ms = bench.time_loop(f, 3, stream)
    print(f"{stage}: {ms:.2f} ms")
