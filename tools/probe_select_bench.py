"""Select on the bench's own mapped scores (Llama/32k: 256 slices x 32768) vs
uniform random scores of the same shape: device time of the library's select
(C ABI, preallocated outputs, behind a spin kernel) and how concentrated the
rows are (keys in the top-12-bit bin holding the k-th key). The first timed
loop in the process reads ~45 % slow whatever the data (bench.py therefore
runs one untimed loop before timing the short stages)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_16360_b200 as P  # noqa: E402

c = bench.CONFIGS["llama32k"]
dev = torch.device("cuda", 0)
ctx = P.Context(0)
arm = bench.Arm(P, ctx, c, dev, "none", 1, 0, 3, 1234)
y = torch.empty(c["Ll"], c["Hl"], c["N"], device=dev)
arm.pr.run(arm.q, arm.kp, arm.kt, arm.vt, arm.ko, arm.vo, arm.idx, scores_out=y)
torch.cuda.synchronize()
K = arm.K
st = torch.cuda.current_stream()
S = c["Ll"] * c["Hl"]
mask = torch.empty(S, c["N"], dtype=torch.uint8, device=dev)
idx = torch.empty(S, K, dtype=torch.int32, device=dev)
r = torch.rand(S, c["N"], device=dev)
for name, s in (("uniform random", r), ("bench mapped scores", y.reshape(S, -1)), ("uniform random", r),
                ("bench mapped scores", y.reshape(S, -1)), ("bench scores, fresh copy", y.reshape(S, -1).clone())):
    s = s.contiguous()
    t = bench.time_loop(lambda: P.lib().pkv_topk_select(ctx.h, P.proxykv._ptr(s), S, c["N"], K, None,
                                                         P.proxykv._ptr(idx), P.proxykv._stream(st)), 20, st)
    u = s.cpu().numpy().view(np.uint32)
    key = np.where(u >> 31, ~u, u | 0x80000000).astype(np.uint32)
    top = key >> 20
    kth = np.sort(key, axis=1)[:, -K]
    inbin = (top == (kth >> 20)[:, None]).sum(axis=1)
    print(f"{name}: select {t * 1e3:.1f} us; keys in the k-th key's 12-bit bin per row: "
          f"median {int(np.median(inbin))}, max {int(inbin.max())} (of {c['N']})", flush=True)
