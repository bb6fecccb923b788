"""Full-size scoring parity on every key: the GPU's Llama/32k scores X (both
tcgen05 passes, max-pooled over queries and the GQA group; the bench's inputs)
against an fp64 evaluation of the same bf16 Q/K over all 16 x 8 x 32768 keys —
torch float64 on the device, query chunk by query chunk (S = Q·Kᵀ/√d,
lse per query over all keys, max_q exp(S − lse)). Test infrastructure (the
fp64 reference), run once per change; the suite keeps sampled keys
(tests/test_fullsize_gpu.py).

    python tools/fullsize_x_fp64.py      -> one summary line
"""
import math
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2605_16360_b200 as P  # noqa: E402

c = bench.CONFIGS["llama32k"]
dev = torch.device("cuda", 0)
ctx = P.Context(0)
q, kp, _, _ = bench.make_inputs(c, dev, seed=1234)
x = P.score(q, kp, ctx=ctx).double()  # [L_s, H_s, N]
Ls, Hq, Hs, N, d = c["Ls"], c["Hq"], c["Hs"], c["N"], c["dp"]
g = Hq // Hs
ch = 2048
worst, worst_at, ssum = 0.0, None, 0.0
for l in range(Ls):
    for h in range(Hs):
        kk = kp[l, h].double()  # [N, d]
        xr = torch.full((N,), -math.inf, dtype=torch.float64, device=dev)
        for hh in range(h * g, (h + 1) * g):
            for q0 in range(0, N, ch):
                s = (q[l, hh, q0:q0 + ch].double() @ kk.T) / math.sqrt(d)  # [ch, N]
                s -= torch.logsumexp(s, dim=1, keepdim=True)
                xr = torch.maximum(xr, s.max(dim=0).values)
        xr = xr.exp()
        rel = ((x[l, h] - xr).abs() / xr).max().item()
        ssum += ((x[l, h] - xr).abs() / xr).sum().item()
        if rel > worst:
            worst, worst_at = rel, (l, h, int(((x[l, h] - xr).abs() / xr).argmax()))
    print(f"layer {l} done, worst so far {worst:.2e}", flush=True)
print(f"llama32k X (max-pooled, {Ls}x{Hs}x{N} keys) vs float64: max rel {worst:.2e} at (layer, kv head, key) {worst_at}; "
      f"mean rel {ssum / (Ls * Hs * N):.2e}")
