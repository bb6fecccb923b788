"""Runs the Top-K select a few times for ncu (PKV_SEL_N / PKV_SEL_K: row length and k;
default the bench's 256 x 32768, k = 6554)."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import paper_2605_16360_b200 as P  # noqa: E402

n = int(os.environ.get("PKV_SEL_N", "32768"))
k = int(os.environ.get("PKV_SEL_K", "6554"))
ctx = P.Context(0)
s = torch.rand(256, n, device="cuda")
for _ in range(3):
    P.topk_select(s, k, want_mask=False, ctx=ctx)
torch.cuda.synchronize()
