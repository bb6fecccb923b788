"""Small pass-2 launch for ncu (Llama head structure, 4k context)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2605_16360_b200 as P  # noqa: E402
ctx = P.Context(0)
N = 4096
q = (torch.randn(1, 32, N, 64, device="cuda") * 0.35).to(torch.bfloat16)
k = torch.randn(1, 8, N, 64, device="cuda").to(torch.bfloat16)
lse = P.score_lse(q, k, ctx=ctx)
for _ in range(2):
    P.score(q, k, lse=lse, ctx=ctx)
torch.cuda.synchronize()
