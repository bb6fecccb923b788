"""Time the encoder attention kernel alone at the mapper's Llama/32k shape
(496 windows x 2048 tokens, 8 heads of 64) through the test hook; run under
`ncu --metrics gpu__time_duration.sum` to isolate attn_kernel."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_16360_b200 as P  # noqa: E402

nwin = int(os.environ.get("NWIN", "124"))
Lw, heads = 2048, 8
D = 64 * heads
ctx = P.Context(0)
f = P.lib().pkv_test_attention
f.restype = ctypes.c_int
f.argtypes = [ctypes.c_void_p, ctypes.c_void_p] + [ctypes.c_int64] * 4 + [ctypes.c_void_p, ctypes.c_void_p]
qkv = torch.randn(nwin * Lw, 3 * D, device="cuda") * 1.5
out = torch.empty(nwin * Lw, D, device="cuda")
for _ in range(2):
    P.check(f(ctx.h, qkv.data_ptr(), nwin, Lw, D, heads, out.data_ptr(), None))
torch.cuda.synchronize()
print("ok", out.abs().mean().item())
