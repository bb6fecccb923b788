"""Mapper encoder attention at one Llama/32k layer (496 windows x 2048 tokens,
8 heads of 64) through the test hook (which also converts the fp32 inputs and
outputs around the kernel). For the kernel alone run it under
    ncu --metrics gpu__time_duration.sum,smsp__cycles_elapsed.avg.per_second -k regex:attn_kernel
and compare with the MUFU ex2 bound this script prints for the clock ncu reports.

    PKV_ATTN_POLY=4 python tools/time_attn_clocked.py
"""
import ctypes
import os
import subprocess
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_16360_b200 as P  # noqa: E402

nwin, Lw, heads = 496, 2048, 8
D = 64 * heads
ctx = P.Context(0)
f = P.lib().pkv_test_attention
f.restype = ctypes.c_int
f.argtypes = [ctypes.c_void_p, ctypes.c_void_p] + [ctypes.c_int64] * 4 + [ctypes.c_void_p, ctypes.c_void_p]
qkv = torch.randn(nwin * Lw, 3 * D, device="cuda") * 1.5
out = torch.empty(nwin * Lw, D, device="cuda")
call = lambda: P.check(f(ctx.h, qkv.data_ptr(), nwin, Lw, D, heads, out.data_ptr(), None))
for _ in range(3):
    call()
torch.cuda.synchronize()
clk, stop = [], [False]


def sample():
    while not stop[0]:
        r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits"],
                           capture_output=True, text=True)
        try:
            clk.append(float(r.stdout.strip().split()[0]))
        except (ValueError, IndexError):
            pass
        time.sleep(0.05)


th = threading.Thread(target=sample)
th.start()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
n = 20
for _ in range(n):
    call()
b.record()
torch.cuda.synchronize()
stop[0] = True
th.join()
ms = a.elapsed_time(b) / n
mhz = sorted(clk)[len(clk) // 2] if clk else 0.0
exps = nwin * heads * Lw * Lw
poly = int(os.environ.get("PKV_ATTN_POLY", "4"))
mufu_share = 1.0 - poly / 16.0
bound_ms = exps * mufu_share / (16 * 148 * mhz * 1e6) * 1e3 if mhz else float("nan")
print(f"poly={poly}: {ms:.3f} ms per layer at {mhz:.0f} MHz; MUFU-only bound for the "
      f"{mufu_share:.2f} MUFU share {bound_ms:.3f} ms -> {bound_ms / ms:.0%}")
