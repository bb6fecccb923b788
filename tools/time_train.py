"""Time one GPU mapper training step (pkv_trainer forward + backward) at the
Llama-3.2-1B -> Llama-3.1-8B mapper geometry (D 512, 6 encoder layers, 8 heads,
H_s = H_l = 8), B windows of 2048 tokens, and print ms per step and the
GEMM-equivalent TFLOP/s (3x the forward's FLOPs).

    python tools/time_train.py [--B 2] [--iters 3]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2605_16360_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=2)
ap.add_argument("--n", type=int, default=2048)
ap.add_argument("--iters", type=int, default=3)
a = ap.parse_args()
geom = P.ModelGeometry(32, 8, 16, 8, 128)
cfg = P.MapperConfig()
ctx = P.Context(0)
tr = P.MapperTrainer(geom, cfg, seed=1, ctx=ctx)
x = torch.rand(a.B, 8, a.n, device="cuda")
dl = torch.randn(a.B, 8, a.n, dtype=torch.float64, device="cuda")
g = torch.zeros(tr.n_params, dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream()
for _ in range(2):
    tr.forward(x, stream=st)
    tr.backward(dl, grad=g, stream=st)
torch.cuda.synchronize()
e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
tf = tb = 0.0
for _ in range(a.iters):
    e0.record(st)
    tr.forward(x, stream=st)
    e1.record(st)
    tr.backward(dl, grad=g, stream=st)
    e2.record(st)
    torch.cuda.synchronize()
    tf += e0.elapsed_time(e1)
    tb += e1.elapsed_time(e2)
tf /= a.iters
tb /= a.iters
D, F, n = 512, 2048, a.n
fwd = a.B * (6 * (24 * n * D * D + 4 * n * n * D) + 2 * n * D * 768 + 2 * n * 8 * 3 * 256 + 4 * n * D * 8 * 64)
print(f"B={a.B} n={n}: forward {tf:.2f} ms, backward {tb:.2f} ms, step {tf + tb:.2f} ms "
      f"({3 * fwd / (tf + tb) / 1e9:.1f} TFLOP/s GEMM-equivalent, fp32)")
