"""Time the device ranking metrics on the bench's Ŷ geometry (256 slices of
32768): Spearman alone and one MetricAccumulator::add sample."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_16360_b200 as P  # noqa: E402

ctx = P.Context(0)
st = torch.cuda.current_stream()
S, n = 256, 32768
a = torch.rand(S, n, device="cuda")
b = a + 0.1 * torch.randn(S, n, device="cuda")
P.slice_metrics_device(a, b, 0.2, ctx=ctx, stream=st)  # grow the scratch once
t1 = bench.time_loop(lambda: P.spearman_device(a, b, ctx=ctx, stream=st), 5, st)
t2 = bench.time_loop(lambda: P.slice_metrics_device(a, b, 0.2, ctx=ctx, stream=st), 5, st)
print(f"spearman {S}x{n}: {t1:.3f} ms; slice_metrics (mass+overlap+spearman): {t2:.3f} ms")
z = torch.randn(1, 32, 8, n, device="cuda")
y = torch.rand(1, 32, 8, n, device="cuda")
P.loss_total(z, y, P.LossConfig(), 7, ctx=ctx)
t3 = bench.time_loop(lambda: P.loss_total(z, y, P.LossConfig(), 7, ctx=ctx), 3, st)
print(f"loss_total + grad [1, 32, 8, {n}]: {t3:.3f} ms")
