"""GPU side of the all-slice full-size parity check (tools/fullsize_oracle.py):
scores X and mapped scores Ŷ of the bench's Llama/32k context (the same
inputs and mapper weights as tests/test_fullsize_gpu.py), saved as float32
.npy under gpurun_out/fullsize/ (16.8 + 33.6 MB).

    python tools/fullsize_dump.py [precision] [--no-x] [--x-only] [--config NAME]

--config picks another bench config (X only fits gpurun's 64 MiB return for
qwen3_64k: 58.7 MB; its Ŷ is compared on the box, tools/fullsize_compare_gpu.py)."""
import hashlib
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2605_16360_b200 as P  # noqa: E402

prec = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 3
cfg = sys.argv[sys.argv.index("--config") + 1] if "--config" in sys.argv else "llama32k"
c = bench.CONFIGS[cfg]
ctx = P.Context(0)
q, kp, _, _ = bench.make_inputs(c, torch.device("cuda"), 1234)
x = P.score(q, kp, ctx=ctx)  # [L_s, H_s, N]
out = os.path.join(ROOT, "gpurun_out", "fullsize" if cfg == "llama32k" else f"fullsize_{cfg}")
os.makedirs(out, exist_ok=True)
if "--x-only" in sys.argv:
    xs = x.cpu().numpy()
    np.save(os.path.join(out, "x.npy"), xs)
    print("saved", x.shape, "sha256", hashlib.sha256(xs.tobytes()).hexdigest())
    sys.exit(0)
geom = P.ModelGeometry(c["Ll"], c["Hl"], c["Ls"], c["Hs"], c["dt"])
m = P.Mapper(geom, P.MapperConfig(), seed=7, precision=prec, ctx=ctx)
y = torch.empty(1, c["Ll"], c["Hl"], c["N"], device="cuda")
m.forward_full(x[None], out=y)
torch.cuda.synchronize()
if "--no-x" not in sys.argv:  # gpurun copies back at most 64 MiB per call
    np.save(os.path.join(out, "x.npy"), x.cpu().numpy())
np.save(os.path.join(out, f"yhat_p{prec}.npy"), y[0].cpu().numpy())
print("saved", x.shape, y.shape)
