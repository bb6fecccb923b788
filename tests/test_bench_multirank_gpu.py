"""bench.py's N > 1 path end to end on a one-GPU box (functional, not a scaling
measurement): torchrun with two ranks sharing cuda:0 (PKV_BENCH_ONE_DEVICE=1,
gloo for the timing collectives). Checks the driver contract: exactly one JSON
line on stdout from rank 0, strong scaling over the layer-sharded context, one
per-rank record per rank."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_two_ranks_one_line(gpu):
    env = dict(os.environ, PKV_BENCH_ONE_DEVICE="1", PKV_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(ROOT, "bench.py"), "--gpus", "2",
           "--config", "tiny", "--steps", "2", "--warmup", "3", "--no-cpu-baseline", "--no-e2e", "--no-extras"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0
    assert [p["rank"] for p in d["per_rank"]] == [0, 1]
