"""All-slice full-size parity for BASELINE configs[3] (Qwen-3-0.6B proxy ->
Qwen-3-32B target, d 128 proxy heads, 28 -> 64 layer pairing, N = 65536) and
configs[2] (Qwen-2.5-0.5B -> 7B, GQA 7, 24 -> 28 pairing, N = 131072), rho = 0.2:
the GPU pruner's mapped scores Ŷ on every (target layer, head) slice (512 / 112)
against the fp64 oracle mapper run on the GPU's own scores X.

The oracle side takes 30-55 min on 8 cores and its output (50-59 MB) is not
committed, so it is produced off the box and shipped with the repo snapshot:
  1. python tools/fullsize_dump.py --config CFG --x-only     (GPU: X)
  2. python tools/fullsize_oracle_cfg.py DIR --config CFG    (CPU: oracle Ŷ)
  3. copy DIR/oracle_y_f32.npy and DIR/x.sha256 to gpurun_in/fullsize_CFG/
The test skips when that fixture is absent (the driver's round-end run). It
checks that the GPU recomputes the same X (sha256 of its bytes: the scoring
kernels are deterministic), then norm-wise rel <= 1e-3 per slice and the Top-K
index overlap between the GPU's select on Ŷ and the oracle select
on the oracle Ŷ: mean >= 0.999, min reported (and written to
gpurun_out/fullsize_CFG_summary.txt)."""
import hashlib
import math
import os

import numpy as np
import pytest

from oracle import pkv_oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _fix(cfg):
    return os.path.join(ROOT, "gpurun_in", f"fullsize_{cfg}")


@pytest.mark.parametrize("cfg", ["qwen3_64k", "qwen25_128k"])
@pytest.mark.parametrize("prec", [3, 6])
def test_fullsize_all_slices(gpu, cfg, prec):
    """prec 3 (FP16X3, the default) must hold the bars; prec 6 (e4m3 corrections) is
    measured for the precision table and held to the rel bar only."""
    import torch
    import bench
    import paper_2605_16360_b200 as P
    fix = _fix(cfg)
    if not os.path.exists(os.path.join(fix, "oracle_y_f32.npy")):
        pytest.skip("oracle fixture not shipped (tools/fullsize_oracle_cfg.py)")
    c = bench.CONFIGS[cfg]
    geom = P.ModelGeometry(c["Ll"], c["Hl"], c["Ls"], c["Hs"], c["dt"])
    m = P.Mapper(geom, P.MapperConfig(), seed=7, precision=prec, ctx=gpu)
    pr = P.Pruner(m, c["Hq"], c["dp"], c["dt"], c["N"], c["rho"])
    q, kp, kt, vt = bench.make_inputs(c, torch.device("cuda"), 1234)
    K = pr.k
    assert K == math.ceil(c["rho"] * c["N"])
    ko = torch.empty(c["Ll"], c["Hl"], K, c["dt"], dtype=torch.bfloat16, device="cuda")
    vo = torch.empty_like(ko)
    idx = torch.empty(c["Ll"], c["Hl"], K, dtype=torch.int32, device="cuda")
    yhat = torch.empty(c["Ll"], c["Hl"], c["N"], device="cuda")
    pr.run(q, kp, kt, vt, ko, vo, idx, yhat)
    x = P.score(q, kp, ctx=gpu)
    torch.cuda.synchronize()
    want_sha = open(os.path.join(fix, "x.sha256")).read().strip()
    assert hashlib.sha256(x.cpu().numpy().tobytes()).hexdigest() == want_sha, "GPU scores X differ from the dump"
    del q, kp, kt, vt, ko, vo
    oracle = np.load(os.path.join(fix, "oracle_y_f32.npy"))  # [L_s, H_l, N], one row per proxy layer
    og = O.Geometry(c["Ll"], c["Hl"], c["Ls"], c["Hs"], c["dt"])
    # the GPU's own select on its Ŷ (all 512 slices) -> retained masks
    mask_g, _ = P.topk_select(yhat.reshape(c["Ll"] * c["Hl"], c["N"]), K, ctx=gpu)
    mask_g = mask_g.cpu().numpy().reshape(c["Ll"], c["Hl"], c["N"])
    y = yhat.cpu().numpy()
    rel, ov = [], []
    for ll in range(1, c["Ll"] + 1):
        w = oracle[O.layer_pair(ll, og) - 1]
        g = y[ll - 1].astype(np.float64)
        rel.append(np.linalg.norm(g - w, axis=1) / np.linalg.norm(w.astype(np.float64), axis=1))
        om, _ = O.topk_select(w, K)
        ov.append(O.topk_overlap_per_slice(mask_g[ll - 1], om, K))
    rel, ov = np.concatenate(rel), np.concatenate(ov)
    line = (f"{cfg} mapper precision {prec}: {rel.size} slices; mapped-score norm-rel max {rel.max():.2e} "
            f"mean {rel.mean():.2e}; Top-K overlap mean {ov.mean():.5f} min {ov.min():.5f}; slices below 0.999: {(ov < 0.999).sum()}")
    print(line)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"fullsize_{cfg}_summary.txt"), "a") as f:
        f.write(line + "\n")
    assert rel.max() <= 1e-3
    if prec == 3:
        assert ov.mean() >= 0.999
