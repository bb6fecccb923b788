"""The device loss suite (loss.cu) against the
reference's own loss_total and its tape's gradient (oracle/_ref, compiled from
proj/src/loss.cpp + ops.cpp): pair counts exact (same RNG streams, same
sampling, same filter), every term and the total within 1e-10 relative, the
gradient within 1e-10 of its max magnitude (fp64 both sides; only summation
order differs). Inputs are fp32-representable, with ties."""
import numpy as np
import pytest

from oracle import pkv_oracle as O

pytestmark = pytest.mark.gpu

FIELDS = ["bin", "mse", "fine", "global_", "cos", "weighted_bin", "weighted_mse", "weighted_fine",
          "weighted_global", "weighted_cos", "total", "s_max"]
COUNTS = ["fine_used", "fine_filtered", "global_used", "global_filtered", "cos_floor_hits"]


def _inputs(shape, seed):
    r = np.random.RandomState(seed)
    y = (np.floor(r.rand(*shape) * 97) / 97).astype(np.float32)  # ties
    z = (r.standard_normal(shape) * 1.5).astype(np.float32)
    return z, y


def _check(gpu, z, y, cfg, seed):
    import torch
    import paper_2605_16360_b200 as P
    rep, grad = P.loss_total(torch.from_numpy(z).cuda(), torch.from_numpy(y).cuda(), cfg, seed, ctx=gpu)
    want, wgrad = O.RefLib().loss_total(z.astype(np.float64), y.astype(np.float64), cfg, seed)
    for f in COUNTS:
        assert getattr(rep, f) == want[f], (f, getattr(rep, f), want[f])
    for f in FIELDS:
        w = want[f.rstrip("_")]
        assert getattr(rep, f) == pytest.approx(w, rel=1e-10, abs=1e-14), (f, getattr(rep, f), w)
    g = grad.cpu().numpy()
    scale = max(np.abs(wgrad).max(), 1e-300)
    assert np.abs(g - wgrad).max() <= 1e-10 * scale, np.abs(g - wgrad).max() / scale
    return rep


@pytest.mark.parametrize("shape,seed", [((2, 2, 3, 1000), 42), ((1, 1, 4), 3), ((3, 8, 64), 7), ((1, 2, 8192), 11)])
def test_loss_total_default_config_vs_reference(gpu, shape, seed):
    import paper_2605_16360_b200 as P
    z, y = _inputs(shape, seed)
    rep = _check(gpu, z, y, P.LossConfig(), seed)
    if shape[-1] >= 1000:
        assert rep.fine_used > 0 and rep.global_used > 0  # sampling paths (Fisher-Yates, Floyd) exercised


def test_loss_total_hand_built_case(gpu):
    """test_loss.cpp:276-287 on the device (topk_ratio_for_rank 0.5)."""
    import paper_2605_16360_b200 as P
    z = np.array([[[1.2, 0.3, -0.5, -1.0]]], np.float32)
    y = np.array([[[0.9, 0.4, 0.1, 0.0]]], np.float32)
    _check(gpu, z, y, P.LossConfig(topk_ratio_for_rank=0.5), 3)


def test_loss_total_all_pairs_and_large_cap(gpu):
    """max_pairs above the candidate count (every pair, in order) and a cap too
    large for the shared-memory tables (global-memory table path)."""
    import paper_2605_16360_b200 as P
    z, y = _inputs((2, 3, 300), 5)
    _check(gpu, z, y, P.LossConfig(max_pairs=100000), 5)
    z, y = _inputs((1, 2, 4096), 6)
    _check(gpu, z, y, P.LossConfig(max_pairs=20000), 6)


def test_loss_total_ablation_removes_terms_exactly(gpu):
    """A zero λ drops its term from the total and the gradient (loss.cpp:355-361)."""
    import paper_2605_16360_b200 as P
    z, y = _inputs((2, 2, 512), 9)
    for drop in ["lambda_fine", "lambda_global", "lambda_bin", "lambda_mse", "lambda_cos"]:
        cfg = P.LossConfig(**{drop: 0.0})
        _check(gpu, z, y, cfg, 9)


def test_loss_total_errors(gpu):
    import torch
    import paper_2605_16360_b200 as P
    x = torch.zeros(1, 4, device="cuda")
    with pytest.raises(P.PkvValueError, match="degenerate oracle"):
        P.loss_total(x, x, ctx=gpu)
    with pytest.raises(P.PkvValueError, match="nonnegative"):
        P.loss_total(x, x + 1, P.LossConfig(lambda_bin=-1.0), ctx=gpu)
    with pytest.raises(P.PkvValueError, match="ratio"):
        P.loss_total(x, x + 1, P.LossConfig(ratios=(0.5, 1.5)), ctx=gpu)
    with pytest.raises(P.ShapeError):
        P.loss_total(x, torch.zeros(1, 5, device="cuda"), ctx=gpu)
