"""Pins the reference-loss harness (oracle/_ref: loss.cpp + its tape, compiled
from the reference's sources) before it checks the device loss suite: the
reference's own known answers (test_loss.cpp:259-287) and a finite-difference
check of the gradient the harness reads back. CPU only."""
import numpy as np
import pytest

from oracle import pkv_oracle as O


class Cfg:  # loss.hpp LossConfig defaults
    lambda_mse, lambda_bin, lambda_fine, lambda_global, lambda_cos = 20.0, 10.0, 3.0, 2.0, 0.5
    ratios = (0.05, 0.1, 0.15, 0.2, 0.3, 0.4, 0.5)
    gamma, epsilon, mse_exponent, margin, clip_lo, clip_hi = 1.0, 0.1, 1.5, 1.0, 1.0, 5.0
    pair_filter_frac, topk_ratio_for_rank, max_pairs = 0.01, 0.2, 4096


def test_reference_loss_degenerate_oracle_raises():
    ref = O.RefLib()
    with pytest.raises(Exception, match="degenerate oracle"):
        ref.loss_total(np.zeros((1, 4)), np.zeros((1, 4)), Cfg(), 1)


def test_reference_loss_hand_built_case():
    """test_loss.cpp:276-287: y = [0.9, 0.4, 0.1, 0], z = [1.2, 0.3, -0.5, -1],
    topk_ratio_for_rank 0.5: the weighted terms compose the total."""
    ref = O.RefLib()
    c = Cfg()
    c.topk_ratio_for_rank = 0.5
    r, g = ref.loss_total(np.array([[[1.2, 0.3, -0.5, -1.0]]]), np.array([[[0.9, 0.4, 0.1, 0.0]]]), c, 3)
    assert r["s_max"] == 0.9
    parts = r["weighted_bin"] + r["weighted_mse"] + r["weighted_fine"] + r["weighted_global"] + r["weighted_cos"]
    assert r["total"] == pytest.approx(parts, rel=1e-12)
    # k = 2: one Top-K pair (< 2 used -> the fine term is 0 with used reported 0), 2 x 2 cross pairs
    assert r["fine_used"] == 0 and r["fine"] == 0.0 and r["global_used"] == 4
    assert np.isfinite(g).all() and np.abs(g).max() > 0


def test_reference_loss_gradient_finite_differences():
    """The gradient read back through the harness is the tape's: central
    differences of the reference total (fixed pair samples: the pairs depend
    on y and the seed only)."""
    ref = O.RefLib()
    r = np.random.RandomState(8)
    y = r.rand(2, 2, 8)
    z = r.uniform(-1, 1, (2, 2, 8))
    _, g = ref.loss_total(z, y, Cfg(), 99)
    h = 1e-6
    for idx in [(0, 0, 0), (0, 1, 3), (1, 0, 7), (1, 1, 5)]:
        zp, zm = z.copy(), z.copy()
        zp[idx] += h
        zm[idx] -= h
        fd = (ref.loss_total(zp, y, Cfg(), 99, False)[0]["total"] - ref.loss_total(zm, y, Cfg(), 99, False)[0]["total"]) / (2 * h)
        assert fd == pytest.approx(g[idx], rel=1e-5, abs=1e-8)
