"""Ranking metrics on the device (metrics.cu) against
the reference's own topk_overlap_per_slice / captured_mass_per_slice
(oracle/_ref, compiled from proj/src/pruning.cpp): overlap bit-exact,
captured mass within 1e-12 relative (fp64 sums, different order)."""
import numpy as np
import pytest

from oracle import pkv_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("slices,n,rho", [(32, 2048, 0.2), (8, 32768, 0.1), (5, 1000, 0.5), (3, 7, 1.0)])
def test_overlap_and_captured_mass_vs_reference(gpu, slices, n, rho):
    import torch
    import paper_2605_16360_b200 as P
    ref = O.RefLib()
    r = np.random.RandomState(n)
    y = (np.floor(r.rand(slices, n) * 64) / 64).astype(np.float32)  # ties included
    pred = (y + r.standard_normal(y.shape).astype(np.float32) * 0.05).astype(np.float32)
    k = P.retention_count(rho, n)
    mp, _ = P.topk_select(torch.from_numpy(pred).cuda(), k, want_idx=False, ctx=gpu)
    mt, _ = P.topk_select(torch.from_numpy(y).cuda(), k, want_idx=False, ctx=gpu)
    ov = P.topk_overlap_device(mp, mt, k, ctx=gpu).cpu().numpy()
    cm = P.captured_mass_device(mp, torch.from_numpy(y).cuda(), k, ctx=gpu).cpu().numpy()
    rbits_p, _ = ref.topk_mask(pred.astype(np.float64), rho)
    rbits_t, _ = ref.topk_mask(y.astype(np.float64), rho)
    np.testing.assert_array_equal(mp.cpu().numpy(), rbits_p)
    ov_ref = O.topk_overlap_per_slice(rbits_p, rbits_t, k)
    np.testing.assert_array_equal(ov, ov_ref)
    cm_ref = ref.captured_mass_per_slice(rbits_p, k, y.astype(np.float64))
    np.testing.assert_allclose(cm, cm_ref, rtol=1e-12, atol=0)
