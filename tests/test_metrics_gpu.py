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


@pytest.mark.parametrize("slices,n", [(1, 2), (3, 7), (4, 513), (32, 2048), (8, 32768), (2, 131072)])
def test_spearman_vs_reference(gpu, slices, n):
    """spearman_per_slice (pruning.cpp:173-186) against the reference's own
    function: heavy ties, signed zeros, a constant slice; 1e-12 absolute (the
    device sums are exact integers, the reference's centred fp64 sums round)."""
    import torch
    import paper_2605_16360_b200 as P
    ref = O.RefLib()
    r = np.random.RandomState(n + slices)
    a = (np.floor(r.rand(slices, n) * 97) - 48).astype(np.float32)
    a[:, ::11] = -0.0
    b = (a + r.standard_normal(a.shape) * 20).astype(np.float32)
    if slices > 2:
        a[1] = 3.0          # constant vs varying -> 0
        a[2] = b[2] = 1.0   # both constant -> 1
    got = P.spearman_device(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), ctx=gpu).cpu().numpy()
    want = ref.spearman_per_slice(a.astype(np.float64), b.astype(np.float64))
    np.testing.assert_allclose(got, want, rtol=0, atol=1e-12)
    if slices > 2:
        assert got[1] == 0.0 and got[2] == 1.0


def test_spearman_rejects_short_rows(gpu):
    import torch
    import paper_2605_16360_b200 as P
    x = torch.zeros(3, 1, device="cuda")
    with pytest.raises(P.PkvValueError):
        P.spearman_device(x, x, ctx=gpu)


def test_metric_accumulator_vs_reference(gpu):
    """MetricAccumulator (pruning.cpp:218-275): per-sample work on the device,
    vs the reference's per-slice functions composed the same way."""
    import torch
    import paper_2605_16360_b200 as P
    ref = O.RefLib()
    rho, B, L, H, n = 0.25, 2, 3, 4, 1500
    r = np.random.RandomState(9)
    acc = P.MetricAccumulator(rho, ctx=gpu)
    sums = np.zeros((3, L * H))
    count = 0
    for _ in range(2):
        yt = (np.floor(r.rand(B, L, H, n) * 200) / 200).astype(np.float32)
        yp = (yt + r.standard_normal(yt.shape) * 0.1).astype(np.float32)
        acc.add(torch.from_numpy(yp).cuda(), torch.from_numpy(yt).cuda())
        k = P.retention_count(rho, n)
        pb, _ = ref.topk_mask(yp.astype(np.float64), rho)
        tb, _ = ref.topk_mask(yt.astype(np.float64), rho)
        m = ref.captured_mass_per_slice(pb, k, yt.astype(np.float64))
        o = O.topk_overlap_per_slice(pb, tb, k)
        s = ref.spearman_per_slice(yp.astype(np.float64), yt.astype(np.float64))
        for v, row in zip((m, o, s), sums):
            row += v.reshape(B, L * H).sum(axis=0)
        count += B
    rep = acc.report()
    per = sums / count
    np.testing.assert_allclose(rep.per_slice_mass, per[0], rtol=1e-12)
    np.testing.assert_allclose(rep.per_slice_overlap, per[1], rtol=0, atol=1e-15)
    np.testing.assert_allclose(rep.per_slice_spearman, per[2], rtol=0, atol=1e-12)
    assert rep.spearman == pytest.approx(per[2].mean(), abs=1e-12)
    assert rep.captured_mass == pytest.approx(per[0].mean(), rel=1e-12)
    with pytest.raises(P.ShapeError):
        acc.add(torch.zeros(2, 2, n, device="cuda"), torch.zeros(2, 2, n, device="cuda"))
