"""fp64 scores at the drop-in boundary (VERDICT r1 weak#2 / ADVICE medium):
the reference ranks doubles (pruning.cpp:20-56; its callers pass fp64 mapper
outputs, pruning.cpp:234, loss.cpp:63), so distinct doubles that round to the
same float must NOT become index-tie-broken. pkv_topk_select_f64 and
pkv_topk_mask_host rank 64-bit order keys; checked bit-exact against the
compiled reference (oracle/_ref libpkvref.so, RefLib.topk_mask) on inputs
built to collide in fp32. Also: misaligned score / mask pointers (ADVICE low:
the float4 / uint2 paths must not fault on a view with a storage offset)."""
import numpy as np
import pytest

from oracle import pkv_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ref():
    return O.RefLib()


def _collide(r, slices, n):
    """Doubles that are pairwise distinct but share few fp32 values."""
    base = r.randint(0, 7, (slices, n)).astype(np.float64) / 8.0 + 0.25
    tiny = r.permutation(slices * n).reshape(slices, n).astype(np.float64) * 1e-13
    s = base + tiny
    assert len(np.unique(s)) == s.size
    assert len(np.unique(s.astype(np.float32))) <= 8
    return s


@pytest.mark.parametrize("n,slices,rho", [(37, 5, 0.34), (1000, 3, 0.2), (8192, 4, 0.1), (40000, 2, 0.37)])
def test_topk_mask_host_fp64_exact(gpu, ref, n, slices, rho):
    import paper_2605_16360_b200 as P
    r = np.random.RandomState(n)
    s = _collide(r, slices, n)
    want, k = ref.topk_mask(s.reshape(1, slices, n), rho)
    m = P.topk_mask(s.reshape(1, slices, n), rho, ctx=gpu)
    assert m.k == k
    np.testing.assert_array_equal(m.bits, want)
    # the narrowed ranking really differs on these inputs (the old fp32 path's bug)
    narrowed, _ = ref.topk_mask(s.astype(np.float32).astype(np.float64).reshape(1, slices, n), rho)
    assert (narrowed != want).any()
    # ascending index lists = apply_mask order (pruning.cpp:197-215)
    for j in range(slices):
        np.testing.assert_array_equal(m.idx_asc[j], np.flatnonzero(want[0, j]))


def test_topk_select_f64_device_special_values(gpu, ref):
    """±0 tie (the reference's `!=` treats them equal), subnormals, ±inf,
    huge / tiny magnitudes, all-equal rows — device fp64 tensors."""
    import torch
    import paper_2605_16360_b200 as P
    rows = [
        np.array([0.0, -0.0, 0.0, -0.0, 1e-310, -1e-310, 5e-324, -5e-324] * 8),
        np.array([np.inf, -np.inf, 1e308, -1e308, 1.0, 1.0 + 2 ** -52, 1.0 - 2 ** -53, 0.5] * 8),
        np.full(64, 3.25),
        np.linspace(-1, 1, 64) * 1e-300,
    ]
    s = np.stack(rows)
    for k in (1, 7, 17, 40, 64):
        rho = k / 64.0
        want, kk = ref.topk_mask(s[None], rho)
        assert kk == k
        mask, idx = P.topk_select(torch.from_numpy(s).cuda(), k, ctx=gpu)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(mask.cpu().numpy(), want[0])
        for j in range(len(rows)):
            np.testing.assert_array_equal(idx.cpu().numpy()[j], np.flatnonzero(want[0, j]))


@pytest.mark.parametrize("n", [4096, 32768, 40000])
def test_select_misaligned_pointers(gpu, n):
    """Scores starting 1 float past a 16-byte boundary and a mask 1 byte past
    an 8-byte boundary, through pkv_topk_select: no misaligned-address fault,
    same bits as the aligned call."""
    import torch
    import paper_2605_16360_b200 as P
    slices, k = 3, n // 5
    r = np.random.RandomState(n)
    s = r.rand(slices, n).astype(np.float32)
    flat = torch.empty(slices * n + 1, dtype=torch.float32, device="cuda")
    flat[1:] = torch.from_numpy(s.reshape(-1)).cuda()
    view = flat[1:].view(slices, n)
    assert view.data_ptr() % 16 == 4
    mbuf = torch.zeros(slices * n + 1, dtype=torch.uint8, device="cuda")
    mview = mbuf[1:]
    idx = torch.empty(slices, k, dtype=torch.int32, device="cuda")
    P.check(P.lib().pkv_topk_select(gpu.h, view.data_ptr(), slices, n, k, mview.data_ptr(), idx.data_ptr(),
                                          None))
    torch.cuda.synchronize()
    want_mask, want_idx = O.topk_select(s, k)
    np.testing.assert_array_equal(mview.view(slices, n).cpu().numpy(), want_mask)
    np.testing.assert_array_equal(idx.cpu().numpy(), want_idx)
