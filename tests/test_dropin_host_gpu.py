"""The reference's own calling convention at the boundary (VERDICT r1
missing#4): host fp64 tensors in and out of forward_pair (with StageTrace),
sliding_forward, forward_full (mapper.hpp:111-126) and topk_indices /
topk_overlap (pruning.hpp:18, 41-42), through the C ABI's host forms, against
the oracle (oracle/pkv_oracle.py's fp64 mapper, pinned to the reference's own
outputs; the compiled reference's topk_mask / topk_overlap via RefLib)."""
import numpy as np
import pytest

from oracle import pkv_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mp(gpu):
    import paper_2605_16360_b200 as P
    g, cfg = (4, 8, 2, 4, 64), dict(encoder_layers=2)
    m = P.Mapper(P.ModelGeometry(*g), P.MapperConfig(**cfg), seed=3, ctx=gpu)
    o = O.MapperParams.init(O.Geometry(*g), O.MapperConfig(**cfg), 3)
    return m, o


def _rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def test_forward_pair_host_with_trace(mp):
    m, o = mp
    x = np.random.RandomState(0).uniform(0, 2, (2, 4, 700))
    tr, otr = {}, {}
    y = m.forward_pair_host(x, trace=tr)
    want = O.forward_pair(x, o, trace=otr)
    assert _rel(y, want) <= 1e-3
    a, wa = tr["cross_attention"], otr["cross_attention"]
    assert a.shape == wa.shape == (2, 700, 8, 4)
    assert np.abs(a - wa).max() <= 1e-4
    np.testing.assert_allclose(a.sum(-1), 1.0, atol=1e-5)


def test_forward_pair_device_trace_matches_host(mp):
    import torch
    m, _ = mp
    x = np.random.RandomState(1).uniform(0, 2, (1, 4, 2048)).astype(np.float32)
    tr = {}
    y = m.forward_pair(torch.from_numpy(x).cuda(), trace=tr)
    htr = {}
    yh = m.forward_pair_host(x.astype(np.float64), trace=htr)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(y.cpu().numpy().astype(np.float64), yh)
    np.testing.assert_array_equal(tr["cross_attention"].cpu().numpy().astype(np.float64), htr["cross_attention"])


def test_forward_pair_errors_mirror_reference(mp):
    import paper_2605_16360_b200 as P
    m, _ = mp
    with pytest.raises(P.PkvValueError, match="sliding_forward"):
        m.forward_pair_host(np.zeros((1, 4, 2049)))


def test_sliding_and_full_host(mp):
    m, o = mp
    r = np.random.RandomState(2)
    x = r.uniform(0, 2, (1, 4, 3500))
    np.testing.assert_array_less(_rel(m.sliding_forward_host(x), O.sliding_forward(x, o)), 1e-3)
    xa = r.uniform(0, 2, (1, 2, 4, 2600))
    ya = m.forward_full_host(xa)
    want = O.forward_full(xa, o)
    assert ya.shape == want.shape == (1, 4, 8, 2600)
    assert _rel(ya, want) <= 1e-3
    np.testing.assert_array_equal(ya[0, 0], ya[0, 1])  # layer_pair {1,1,2,2}: shared pairs bit-identical


def test_topk_indices_and_overlap_host(gpu):
    import paper_2605_16360_b200 as P
    ref = O.RefLib()
    r = np.random.RandomState(4)
    v = r.randint(0, 5, 3000) / 4.0 + r.permutation(3000) * 1e-14  # fp32-colliding doubles
    for k in (1, 600, 2999, 3000):
        bits, _ = ref.topk_mask(v[None, None], k / 3000.0)
        np.testing.assert_array_equal(P.topk_indices(v, k, ctx=gpu), np.flatnonzero(bits[0, 0]))
    with pytest.raises(P.PkvValueError, match="out of range"):
        P.topk_indices(v[:10], 11, ctx=gpu)
    a, _ = ref.topk_mask(r.rand(3, 500), 0.2)
    b, k = ref.topk_mask(r.rand(3, 500), 0.2)
    out = np.zeros(3)
    P.check(P.lib().pkv_topk_overlap_host(gpu.h, a.ctypes.data, b.ctypes.data, 3, 500, k, out.ctypes.data))
    np.testing.assert_array_equal(out, O.topk_overlap_per_slice(a, b, k))
