"""Top-K select (select.cu: register-cached one-CTA-per-slice radix select
up to 32768 keys, the L2-re-reading generic kernel beyond) bit-exact against
the oracle restatement of pruning.cpp:20-56 + 197-215 (mask bytes and
ascending indices) at every kernel boundary (256 / 512 / 1024 threads, 8
items x 4 tiles per thread, > 32768 generic) and odd sizes, on random,
tie-heavy (test_pruning.cpp:84-98's floor(8u)/8), all-equal, signed-zero,
single-bucket (every key in one 12-bit digit bucket) and mapper-logit rows.
(Written for the round-2 cluster-select experiment, see
profiles/r02_select_cluster_experiment.txt; kept as coverage of the default.)"""
import numpy as np
import pytest

from oracle import pkv_oracle as O

pytestmark = pytest.mark.gpu

NS = [1, 7, 8, 100, 8191, 8192, 8193, 16384, 16385, 24576, 32768, 40000, 65536, 98304, 131072, 170000, 262144]


def _rows(kind, slices, n, r):
    if kind == "uniform":
        return r.rand(slices, n).astype(np.float32)
    if kind == "ties":
        return (np.floor(r.rand(slices, n) * 8) / 8).astype(np.float32)
    if kind == "equal":
        return np.full((slices, n), 0.375, np.float32)
    if kind == "zeros":
        return np.where(r.rand(slices, n) < 0.5, np.float32(0.0), np.float32(-0.0)).astype(np.float32) + \
            (r.rand(slices, n) < 0.1).astype(np.float32) * np.float32(-1.0)
    if kind == "bucket":  # all keys share their top 12 bits, distinct below
        return (np.float32(1.0) + r.randint(0, 1 << 20, (slices, n)).astype(np.float32) * np.float32(2.0 ** -23))
    if kind == "logits":  # the mapper's output distribution
        return (r.standard_normal((slices, n)) * 0.08 - 0.05).astype(np.float32)
    raise ValueError(kind)


def _check(gpu, s, k):
    import torch
    import paper_2605_16360_b200 as P
    dev = torch.from_numpy(s).cuda()
    mask, idx = P.topk_select(dev, k, ctx=gpu)
    torch.cuda.synchronize()
    wm, wi = O.topk_select(s, k)
    np.testing.assert_array_equal(mask.cpu().numpy(), wm)
    np.testing.assert_array_equal(idx.cpu().numpy(), wi)


@pytest.mark.parametrize("n", NS)
@pytest.mark.parametrize("kind", ["uniform", "ties", "logits"])
def test_cluster_select_sizes(gpu, n, kind):
    r = np.random.RandomState(n % 1000 + len(kind))
    slices = 3 if n > 100000 else 5
    s = _rows(kind, slices, n, r)
    for k in sorted({1, max(1, n // 10), O.retention_count(0.2, n), max(1, n - 1), n}):
        _check(gpu, s, k)


@pytest.mark.parametrize("kind", ["equal", "zeros", "bucket"])
@pytest.mark.parametrize("n", [5000, 32768, 131072])
def test_cluster_select_degenerate_rows(gpu, kind, n):
    r = np.random.RandomState(n)
    s = _rows(kind, 2, n, r)
    for k in (1, n // 3, n):
        _check(gpu, s, k)


def test_cluster_select_idx_only_large_batch(gpu):
    """The pruner's call form (no mask) at 256 x 32768 (Llama / 32k)."""
    import torch
    import paper_2605_16360_b200 as P
    r = np.random.RandomState(0)
    s = _rows("logits", 256, 32768, r)
    k = O.retention_count(0.2, 32768)
    _, idx = P.topk_select(torch.from_numpy(s).cuda(), k, want_mask=False, ctx=gpu)
    torch.cuda.synchronize()
    _, wi = O.topk_select(s, k)
    np.testing.assert_array_equal(idx.cpu().numpy(), wi)
