"""GPU parity of Top-K select (+ ascending index lists) and KV compaction,
through the C ABI, against the reference's golden vectors and the oracle.
Bit-exact bar (integer / index / byte work)."""
import os

import numpy as np
import pytest

from oracle import pkv_oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pr():
    return np.load(os.path.join(GOLD, "pruning.npz"))


def _set_path(mode):
    import ctypes
    import paper_2605_16360_b200 as P
    f = P.lib().pkv_test_select_path
    f.restype, f.argtypes = ctypes.c_int, [ctypes.c_int]
    return f(mode)


# every test of this module runs on both select kernels, each forced at every
# size: the register-cached radix kernel (select.cu) and the streaming one with
# candidate compaction (select_stream.cu; the library's choice for rows longer
# than 32768 whose score tensor fits in L2)
@pytest.fixture(autouse=True, params=[0, 1], ids=["cached_radix", "streaming"])
def select_path(request):
    prev = _set_path(request.param)
    yield request.param
    _set_path(prev)


def _sel(scores_np, k, ctx):
    import torch
    import paper_2605_16360_b200 as P
    dev = torch.from_numpy(np.ascontiguousarray(scores_np, np.float32)).cuda()
    mask, idx = P.topk_select(dev, k, ctx=ctx)
    torch.cuda.synchronize()
    return mask.cpu().numpy(), idx.cpu().numpy()


def test_basic_and_errors(gpu, pr):
    import paper_2605_16360_b200 as P
    for name, want in [("basic", [0, 2]), ("basic_all", [0, 1, 2]), ("tie", [0]), ("loss_gt", [0, 2])]:
        m = P.topk_mask(pr[f"{name}_scores"].reshape(1, 1, -1), float(pr[f"{name}_rho"]))
        assert m.k == int(pr[f"{name}_k"])
        assert np.flatnonzero(m.bits).tolist() == want
        assert P.apply_mask(m, 128).retained[0].tolist() == want
    y = np.array([[[3.0, 1.0, 2.0]]])
    with pytest.raises(P.PkvValueError):
        P.topk_mask(y, 0.0)
    with pytest.raises(P.PkvValueError):
        P.topk_mask(y, 1.5)


def test_exhaustive_3pow8(gpu, pr):
    vecs = pr["exhaustive_vectors"]
    for k in range(1, 9):
        mask, idx = _sel(vecs, k, gpu)
        np.testing.assert_array_equal(mask, pr["exhaustive_bits"][k - 1])
        for r in (0, 100, 6560):
            assert idx[r].tolist() == np.flatnonzero(mask[r]).tolist()


def test_tie_heavy_1000(gpu, pr):
    for v, k, bits in zip(pr["ties_vectors"], pr["ties_k"], pr["ties_bits"]):
        mask, idx = _sel(v[None], int(k), gpu)
        np.testing.assert_array_equal(mask[0], bits)
        assert idx[0].tolist() == np.flatnonzero(bits).tolist()


def test_affine_invariance(gpu, pr):
    for v, a, c, bits in zip(pr["affine_vectors"], pr["affine_alpha"], pr["affine_c"], pr["affine_bits"]):
        k = O.retention_count(0.25, 16)
        m1, _ = _sel(v, k, gpu)
        m2, _ = _sel((a * v + c), k, gpu)
        np.testing.assert_array_equal(m1, bits)
        np.testing.assert_array_equal(m2, bits)


def test_apply_mask_bytes(gpu, pr):
    import paper_2605_16360_b200 as P
    m = P.topk_mask(pr["apply_big_scores"], 0.5)
    app = P.apply_mask(m, 128, 2)
    np.testing.assert_array_equal(app.retained[0], pr["apply_big_idx"][0])
    assert app.bytes_saved_per_head == 262144
    assert P.apply_mask(P.topk_mask(pr["apply_big_scores"], 1.0), 128, 2).bytes_saved_per_head == 0


def test_signed_zero_subnormal_allequal(gpu, pr):
    mask, idx = _sel(pr["rand_scores"], int(pr["rand_k"]), gpu)
    np.testing.assert_array_equal(mask, pr["rand_bits"])
    np.testing.assert_array_equal(idx.reshape(pr["rand_idx"].shape), pr["rand_idx"])


@pytest.mark.parametrize("slices,n,rho", [(256, 32768, 0.2), (112, 131072, 0.2), (4, 170000, 0.07), (3, 1, 1.0),
                                          (5, 4099, 0.5), (7, 12, 0.1), (2, 65536, 0.5)])
def test_vs_oracle_shapes(gpu, slices, n, rho):
    r = np.random.RandomState(n % 1000 + slices)
    s = r.uniform(0, 1, (slices, n)).astype(np.float32)
    if n > 8:
        s[0, : n // 3] = np.round(s[0, : n // 3] * 64) / 64  # ties
    k = O.retention_count(rho, n)
    mask, idx = _sel(s, k, gpu)
    omask, oidx = O.topk_select(s, k)
    np.testing.assert_array_equal(mask, omask)
    np.testing.assert_array_equal(idx, oidx)


def test_index_only_output(gpu):
    import torch
    import paper_2605_16360_b200 as P
    s = torch.rand(8, 5000, device="cuda")
    k = 1000
    _, idx = P.topk_select(s, k, want_mask=False, ctx=gpu)
    _, oidx = O.topk_select(s.cpu().numpy(), k)
    np.testing.assert_array_equal(idx.cpu().numpy(), oidx)


@pytest.mark.parametrize("S,n,k,d,dtype", [(256, 32768, 6554, 128, "bf16"), (8, 1000, 333, 64, "fp16"),
                                           (3, 50, 11, 4, "bf16"), (2, 77, 5, 3, "bf16")])
def test_compaction_bit_exact(gpu, S, n, k, d, dtype):
    import torch
    import paper_2605_16360_b200 as P
    g = torch.Generator(device="cuda").manual_seed(5)
    kin = torch.randint(0, 1 << 15, (S, n, d), device="cuda", dtype=torch.int32, generator=g).to(torch.int16)
    vin = torch.randint(0, 1 << 15, (S, n, d), device="cuda", dtype=torch.int32, generator=g).to(torch.int16)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float16
    kin, vin = kin.view(tdt), vin.view(tdt)
    scores = torch.rand(S, n, device="cuda", generator=g)
    _, idx = P.topk_select(scores, k, want_mask=False, ctx=gpu)
    ko, vo = P.compact_kv(kin, vin, idx, ctx=gpu)
    torch.cuda.synchronize()
    kb, vb = kin.view(torch.int16).cpu().numpy().view(np.uint16), vin.view(torch.int16).cpu().numpy().view(np.uint16)
    eko, evo = O.compact_kv(kb, vb, idx.cpu().numpy())
    np.testing.assert_array_equal(ko.view(torch.int16).cpu().numpy().view(np.uint16), eko)
    np.testing.assert_array_equal(vo.view(torch.int16).cpu().numpy().view(np.uint16), evo)


@pytest.mark.parametrize("S,n,rho,d,kind", [(256, 32768, 0.2, 128, "uniform"), (16, 20000, 0.1, 64, "ties"),
                                            (3, 8193, 0.5, 128, "allequal"), (5, 4099, 0.3, 64, "signed0"),
                                            (2, 170000, 0.2, 128, "logits"), (4, 1000, 0.2, 64, "uniform"),
                                            (9, 16387, 0.37, 8, "ties"),
                                            # budget-sweep rows, one slice per co-resident CTA and beyond
                                            (256, 8192, 0.1, 128, "uniform"), (256, 16384, 0.1, 128, "logits"),
                                            (296, 4096, 0.5, 128, "ties"), (7, 100, 1.0, 16, "uniform"),
                                            (40, 3000, 0.01, 24, "signed0"),
                                            (600, 2048, 0.2, 64, "uniform")])
def test_select_compact(gpu, S, n, rho, d, kind):
    """pkv_select_compact == oracle select + oracle gather, bit for bit (indices and packed rows)."""
    import torch
    import paper_2605_16360_b200 as P
    r = np.random.RandomState(S * 7 + n)
    if kind == "uniform":
        s = r.uniform(0, 1, (S, n))
    elif kind == "ties":
        s = np.floor(r.uniform(0, 8, (S, n))) / 8
    elif kind == "allequal":
        s = np.full((S, n), 0.25)
    elif kind == "signed0":
        s = r.choice([0.0, -0.0, 1e-40, -1e-40, 1.0, -1.0], (S, n))
    else:
        s = r.standard_normal((S, n)) * 3
    s = s.astype(np.float32)
    k = O.retention_count(rho, n)
    g = torch.Generator(device="cuda").manual_seed(n)
    kin = torch.randint(-(1 << 15), 1 << 15, (S, n, d), device="cuda", dtype=torch.int32, generator=g).to(torch.int16)
    vin = torch.randint(-(1 << 15), 1 << 15, (S, n, d), device="cuda", dtype=torch.int32, generator=g).to(torch.int16)
    idx, ko, vo = P.select_compact(torch.from_numpy(s).cuda(), kin, vin, k, ctx=gpu)
    torch.cuda.synchronize()
    _, oidx = O.topk_select(s, k)
    np.testing.assert_array_equal(idx.cpu().numpy(), oidx)
    kb, vb = kin.cpu().numpy().view(np.uint16), vin.cpu().numpy().view(np.uint16)
    eko, evo = O.compact_kv(kb, vb, oidx)
    np.testing.assert_array_equal(ko.cpu().numpy().view(np.uint16), eko)
    np.testing.assert_array_equal(vo.cpu().numpy().view(np.uint16), evo)


def test_repeated_calls_and_offset_views(gpu):
    """Many calls of changing geometry in a row, misaligned (storage-offset) score
    pointers (scalar-load paths), all vs the oracle."""
    import torch
    import paper_2605_16360_b200 as P
    r = np.random.RandomState(3)
    for it, (S, n) in enumerate([(4, 9000), (64, 32768), (4, 9000), (1, 70001), (300, 4096), (4, 9000)]):
        s = r.uniform(0, 1, (S, n)).astype(np.float32)
        k = O.retention_count(0.2 + 0.05 * it, n)
        big = torch.zeros(S * n + 3, device="cuda")
        view = big[1:1 + S * n].view(S, n)  # 4-byte aligned only
        view.copy_(torch.from_numpy(s).cuda())
        mask, idx = P.topk_select(view, k, ctx=gpu)
        omask, oidx = O.topk_select(s, k)
        np.testing.assert_array_equal(mask.cpu().numpy(), omask)
        np.testing.assert_array_equal(idx.cpu().numpy(), oidx)


def test_select_compact_two_streams_repeated(gpu):
    """pkv_select_compact called many times on two streams with changing geometry
    (register-cached and streaming selects, several row widths): every call vs the oracle."""
    import torch
    import paper_2605_16360_b200 as P
    r = np.random.RandomState(11)
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = []
    for it, (S, n, d) in enumerate([(64, 8192, 128), (256, 4096, 64), (3, 16384, 128), (64, 8192, 128),
                                    (128, 12000, 8), (256, 4096, 64)] * 2):
        s = r.uniform(0, 1, (S, n)).astype(np.float32)
        k = O.retention_count(0.1 + 0.07 * (it % 6), n)
        st = streams[it % 2]
        with torch.cuda.stream(st):
            sc = torch.from_numpy(s).to("cuda", non_blocking=False)
            kin = torch.randint(-(1 << 15), 1 << 15, (S, n, d), device="cuda", dtype=torch.int32).to(torch.int16)
            vin = torch.randint(-(1 << 15), 1 << 15, (S, n, d), device="cuda", dtype=torch.int32).to(torch.int16)
            idx, ko, vo = P.select_compact(sc, kin, vin, k, ctx=gpu, stream=st)
        outs.append((s, k, kin, vin, idx, ko, vo, st))
    torch.cuda.synchronize()
    for s, k, kin, vin, idx, ko, vo, st in outs:
        _, oidx = O.topk_select(s, k)
        np.testing.assert_array_equal(idx.cpu().numpy(), oidx)
        eko, evo = O.compact_kv(kin.cpu().numpy().view(np.uint16), vin.cpu().numpy().view(np.uint16), oidx)
        np.testing.assert_array_equal(ko.cpu().numpy().view(np.uint16), eko)
        np.testing.assert_array_equal(vo.cpu().numpy().view(np.uint16), evo)
