"""End-to-end pruning at the head structure of every BASELINE.json config
(configs[2]-[4]) against the oracle pipeline (fp64 C scoring -> numpy fp64
mapper -> reference select): the same checks as tests/test_pruner_gpu.py on
the tiny config (mapped scores within rel 1e-3, Top-K overlap >= 99.9%,
select/compaction bit-exact from the GPU's own mapped scores).

Layer counts and the context are reduced so the fp64 oracle finishes in
seconds; everything that changes per config is kept: GQA group size (7 for
Qwen-2.5-0.5B, 2 for Qwen-3-0.6B), proxy head_dim (64 / 128), proxy and
target KV head counts (mapper conv-stem channels and stage-3 heads), target
head_dim 128, a context that is not a multiple of any tile and gets a
right-aligned tail window (mapper.cpp:66-79), and non-trivial layer pairing.
The full-N select/compaction sizes of these configs are covered in
tests/test_select_compact_gpu.py; Llama/32k at full size in
tests/test_fullsize_gpu.py."""
import numpy as np
import pytest

from oracle import pkv_oracle as O

pytestmark = pytest.mark.gpu

CASES = {
    # name: proxy (L_s, Hq, H_s, dp), target (L_l, H_l, dt), N, rho
    "qwen25_heads": ((2, 14, 2, 64), (3, 4, 128), 2600, 0.2),
    "qwen3_heads": ((2, 16, 8, 128), (5, 8, 128), 2300, 0.2),
    "sweep_rho10": ((2, 8, 4, 64), (4, 8, 128), 2200, 0.1),
    "sweep_rho50": ((2, 8, 4, 64), (4, 8, 128), 2200, 0.5),
}


def _bits(t):
    import torch
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


@pytest.mark.parametrize("name", sorted(CASES))
def test_config_end_to_end_vs_oracle(gpu, name):
    import torch
    import paper_2605_16360_b200 as P
    (Ls, Hq, Hs, dp), (Ll, Hl, dt), N, rho = CASES[name]
    geom = P.ModelGeometry(Ll, Hl, Ls, Hs, dt)
    m = P.Mapper(geom, P.MapperConfig(), seed=11, precision=3, ctx=gpu)
    pr = P.Pruner(m, Hq, dp, dt, N, rho)
    K = pr.k
    assert K == O.retention_count(rho, N)
    r = np.random.RandomState(len(name))
    q = r.standard_normal((Ls, Hq, N, dp)).astype(np.float32) * 0.35
    kp = r.standard_normal((Ls, Hs, N, dp)).astype(np.float32)
    u = r.standard_normal(dp).astype(np.float32)
    u /= np.linalg.norm(u)
    kp[:, :, : N // 50] += 3.0 * u  # attention-sink structure
    q += 0.8 * u
    qb, kpb = O.f32_to_bf16_bits(q), O.f32_to_bf16_bits(kp)
    kt = r.randint(0, 1 << 15, (Ll, Hl, N, dt)).astype(np.uint16)
    vt = r.randint(0, 1 << 15, (Ll, Hl, N, dt)).astype(np.uint16)
    dev = lambda a: torch.from_numpy(a.view(np.int16)).cuda().view(torch.bfloat16)
    ko = torch.empty(Ll, Hl, K, dt, dtype=torch.bfloat16, device="cuda")
    vo = torch.empty_like(ko)
    idx = torch.empty(Ll, Hl, K, dtype=torch.int32, device="cuda")
    yhat = torch.empty(Ll, Hl, N, device="cuda")
    pr.run(dev(qb), dev(kpb), dev(kt), dev(vt), ko, vo, idx, yhat)
    torch.cuda.synchronize()

    x = O.score(qb, kpb, reduce="max")
    mp = O.MapperParams.init(O.Geometry(Ll, Hl, Ls, Hs, dt), O.MapperConfig(), 11)
    y_ref = O.forward_full(x[None].astype(np.float64), mp)[0]
    y = yhat.cpu().numpy()
    nrm = (np.linalg.norm((y - y_ref).reshape(-1, N), axis=1) / np.linalg.norm(y_ref.reshape(-1, N), axis=1)).max()
    assert nrm <= 1e-3, nrm
    omask, _ = O.topk_select(y_ref.astype(np.float32), K)
    gmask = np.zeros((Ll * Hl, N), np.uint8)
    np.put_along_axis(gmask, idx.view(-1, K).cpu().numpy().astype(np.int64), 1, axis=1)
    ov = O.topk_overlap_per_slice(gmask, omask.reshape(-1, N), K)
    print(f"{name}: Top-K overlap mean {ov.mean():.5f} min {ov.min():.5f}; mapped-score norm-rel {nrm:.2e}")
    assert ov.mean() >= 0.999

    _, i2 = O.topk_select(y.reshape(-1, N), K)
    np.testing.assert_array_equal(idx.view(-1, K).cpu().numpy(), i2)
    eko, evo = O.compact_kv(kt.reshape(-1, N, dt), vt.reshape(-1, N, dt), i2)
    np.testing.assert_array_equal(_bits(ko).reshape(-1, K, dt), eko)
    np.testing.assert_array_equal(_bits(vo).reshape(-1, K, dt), evo)


@pytest.mark.parametrize("seed", range(6))
def test_random_geometry_end_to_end_vs_oracle(gpu, seed):
    """Randomised geometries (GQA 1/2/4/7, proxy / target head_dim 64/128,
    odd contexts with and without tail windows, max / sum pooling, causal or
    not, budgets 5-90 %) through pkv_pruner_run against the oracle pipeline:
    mapped scores within rel 1e-3, select + compaction bit-exact from the GPU's
    own mapped scores, Top-K overlap >= 99.9 %."""
    import torch
    import paper_2605_16360_b200 as P
    r = np.random.RandomState(1000 + seed)
    Hs = int(r.choice([1, 2, 4, 8]))
    g = int(r.choice([1, 2, 4, 7]))
    Ls = int(r.randint(1, 3))
    Ll = int(r.randint(Ls, 2 * Ls + 2))
    Hl = int(r.choice([2, 4, 8]))
    dp, dt = int(r.choice([64, 128])), int(r.choice([64, 128]))
    N = int(r.randint(300, 3200))
    rho = float(r.choice([0.05, 0.2, 0.37, 0.9]))
    reduce = "sum" if seed % 3 == 2 else "max"
    causal = seed % 2 == 1
    Hq = Hs * g
    geom = P.ModelGeometry(Ll, Hl, Ls, Hs, dt)
    cfg = P.MapperConfig(encoder_layers=2)
    m = P.Mapper(geom, cfg, seed=seed, ctx=gpu)
    pr = P.Pruner(m, Hq, dp, dt, N, rho, reduce=reduce, causal=causal)
    K = pr.k
    q = r.standard_normal((Ls, Hq, N, dp)).astype(np.float32) * 0.35
    kp = r.standard_normal((Ls, Hs, N, dp)).astype(np.float32)
    qb, kpb = O.f32_to_bf16_bits(q), O.f32_to_bf16_bits(kp)
    kt = r.randint(0, 1 << 15, (Ll, Hl, N, dt)).astype(np.uint16)
    vt = r.randint(0, 1 << 15, (Ll, Hl, N, dt)).astype(np.uint16)
    dev = lambda a: torch.from_numpy(a.view(np.int16)).cuda().view(torch.bfloat16)
    ko = torch.empty(Ll, Hl, K, dt, dtype=torch.bfloat16, device="cuda")
    vo = torch.empty_like(ko)
    idx = torch.empty(Ll, Hl, K, dtype=torch.int32, device="cuda")
    yhat = torch.empty(Ll, Hl, N, device="cuda")
    pr.run(dev(qb), dev(kpb), dev(kt), dev(vt), ko, vo, idx, yhat)
    torch.cuda.synchronize()
    x = O.score(qb, kpb, reduce=reduce, causal=causal)
    mp = O.MapperParams.init(O.Geometry(Ll, Hl, Ls, Hs, dt), O.MapperConfig(encoder_layers=2), seed)
    y_ref = O.forward_full(x[None].astype(np.float64), mp)[0]
    y = yhat.cpu().numpy()
    nrm = (np.linalg.norm((y - y_ref).reshape(-1, N), axis=1) / np.linalg.norm(y_ref.reshape(-1, N), axis=1)).max()
    desc = f"Ls={Ls} Hq={Hq} Hs={Hs} dp={dp} Ll={Ll} Hl={Hl} dt={dt} N={N} rho={rho} {reduce} causal={causal}"
    assert nrm <= 1e-3, (desc, nrm)
    omask, _ = O.topk_select(y_ref.astype(np.float32), K)
    gmask = np.zeros((Ll * Hl, N), np.uint8)
    np.put_along_axis(gmask, idx.view(-1, K).cpu().numpy().astype(np.int64), 1, axis=1)
    ov = O.topk_overlap_per_slice(gmask, omask.reshape(-1, N), K)
    print(f"{desc}: overlap mean {ov.mean():.5f} min {ov.min():.5f}; norm-rel {nrm:.2e}")
    assert ov.mean() >= 0.999, (desc, ov.mean())
    _, i2 = O.topk_select(y.reshape(-1, N), K)
    np.testing.assert_array_equal(idx.view(-1, K).cpu().numpy(), i2)
    eko, evo = O.compact_kv(kt.reshape(-1, N, dt), vt.reshape(-1, N, dt), i2)
    np.testing.assert_array_equal(_bits(ko).reshape(-1, K, dt), eko)
    np.testing.assert_array_equal(_bits(vo).reshape(-1, K, dt), evo)
