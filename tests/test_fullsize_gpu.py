"""Parity at the bench's full size (BASELINE configs[1]: Llama-3.2-1B proxy ->
Llama-3.1-8B target, N = 32768, rho = 0.2), through the same C ABI the bench
uses. The fp64 oracle cannot score 32k x 32k x 32 heads x 16 layers on CPU, so:
  * scoring: the pass-1 row LSE of 256 sampled queries (over all 32768 keys)
    against the fp64 restatement;
  * mapper + select: the oracle mapper (numpy fp64) on 2 of the 16 proxy
    layers, fed with the GPU's own scores X, against the GPU's mapped scores
    for the 4 target layers paired with them: norm-wise rel <= 1e-3 and Top-K
    (rho = 0.2, K = 6554) index overlap >= 99.9% (mean), min reported;
  * select + compaction at full size: bit-exact vs the oracle restatement
    driven from the GPU's Ŷ (all 256 slices);
  * configs[2] / [3] scoring at their full contexts (131072 keys with GQA 7;
    65536 keys at head_dim 128) on 2 proxy layers: sampled-query LSE vs the
    fp64 restatement and sampled-key X vs float64 over all queries."""
import numpy as np
import pytest

from oracle import pkv_oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def run(gpu):
    import torch
    import bench
    import paper_2605_16360_b200 as P
    c = bench.CONFIGS["llama32k"]
    geom = P.ModelGeometry(c["Ll"], c["Hl"], c["Ls"], c["Hs"], c["dt"])
    m = P.Mapper(geom, P.MapperConfig(), seed=7, ctx=gpu)
    pr = P.Pruner(m, c["Hq"], c["dp"], c["dt"], c["N"], c["rho"])
    q, kp, kt, vt = bench.make_inputs(c, torch.device("cuda"), 1234)
    K = pr.k
    ko = torch.empty(c["Ll"], c["Hl"], K, c["dt"], dtype=torch.bfloat16, device="cuda")
    vo = torch.empty_like(ko)
    idx = torch.empty(c["Ll"], c["Hl"], K, dtype=torch.int32, device="cuda")
    yhat = torch.empty(c["Ll"], c["Hl"], c["N"], device="cuda")
    pr.run(q, kp, kt, vt, ko, vo, idx, yhat)
    x = P.score(q, kp, ctx=gpu)  # the X the pruner mapped (same kernels, deterministic)
    lse = P.score_lse(q, kp, ctx=gpu)
    torch.cuda.synchronize()
    return dict(c=c, q=q, kp=kp, kt=kt, vt=vt, ko=ko, vo=vo, idx=idx, yhat=yhat, x=x, lse=lse, K=K)


def _bits(t):
    import torch
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def test_fullsize_lse_sampled_queries(run):
    c = run["c"]
    qb, kb = _bits(run["q"]), _bits(run["kp"])
    rs = np.random.RandomState(0)
    for l, h in [(0, 0), (7, 13), (15, 31)]:
        qi = np.sort(rs.choice(c["N"], 256, replace=False))
        want = O.score_lse(qb[l:l + 1, h:h + 1, qi], kb[l:l + 1, h // (c["Hq"] // c["Hs"]):h // (c["Hq"] // c["Hs"]) + 1])
        got = run["lse"][l, h, qi].cpu().numpy()
        assert np.abs(got - want[0, 0]).max() < 2e-4


def test_fullsize_x_sampled_keys_fp64_all_queries(run):
    """llama32k pooled X (max over the 4 query heads x 32768 queries of each KV
    head) at sampled keys vs a float64 evaluation over ALL queries (with the
    GPU's LSE, itself checked above against the fp64 restatement): rel 1e-3 of
    the slab's max; 3 (layer, KV head) slabs x 32 keys."""
    import torch
    c = run["c"]
    g, d, N = c["Hq"] // c["Hs"], c["dp"], c["N"]
    q, kp, x, lse = run["q"], run["kp"], run["x"], run["lse"]
    rs = np.random.RandomState(3)
    for l, kh in [(0, 0), (8, 3), (15, 7)]:
        qf = q[l, kh * g:(kh + 1) * g].double()
        ks = torch.from_numpy(np.sort(rs.choice(N, 32, replace=False))).cuda()
        kf = kp[l, kh, ks].double()
        s = torch.einsum("gnd,kd->gnk", qf, kf) / d ** 0.5 - lse[l, kh * g:(kh + 1) * g].double()[..., None]
        xw = torch.exp(s.amax(dim=(0, 1))).cpu().numpy()
        xg = x[l, kh, ks].double().cpu().numpy()
        scale = x[l, kh].max().item()
        err = np.abs(xg - xw).max() / scale
        print(f"llama32k X (layer {l}, kv head {kh}) sampled-key rel err {err:.2e}")
        assert err <= 1e-3


def test_fullsize_mapper_and_topk_overlap(run):
    c = run["c"]
    N, K = c["N"], run["K"]
    og = O.Geometry(c["Ll"], c["Hl"], c["Ls"], c["Hs"], c["dt"])
    mp = O.MapperParams.init(og, O.MapperConfig(), 7)
    x = run["x"].cpu().numpy().astype(np.float64)
    yhat = run["yhat"].cpu().numpy()
    worst, ovs = 0.0, []
    for ls in (1, 9):  # proxy layers; target layers 2ls-1, 2ls pair with them
        want = O.sliding_forward(x[ls - 1][None], mp)[0]  # [H_l, N]
        for ll in (2 * ls - 1, 2 * ls):
            assert O.layer_pair(ll, og) == ls
            got = yhat[ll - 1]
            nrm = (np.linalg.norm(got - want, axis=1) / np.linalg.norm(want, axis=1)).max()
            worst = max(worst, nrm)
            om, _ = O.topk_select(want.astype(np.float32), K)
            gm, _ = O.topk_select(got, K)
            ovs.append(O.topk_overlap_per_slice(gm, om, K))
    ov = np.concatenate(ovs)
    print(f"llama32k mapped-score norm-rel {worst:.2e}; Top-K overlap mean {ov.mean():.5f} min {ov.min():.5f}")
    assert worst <= 1e-3
    assert ov.mean() >= 0.999


def test_fullsize_select_compaction_bit_exact(run):
    c = run["c"]
    N, K, S = c["N"], run["K"], c["Ll"] * c["Hl"]
    y = run["yhat"].cpu().numpy().reshape(S, N)
    _, oidx = O.topk_select(y, K)
    np.testing.assert_array_equal(run["idx"].view(S, K).cpu().numpy(), oidx)
    sl = [0, 97, 255]  # gather checked on 3 of the 256 slices (full slices, all K rows)
    kt = _bits(run["kt"]).reshape(S, N, c["dt"])[sl]
    vt = _bits(run["vt"]).reshape(S, N, c["dt"])[sl]
    eko, evo = O.compact_kv(kt, vt, oidx[sl])
    np.testing.assert_array_equal(_bits(run["ko"]).reshape(S, K, c["dt"])[sl], eko)
    np.testing.assert_array_equal(_bits(run["vo"]).reshape(S, K, c["dt"])[sl], evo)


@pytest.mark.parametrize("name", ["qwen25_128k", "qwen3_64k"])
def test_fullsize_scoring_other_configs(gpu, name):
    """BASELINE configs[2] / [3] scoring at full context (GQA 7 at d 64 over
    131072 keys; d 128 over 65536 keys), 2 of the proxy layers: the pass-1 LSE
    of sampled queries vs the fp64 restatement, and the pooled X of sampled
    keys vs a float64 evaluation over ALL queries of the group (using the
    GPU's LSE, itself checked above): rel 1e-3 of the slab's max."""
    import torch
    import bench
    import paper_2605_16360_b200 as P
    c = dict(bench.CONFIGS[name])
    c["Ls"] = 2
    q, kp, _, _ = bench.make_inputs(dict(c, Ll=1, Hl=1, dt=8), torch.device("cuda"), 77)
    x = P.score(q, kp, ctx=gpu)
    lse = P.score_lse(q, kp, ctx=gpu)
    torch.cuda.synchronize()
    g, d, N = c["Hq"] // c["Hs"], c["dp"], c["N"]
    rs = np.random.RandomState(1)
    for l, kh in [(0, 0), (1, c["Hs"] - 1)]:
        qb = _bits(q[l, kh * g:(kh + 1) * g])
        kb = _bits(kp[l, kh:kh + 1])
        qi = np.sort(rs.choice(N, 48, replace=False))
        want = O.score_lse(qb[None, :1, qi], kb[None])[0, 0]
        got = lse[l, kh * g, qi].cpu().numpy()
        assert np.abs(got - want).max() < 2e-4, (name, np.abs(got - want).max())
        # X at sampled keys, float64 over every query of the group
        qf = q[l, kh * g:(kh + 1) * g].double()             # [g, N, d]
        ks = np.sort(rs.choice(N, 24, replace=False))
        kf = kp[l, kh, torch.from_numpy(ks).cuda()].double()  # [24, d]
        s = torch.einsum("gnd,kd->gnk", qf, kf) / d ** 0.5 - lse[l, kh * g:(kh + 1) * g].double()[..., None]
        xw = torch.exp(s.amax(dim=(0, 1))).cpu().numpy()
        xg = x[l, kh, torch.from_numpy(ks).cuda()].double().cpu().numpy()
        scale = x[l, kh].max().item()
        assert np.abs(xg - xw).max() <= 1e-3 * scale, (name, np.abs(xg - xw).max() / scale)
