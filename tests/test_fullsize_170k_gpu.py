"""BASELINE configs[2] at its longest context, end to end (VERDICT r1
missing#2): Qwen-2.5-0.5B (24L, 14Q/2KV, d64) -> Qwen-2.5-7B (28L, 4KV, d128),
N = 170000 (166 mapper windows; the right-aligned tail window at 167952,
mapper.cpp:66-79, 344-377), rho = 0.2 (K = 34000), through pkv_pruner_run:
  * scoring: the pass-1 LSE of sampled queries over all 170000 keys vs the
    fp64 restatement;
  * mapper: the oracle mapper (numpy fp64, pinned to the reference's outputs)
    fed the GPU's X on the first two windows, the windows around the middle and
    the last three (the tail window and its regular neighbours) of 2 proxy
    layers, against the GPU's Ŷ for the target layers paired with them:
    norm-wise rel <= 1e-3 on every token those windows fully determine, and
    Top-K (K = 34000) overlap >= 99.9 % between the GPU Ŷ and the GPU Ŷ with
    those spans replaced by the oracle's values;
  * select + compaction: bit-exact vs the oracle restatement driven from the
    GPU's Ŷ on all 112 slices (indices) and 3 slices (packed K/V)."""
import numpy as np
import pytest

from oracle import pkv_oracle as O
from tests.test_sum_longctx_gpu import check_spans, oracle_windows

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _bits(t):
    import torch
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


@pytest.fixture(scope="module")
def run(gpu):
    import torch
    import bench
    import paper_2605_16360_b200 as P
    c = bench.CONFIGS["qwen25_170k"]
    geom = P.ModelGeometry(c["Ll"], c["Hl"], c["Ls"], c["Hs"], c["dt"])
    m = P.Mapper(geom, P.MapperConfig(), seed=7, ctx=gpu)
    pr = P.Pruner(m, c["Hq"], c["dp"], c["dt"], c["N"], c["rho"])
    q, kp, kt, vt = bench.make_inputs(c, torch.device("cuda"), 4321)
    K = pr.k
    assert K == 34000
    ko = torch.empty(c["Ll"], c["Hl"], K, c["dt"], dtype=torch.bfloat16, device="cuda")
    vo = torch.empty_like(ko)
    idx = torch.empty(c["Ll"], c["Hl"], K, dtype=torch.int32, device="cuda")
    yhat = torch.empty(c["Ll"], c["Hl"], c["N"], device="cuda")
    pr.run(q, kp, kt, vt, ko, vo, idx, yhat)
    x = P.score(q, kp, ctx=gpu)
    lse = P.score_lse(q, kp, ctx=gpu)
    torch.cuda.synchronize()
    return dict(c=c, q=q, kp=kp, kt=kt, vt=vt, ko=ko, vo=vo, idx=idx, yhat=yhat, x=x, lse=lse, K=K)


def test_170k_lse_sampled_queries(run):
    c = run["c"]
    g = c["Hq"] // c["Hs"]
    qb, kb = _bits(run["q"]), _bits(run["kp"])
    rs = np.random.RandomState(0)
    for l, h in [(0, 0), (23, 13)]:
        qi = np.sort(rs.choice(c["N"], 64, replace=False))
        want = O.score_lse(qb[l:l + 1, h:h + 1, qi], kb[l:l + 1, h // g:h // g + 1])
        got = run["lse"][l, h, qi].cpu().numpy()
        assert np.abs(got - want[0, 0]).max() < 2e-4


def test_170k_mapper_spans_and_topk(run):
    c = run["c"]
    N, K = c["N"], run["K"]
    offs = O.window_offsets(N, 2048, 1024)
    assert len(offs) == 166 and offs[-1] == 167952 and offs[-2] == 167936
    og = O.Geometry(c["Ll"], c["Hl"], c["Ls"], c["Hs"], c["dt"])
    mp = O.MapperParams.init(og, O.MapperConfig(), 7)
    x = run["x"].cpu().numpy().astype(np.float64)
    yhat = run["yhat"].cpu().numpy()
    wins = [0, 1, 82, 83, 163, 164, 165]
    worst, ovs = 0.0, []
    for ls in (1, 17):
        y_ref, ok = oracle_windows(x[ls - 1][None], mp, wins)
        assert ok[-1] and ok[0] and ok.sum() >= 5 * 1024
        for ll in range(1, c["Ll"] + 1):
            if O.layer_pair(ll, og) != ls:
                continue
            rel, ov = check_spans(yhat[ll - 1], y_ref[0], ok, K)
            worst = max(worst, rel)
            ovs.append(ov)
    ov = np.concatenate(ovs)
    print(f"qwen25_170k mapped-score norm-rel {worst:.2e} over {ok.sum()} tokens; Top-K overlap mean {ov.mean():.5f} "
          f"min {ov.min():.5f} ({len(ov)} slices)")
    assert worst <= 1e-3
    assert ov.min() >= 0.999


def test_170k_select_compaction_bit_exact(run):
    c = run["c"]
    N, K, S = c["N"], run["K"], c["Ll"] * c["Hl"]
    y = run["yhat"].cpu().numpy().reshape(S, N)
    _, oidx = O.topk_select(y, K)
    np.testing.assert_array_equal(run["idx"].view(S, K).cpu().numpy(), oidx)
    sl = [0, 55, 111]
    kt = _bits(run["kt"]).reshape(S, N, c["dt"])[sl]
    vt = _bits(run["vt"]).reshape(S, N, c["dt"])[sl]
    eko, evo = O.compact_kv(kt, vt, oidx[sl])
    np.testing.assert_array_equal(_bits(run["ko"]).reshape(S, K, c["dt"])[sl], eko)
    np.testing.assert_array_equal(_bits(run["vo"]).reshape(S, K, c["dt"])[sl], evo)
