"""Proxy prefill attention with LSE output (prefill.cu).

* LSE against the fp64 oracle restatement of pass 1 (oracle/pkv_oracle.c
  score_lse, the same bf16 inputs): abs error <= 1e-4 (the X bar is rel 1e-3).
* O against a float64 torch softmax(Q·Kᵀ/√d)·V of the same bf16 inputs: the
  output is bf16 and P is bf16 before the P·V MMA, so per-row norm-wise
  relative error <= 1e-2.
* Scoring with the prefill's LSE (single pass) == scoring with its own LSE
  pass within rel 1e-3 (the north-star tolerance)."""
import numpy as np
import pytest

from oracle import pkv_oracle as O

pytestmark = pytest.mark.gpu

CASES = [(2, 4, 2, 300, 300, 64), (1, 8, 8, 1000, 1000, 128), (1, 2, 1, 200, 520, 64), (1, 14, 2, 640, 640, 64),
         (1, 16, 8, 129, 129, 128)]


def _inputs(L, hq, hkv, nq, nk, d, seed):
    import torch
    g = torch.Generator(device="cuda").manual_seed(seed)
    q = (torch.randn(L, hq, nq, d, device="cuda", generator=g) * 0.4).to(torch.bfloat16)
    k = torch.randn(L, hkv, nk, d, device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn(L, hkv, nk, d, device="cuda", generator=g).to(torch.bfloat16)
    return q, k, v


def _bits(t):
    import torch
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


@pytest.mark.parametrize("causal", [True, False])
@pytest.mark.parametrize("L,hq,hkv,nq,nk,d", CASES)
def test_prefill_lse_and_output(gpu, L, hq, hkv, nq, nk, d, causal):
    import torch
    import paper_2605_16360_b200 as P
    q, k, v = _inputs(L, hq, hkv, nq, nk, d, seed=nq + d)
    o, lse = P.proxy_prefill_attention(q, k, v, causal=causal, ctx=gpu)
    torch.cuda.synchronize()
    ref_lse = O.score_lse(_bits(q), _bits(k), causal=causal)
    err = np.abs(lse.cpu().numpy().astype(np.float64) - ref_lse).max()
    assert err <= 1e-4, err
    g = hq // hkv
    kk = k.double().repeat_interleave(g, dim=1)
    vv = v.double().repeat_interleave(g, dim=1)
    s = q.double() @ kk.transpose(-1, -2) / d ** 0.5
    if causal:
        off = nk - nq
        mask = torch.arange(nk, device="cuda")[None, :] > (torch.arange(nq, device="cuda")[:, None] + off)
        s = s.masked_fill(mask, float("-inf"))
    ref_o = torch.softmax(s, dim=-1) @ vv
    rel = ((o.double() - ref_o).norm(dim=-1) / ref_o.norm(dim=-1)).max().item()
    assert rel <= 1e-2, rel


@pytest.mark.parametrize("reduce", ["max", "sum"])
def test_single_pass_scoring_with_prefill_lse(gpu, reduce):
    import torch
    import paper_2605_16360_b200 as P
    q, k, v = _inputs(2, 8, 2, 700, 700, 64, seed=5)
    _, lse = P.proxy_prefill_attention(q, k, v, causal=True, want_out=False, ctx=gpu)
    x1 = P.score(q, k, reduce=reduce, causal=True, lse=lse, ctx=gpu)
    x2 = P.score(q, k, reduce=reduce, causal=True, ctx=gpu)
    torch.cuda.synchronize()
    a, b = x1.cpu().numpy().astype(np.float64), x2.cpu().numpy().astype(np.float64)
    rel = (np.linalg.norm(a - b, axis=-1) / np.linalg.norm(b, axis=-1)).max()
    assert rel <= 1e-3, rel
