"""Decode attention over the packed cache (decode.cu)
against a float64 torch softmax(q·Kᵀ·scale)·V of the same bf16 inputs
(fp32 math: per-head norm-wise relative error <= 1e-4), for GQA groups
1/2/4/8, head_dim 64/128 and split counts from 1 to many; and end to end:
decoding over the cache pkv_pruner_run compacted equals decoding over the
full cache restricted to the retained rows."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _ref(q, k, v, scale):
    import torch
    g = q.shape[1] // k.shape[1]
    kk = k.double().repeat_interleave(g, dim=1)
    vv = v.double().repeat_interleave(g, dim=1)
    s = torch.einsum("lhd,lhkd->lhk", q.double(), kk) * scale
    return torch.einsum("lhk,lhkd->lhd", torch.softmax(s, dim=-1), vv)


@pytest.mark.parametrize("L,hq,hkv,K,d", [(1, 32, 8, 6554, 128), (32, 32, 8, 300, 128), (2, 8, 8, 1000, 64),
                                          (3, 16, 2, 77, 128), (1, 14, 2, 4096, 64), (4, 4, 2, 1, 128)])
def test_packed_decode_vs_torch(gpu, L, hq, hkv, K, d):
    import torch
    import paper_2605_16360_b200 as P
    g = torch.Generator(device="cuda").manual_seed(K + d)
    q = (torch.randn(L, hq, d, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    k = torch.randn(L, hkv, K, d, device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn(L, hkv, K, d, device="cuda", generator=g).to(torch.bfloat16)
    o = P.packed_decode_attention(q, k, v, ctx=gpu)
    torch.cuda.synchronize()
    ref = _ref(q, k, v, 1.0 / d ** 0.5)
    rel = ((o.double() - ref).norm(dim=-1) / ref.norm(dim=-1)).max().item()
    assert rel <= 1e-4, rel


def test_decode_over_pruner_output(gpu):
    import torch
    import paper_2605_16360_b200 as P
    Ls, Hq, Hs, dp, Ll, Hl, dt, N, rho = 2, 4, 4, 64, 4, 8, 128, 2048, 0.2
    m = P.Mapper(P.ModelGeometry(Ll, Hl, Ls, Hs, dt), P.MapperConfig(), seed=7, precision=3, ctx=gpu)
    pr = P.Pruner(m, Hq, dp, dt, N, rho)
    g = torch.Generator(device="cuda").manual_seed(0)
    q = (torch.randn(Ls, Hq, N, dp, device="cuda", generator=g) * 0.35).to(torch.bfloat16)
    kp = torch.randn(Ls, Hs, N, dp, device="cuda", generator=g).to(torch.bfloat16)
    kt = torch.randn(Ll, Hl, N, dt, device="cuda", generator=g).to(torch.bfloat16)
    vt = torch.randn(Ll, Hl, N, dt, device="cuda", generator=g).to(torch.bfloat16)
    K = pr.k
    ko = torch.empty(Ll, Hl, K, dt, dtype=torch.bfloat16, device="cuda")
    vo = torch.empty_like(ko)
    idx = torch.empty(Ll, Hl, K, dtype=torch.int32, device="cuda")
    pr.run(q, kp, kt, vt, ko, vo, idx)
    qd = (torch.randn(Ll, 4 * Hl, dt, device="cuda", generator=g) * 0.5).to(torch.bfloat16)  # GQA 4 target heads
    o = P.packed_decode_attention(qd, ko, vo, ctx=gpu)
    torch.cuda.synchronize()
    gi = idx.long()[..., None].expand(-1, -1, -1, dt)
    ref = _ref(qd, torch.gather(kt, 2, gi), torch.gather(vt, 2, gi), 1.0 / dt ** 0.5)
    rel = ((o.double() - ref).norm(dim=-1) / ref.norm(dim=-1)).max().item()
    assert rel <= 1e-4, rel
