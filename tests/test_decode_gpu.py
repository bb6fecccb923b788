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


def _to_pages(k, page, perm_seed):
    """Scatter a packed [L, Hkv, K, d] cache into a shuffled page pool."""
    import torch
    L, hkv, K, d = k.shape
    nb = (K + page - 1) // page
    npages = L * hkv * nb
    g = torch.Generator().manual_seed(perm_seed)
    perm = torch.randperm(npages + 5, generator=g)[:npages].to(torch.int32)  # spare pages unused
    table = perm.view(L, hkv, nb)
    pool = torch.zeros(npages + 5, page, d, dtype=k.dtype, device=k.device)
    for s in range(L * hkv):
        rows = k.view(L * hkv, K, d)[s]
        for b in range(nb):
            r0, r1 = b * page, min(K, (b + 1) * page)
            pool[int(table.view(-1, nb)[s, b]), : r1 - r0] = rows[r0:r1]
    return pool, table.cuda()


@pytest.mark.parametrize("L,hq,hkv,K,d,page", [(2, 32, 8, 700, 128, 16), (1, 14, 2, 4096, 64, 64),
                                               (3, 8, 8, 77, 64, 32)])
def test_paged_decode_equals_packed(gpu, L, hq, hkv, K, d, page):
    """Same rows in a shuffled page pool decode like the packed cache (same
    splits and key order; the in-CTA merge uses shared-memory float atomics,
    so agreement is to rounding, not bits)."""
    import torch
    import paper_2605_16360_b200 as P
    g = torch.Generator(device="cuda").manual_seed(K)
    q = (torch.randn(L, hq, d, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    k = torch.randn(L, hkv, K, d, device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn(L, hkv, K, d, device="cuda", generator=g).to(torch.bfloat16)
    kp, table = _to_pages(k, page, 1)
    vp, _ = _to_pages(v, page, 1)
    lens = torch.full((L, hkv), K, dtype=torch.int32, device="cuda")
    o1 = P.packed_decode_attention(q, k, v, ctx=gpu)
    o2 = P.paged_decode_attention(q, kp, vp, table, lens, ctx=gpu)
    torch.cuda.synchronize()
    torch.testing.assert_close(o2, o1, rtol=1e-5, atol=1e-6)


def test_paged_decode_variable_lengths_vs_torch(gpu):
    """Per-(layer, KV head) lengths (incl. 0 and 1) against float64 torch."""
    import torch
    import paper_2605_16360_b200 as P
    L, hq, hkv, d, page, Kmax = 2, 16, 4, 128, 32, 1000
    g = torch.Generator(device="cuda").manual_seed(3)
    q = (torch.randn(L, hq, d, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    k = torch.randn(L, hkv, Kmax, d, device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn(L, hkv, Kmax, d, device="cuda", generator=g).to(torch.bfloat16)
    lens = torch.tensor([[1000, 0, 1, 333], [64, 65, 999, 7]], dtype=torch.int32)
    kp, table = _to_pages(k, page, 2)
    vp, _ = _to_pages(v, page, 2)
    o = P.paged_decode_attention(q, kp, vp, table, lens.cuda(), ctx=gpu)
    torch.cuda.synchronize()
    grp = hq // hkv
    for l in range(L):
        for kh in range(hkv):
            n = int(lens[l, kh])
            got = o[l, kh * grp:(kh + 1) * grp]
            if n == 0:
                assert torch.count_nonzero(got) == 0
                continue
            ref = _ref(q[l:l + 1, kh * grp:(kh + 1) * grp], k[l:l + 1, kh:kh + 1, :n], v[l:l + 1, kh:kh + 1, :n],
                       1.0 / d ** 0.5)[0]
            rel = ((got.double() - ref).norm(dim=-1) / ref.norm(dim=-1)).max().item()
            assert rel <= 1e-4, (l, kh, n, rel)


def test_compact_into_pages_equals_packed(gpu):
    """pkv_compact_kv_paged writes exactly the packed gather, page by page."""
    import torch
    import paper_2605_16360_b200 as P
    S, n, d, k, page = 6, 2048, 128, 410, 16
    g = torch.Generator(device="cuda").manual_seed(5)
    kin = torch.randn(S, n, d, device="cuda", generator=g).to(torch.bfloat16)
    vin = torch.randn(S, n, d, device="cuda", generator=g).to(torch.bfloat16)
    idx = torch.sort(torch.stack([torch.randperm(n, device="cuda")[:k] for _ in range(S)]), dim=1).values.to(torch.int32)
    ko, vo = P.compact_kv(kin, vin, idx, ctx=gpu)
    nb = (k + page - 1) // page
    table = torch.randperm(S * nb + 3)[:S * nb].to(torch.int32).view(S, nb).cuda()
    kpool = torch.zeros(S * nb + 3, page, d, dtype=torch.bfloat16, device="cuda")
    vpool = torch.zeros_like(kpool)
    P.compact_kv_paged(kin, vin, idx, table, kpool, vpool, ctx=gpu)
    torch.cuda.synchronize()
    for s in range(S):
        rows_k = kpool[table[s].long()].reshape(-1, d)[:k]
        rows_v = vpool[table[s].long()].reshape(-1, d)[:k]
        assert torch.equal(rows_k.view(torch.int16), ko[s].view(torch.int16))
        assert torch.equal(rows_v.view(torch.int16), vo[s].view(torch.int16))
