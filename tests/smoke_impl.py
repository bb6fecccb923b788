"""__graft_entry__.smoke(): one small pass of the whole hot path on cuda:0
(proxy scoring -> HybridAxialMapper -> Top-K select -> KV compaction, through
pkv_pruner_run), checked against the oracle (the oracle is only the checker
here): scores and mapped scores within rel 1e-3 of the fp64 restatement,
select + compaction bit-exact from the GPU's own mapped scores."""
import numpy as np


def run_smoke():
    import torch
    import paper_2605_16360_b200 as P
    from oracle import pkv_oracle as O

    assert torch.cuda.is_available(), "smoke needs cuda:0"
    ctx = P.Context.default(0)
    Ls, Hq, Hs, dp, Ll, Hl, dt, N, rho = 1, 4, 2, 64, 2, 4, 64, 1024, 0.2
    geom = P.ModelGeometry(Ll, Hl, Ls, Hs, dt)
    cfg = P.MapperConfig(encoder_layers=2)
    m = P.Mapper(geom, cfg, seed=7, precision=P.MAPPER_FP16X3, ctx=ctx)
    pr = P.Pruner(m, Hq, dp, dt, N, rho)
    K = pr.k
    r = np.random.RandomState(0)
    qb = O.f32_to_bf16_bits(r.standard_normal((Ls, Hq, N, dp)).astype(np.float32) * 0.35)
    kb = O.f32_to_bf16_bits(r.standard_normal((Ls, Hs, N, dp)).astype(np.float32))
    kt = r.randint(0, 1 << 15, (Ll, Hl, N, dt)).astype(np.uint16)
    vt = r.randint(0, 1 << 15, (Ll, Hl, N, dt)).astype(np.uint16)
    dev = lambda a: torch.from_numpy(a.view(np.int16)).cuda().view(torch.bfloat16)
    ko = torch.empty(Ll, Hl, K, dt, dtype=torch.bfloat16, device="cuda")
    vo = torch.empty_like(ko)
    idx = torch.empty(Ll, Hl, K, dtype=torch.int32, device="cuda")
    y = torch.empty(Ll, Hl, N, device="cuda")
    pr.run(dev(qb), dev(kb), dev(kt), dev(vt), ko, vo, idx, y)
    torch.cuda.synchronize()

    x_ref = O.score(qb, kb, reduce="max")
    x = P.score(dev(qb), dev(kb), ctx=ctx).cpu().numpy()
    assert np.abs(x - x_ref).max() <= 1e-3 * np.abs(x_ref).max()
    mp = O.MapperParams.init(O.Geometry(Ll, Hl, Ls, Hs, dt), O.MapperConfig(encoder_layers=2), 7)
    y_ref = O.forward_full(x_ref[None].astype(np.float64), mp)[0]
    yy = y.cpu().numpy()
    rel = (np.linalg.norm((yy - y_ref).reshape(-1, N), axis=1) / np.linalg.norm(y_ref.reshape(-1, N), axis=1)).max()
    assert rel <= 1e-3, rel
    _, oidx = O.topk_select(yy.reshape(-1, N), K)
    assert np.array_equal(idx.view(-1, K).cpu().numpy(), oidx)
    eko, _ = O.compact_kv(kt.reshape(-1, N, dt), vt.reshape(-1, N, dt), oidx)
    assert np.array_equal(ko.view(torch.int16).cpu().numpy().view(np.uint16).reshape(-1, K, dt), eko)
    print(f"smoke ok: score -> map -> select -> compact (mapped-score rel {rel:.1e}), launches = {ctx.launches()}")
