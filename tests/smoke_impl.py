"""__graft_entry__.smoke(): one small pass of the hot path on cuda:0, checked
against the oracle (the oracle is only the checker here)."""
import numpy as np


def run_smoke():
    import torch
    import paper_2605_16360_b200 as P
    from oracle import pkv_oracle as O

    assert torch.cuda.is_available(), "smoke needs cuda:0"
    ctx = P.Context.default(0)
    r = np.random.RandomState(0)
    s = r.uniform(size=(16, 4096)).astype(np.float32)
    k = P.retention_count(0.2, 4096)
    mask, idx = P.topk_select(torch.from_numpy(s).cuda(), k, ctx=ctx)
    omask, oidx = O.topk_select(s, k)
    assert np.array_equal(mask.cpu().numpy(), omask) and np.array_equal(idx.cpu().numpy(), oidx)
    kv = torch.randn(16, 4096, 128, device="cuda", dtype=torch.bfloat16)
    ko, vo = P.compact_kv(kv, kv, idx, ctx=ctx)
    assert torch.equal(ko, kv[torch.arange(16, device="cuda")[:, None], idx.long()])
    torch.cuda.synchronize()
    print("smoke ok: select+compact, launches =", ctx.launches())
