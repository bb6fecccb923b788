"""Formats driving the GPU path: a mapper loaded from a checkpoint file
 equals the mapper built from the same blob, and an (X, Ŷ) pair
dumped to a PKVT trace replays bit-identically through the
device mapper."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_checkpoint_and_trace_replay(gpu, tmp_path):
    import torch
    import paper_2605_16360_b200 as P
    geom, cfg = P.ModelGeometry(4, 8, 2, 4, 64), P.MapperConfig()
    blob = P.mapper_init_params(geom, cfg, 3) * 1.01  # "trained" weights
    ck = str(tmp_path / "m.pkvc")
    P.write_checkpoint(ck, geom, cfg, blob)
    m1 = P.Mapper(geom, cfg, blob, ctx=gpu)
    m2 = P.Mapper.from_checkpoint(ck, ctx=gpu)
    x = torch.rand(1, 2, 4, 3000, device="cuda") * 2
    y1, y2 = m1.forward_full(x), m2.forward_full(x)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2)
    tr = str(tmp_path / "xy.pkvt")
    P.write_trace(tr, x.cpu().numpy()[None], y1.cpu().numpy()[None], meta="source=test")
    xs, ys = P.read_trace(tr)
    y3 = m2.forward_full(torch.from_numpy(xs[0]).cuda())
    torch.cuda.synchronize()
    assert np.array_equal(y3.cpu().numpy(), ys[0])
