"""GPU training of the HybridAxialMapper (pkv_trainer) against
the reference itself: oracle/_ref's pkvref_mapper_train_grad runs the
reference's training forward_pair (mapper.cpp:274-342, batchnorm1d on batch
statistics, ops.cpp:806-850) and its tape's reverse sweep (tensor.cpp) of
Σ dlogits ⊙ logits, in fp64. The GPU computes in fp32.

Tolerances (fp32 vs fp64; measured on B200: logits <= 3.5e-7, gradients <=
1.7e-6, BN statistics <= 2e-8): logits norm-wise relative error <= 5e-6 per
(batch, head) row; every parameter's gradient norm-wise relative error <= 2e-5
(for tensors whose true gradient is ~0: error <= 2e-5 of the largest gradient
norm); BN running statistics after the step <= 1e-6 relative."""
import numpy as np
import pytest

from oracle import pkv_oracle as O

pytestmark = pytest.mark.gpu

# (geom5, cfg kwargs, B, n, x range, normalize_input)
CASES = {
    # the reference's own gradient test (test_mapper.cpp:365-390)
    "ref_gradcheck_toy": ((1, 2, 1, 2, 4), dict(d_time=4, encoder_layers=1, encoder_heads=2, ffn_mult=2, d_head=2,
                                                crop_len=8, stride=4), 2, 5),
    "d128_two_layers": ((2, 3, 2, 4, 64), dict(d_time=128, encoder_layers=2, encoder_heads=2, ffn_mult=4, d_head=16,
                                               crop_len=128, stride=64, normalize_input=1), 2, 96),
    "conv_bypass_cross_bypass": ((2, 2, 2, 3, 64), dict(d_time=64, encoder_layers=1, encoder_heads=4, ffn_mult=2,
                                                        d_head=8, crop_len=64, stride=32, stage_conv=1,
                                                        stage_cross=1), 3, 40),
    "enc_bypass_syn3": ((2, 4, 2, 2, 64), dict(d_time=32, encoder_layers=0, encoder_heads=2, ffn_mult=2, d_head=8,
                                               crop_len=64, stride=32, synthetic_heads=3, stage_encoder=1), 2, 33),
    "llama_width_n128": ((32, 8, 16, 8, 128), dict(d_time=512, encoder_layers=2, encoder_heads=8, ffn_mult=4,
                                                   d_head=64, crop_len=2048, stride=1024), 1, 128),
}


def _cfgs(P, g5, kw):
    stage = {0: "active", 1: "bypass"}
    base = {k: v for k, v in kw.items() if not k.startswith("stage") and k != "normalize_input"}
    modes = dict(stage_conv=stage[kw.get("stage_conv", 0)], stage_encoder=stage[kw.get("stage_encoder", 0)],
                 stage_cross=stage[kw.get("stage_cross", 0)], normalize_input=bool(kw.get("normalize_input", 0)))
    return P.ModelGeometry(*g5), P.MapperConfig(**base, **modes), O.Geometry(*g5), O.MapperConfig(**base, **modes)


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("name", list(CASES))
def test_train_step_matches_reference_tape(gpu, name):
    import torch
    import paper_2605_16360_b200 as P
    g5, kw, B, n = CASES[name]
    pg, pc, og, oc = _cfgs(P, g5, kw)
    seed = 23
    ref = O.RefLib()
    rm = ref.mapper(og, oc, seed)
    blob0 = rm.blob()
    rng = np.random.default_rng(7)
    x = rng.uniform(0.0, 2.0, (B, g5[3], n)).astype(np.float32).astype(np.float64)  # the GPU's fp32 input
    dl = rng.normal(size=(B, g5[1], n))
    ref_logits, ref_grad = rm.train_grad(x, dl)
    ref_blob = rm.blob()  # BN running stats after the step

    tr = P.MapperTrainer(pg, pc, blob0, ctx=gpu)
    assert tr.n_params == ref_grad.size and tr.n_total == blob0.size
    logits = tr.forward(torch.from_numpy(x.astype(np.float32)).cuda())
    grad = tr.backward(torch.from_numpy(dl).cuda())
    torch.cuda.synchronize()
    y = logits.cpu().numpy().astype(np.float64)
    lerr = max(_rel(y[b, h], ref_logits[b, h]) for b in range(B) for h in range(g5[1]))
    g = grad.cpu().numpy()
    names = [t[0] for t in rm.tensors()]
    sizes = [t[1].size for t in rm.tensors()]
    gmax = max(np.linalg.norm(ref_grad[o:o + s]) for o, s in zip(np.cumsum([0] + sizes[:-1]), sizes)
               if o + s <= ref_grad.size)
    worst = (0.0, "")
    o = 0
    for nm, s in zip(names, sizes):
        if o >= ref_grad.size:
            break
        gr, gg = ref_grad[o:o + s], g[o:o + s]
        err = _rel(gg, gr) if np.linalg.norm(gr) > 1e-3 * gmax else np.linalg.norm(gg - gr) / gmax
        worst = max(worst, (err, nm))
        o += s
    berr = _rel(tr.blob()[ref_grad.size:], ref_blob[ref_grad.size:]) if ref_blob.size > ref_grad.size else 0.0
    print(f"{name}: logits rel {lerr:.2e}, worst grad rel {worst[0]:.2e} ({worst[1]}), bn stats rel {berr:.2e}")
    assert lerr <= 5e-6
    assert worst[0] <= 2e-5, worst
    assert berr <= 1e-6


def test_train_step_with_device_loss(gpu):
    """logits -> pkv_loss_total's d total / d logits (fp64, on the device) ->
    pkv_trainer_backward: the same parameter gradients as the reference's tape
    for that upstream gradient (the loss itself is pinned by test_loss_gpu)."""
    import torch
    import paper_2605_16360_b200 as P
    g5, kw, B, n = CASES["d128_two_layers"]
    pg, pc, og, oc = _cfgs(P, g5, kw)
    ref = O.RefLib()
    rm = ref.mapper(og, oc, 5)
    blob0 = rm.blob()
    rng = np.random.default_rng(3)
    x = rng.uniform(0.0, 2.0, (B, g5[3], n)).astype(np.float32)
    y = rng.gamma(0.5, 1.0, (B, g5[1], n)).astype(np.float32)
    tr = P.MapperTrainer(pg, pc, blob0, ctx=gpu)
    logits = tr.forward(torch.from_numpy(x).cuda())
    rep, dl = P.loss_total(logits, torch.from_numpy(y).cuda(), P.LossConfig(max_pairs=256), seed=11, ctx=gpu)
    grad = tr.backward(dl)
    torch.cuda.synchronize()
    _, ref_grad = rm.train_grad(x.astype(np.float64), dl.cpu().numpy())
    assert np.isfinite(rep.total)
    assert _rel(grad.cpu().numpy(), ref_grad) <= 2e-5


def test_backward_accumulates_and_errors(gpu):
    import torch
    import paper_2605_16360_b200 as P
    g5, kw, B, n = CASES["ref_gradcheck_toy"]
    pg, pc, _, _ = _cfgs(P, g5, kw)
    tr = P.MapperTrainer(pg, pc, seed=1, ctx=gpu)
    with pytest.raises(P.PkvValueError):
        tr.backward(torch.zeros(B, g5[1], n, dtype=torch.float64, device="cuda"))
    x = torch.rand(B, g5[3], n, device="cuda")
    tr.forward(x)
    dl = torch.randn(B, g5[1], n, dtype=torch.float64, device="cuda")
    g1 = tr.backward(dl)
    g2 = tr.backward(dl, grad=g1.clone())
    torch.cuda.synchronize()
    assert torch.allclose(g2, 2 * g1, rtol=1e-5, atol=1e-12)  # LN parameter sums use atomics
    with pytest.raises(P.PkvValueError, match="sliding_forward"):
        tr.forward(torch.rand(1, g5[3], kw["crop_len"] + 1, device="cuda"))
    with pytest.raises(P.PkvValueError, match="B\\*N >= 2"):
        tr.forward(torch.rand(1, g5[3], 1, device="cuda"))


def test_train_normalize_zero_rows_and_all_bypass(gpu):
    """normalize_input on a window whose mean is 0 (clamp_min(·, 1e-12), mapper.cpp:288-291)
    and the all-bypass pipeline (test_mapper.cpp:139-199's composition) against the
    reference's tape."""
    import torch
    import paper_2605_16360_b200 as P
    for kw in (dict(d_time=64, encoder_layers=1, encoder_heads=2, ffn_mult=2, d_head=8, crop_len=64, stride=32,
                    normalize_input=1),
               dict(d_time=32, encoder_layers=1, encoder_heads=2, ffn_mult=2, d_head=8, crop_len=64, stride=32,
                    stage_conv=1, stage_encoder=1, stage_cross=1)):
        g5 = (2, 3, 2, 2, 64)
        pg, pc, og, oc = _cfgs(P, g5, kw)
        rm = O.RefLib().mapper(og, oc, 9)
        blob0 = rm.blob()
        rng = np.random.default_rng(4)
        x = rng.uniform(0.0, 2.0, (2, 2, 48)).astype(np.float32).astype(np.float64)
        x[1, 0, :] = 0.0  # mean 0: the clamp's floor
        dl = rng.normal(size=(2, 3, 48))
        ref_logits, ref_grad = rm.train_grad(x, dl)
        tr = P.MapperTrainer(pg, pc, blob0, ctx=gpu)
        y = tr.forward(torch.from_numpy(x.astype(np.float32)).cuda()).cpu().numpy()
        g = tr.backward(torch.from_numpy(dl).cuda()).cpu().numpy()
        assert np.isfinite(y).all() and np.isfinite(g).all()
        assert _rel(y.astype(np.float64), ref_logits) <= 5e-6
        assert _rel(g, ref_grad) <= 2e-5


def test_train_config_limits(gpu):
    import paper_2605_16360_b200 as P
    pg, pc, _, _ = _cfgs(P, (1, 33, 1, 2, 64), dict(d_time=32, encoder_layers=1, encoder_heads=2, ffn_mult=2,
                                                   d_head=8, crop_len=64, stride=32))
    tr = P.MapperTrainer(pg, pc, seed=1, ctx=gpu)
    import torch
    with pytest.raises(P.ConfigError, match="target_heads <= 32"):
        tr.forward(torch.rand(1, 2, 16, device="cuda"))
