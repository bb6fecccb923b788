"""GPU unit tests of the internal sm_100a kernels (tcgen05 GEMM with its fused
epilogues) against plain PyTorch fp64/fp32 references of the same op."""
import ctypes
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _hooks():
    import paper_2605_16360_b200 as P
    L = P.lib()
    f = L.pkv_test_gemm
    f.restype = ctypes.c_int
    f.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
                  ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                  ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
    return f


def _f16_round(t):
    import torch
    return t.to(torch.float16).to(torch.float64)


def _split_ref(t, planes):
    """What the kernel multiplies: hi (+ lo) fp16 planes of t, in fp64."""
    import torch
    hi = t.to(torch.float16)
    if planes == 1:
        return hi.to(torch.float64)
    lo = (t - hi.to(torch.float32)).to(torch.float16)
    return hi.to(torch.float64) + lo.to(torch.float64)


@pytest.mark.parametrize("M,K,N,bn,na,nb", [
    (128, 64, 64, 64, 1, 1), (300, 200, 72, 128, 1, 1), (1024, 512, 1536, 256, 1, 1), (1000, 512, 512, 256, 2, 1),
    (777, 768, 512, 256, 2, 2), (4096, 2048, 512, 256, 2, 1), (130, 16, 80, 128, 2, 2), (2048, 512, 2048, 128, 2, 1)])
def test_gemm_f32_epilogue(gpu, M, K, N, bn, na, nb):
    import torch
    import paper_2605_16360_b200 as P
    g = torch.Generator(device="cuda").manual_seed(M + K + N)
    a = torch.randn(M, K, device="cuda", generator=g)
    b = torch.randn(N, K, device="cuda", generator=g) / math.sqrt(K)
    bias = torch.randn(N, device="cuda", generator=g)
    out = torch.full((M, N), float("nan"), device="cuda")
    P.check(_hooks()(gpu.h, a.data_ptr(), M, K, b.data_ptr(), N, na, nb, bn, 0, bias.data_ptr(), None, 1,
                     out.data_ptr(), None))
    want = _split_ref(a, na) @ _split_ref(b, nb).T + bias.double()
    err = (out.double() - want).abs().max().item()
    scale = want.abs().max().item()
    assert err <= 2e-5 * scale, (err, scale)
    if na == 2 and nb == 2:
        exact = a.double() @ b.double().T + bias.double()
        assert (out.double() - exact).abs().max().item() <= 1e-5 * scale


@pytest.mark.parametrize("epi", [1, 2, 3, 4])
def test_gemm_fused_epilogues(gpu, epi):
    import torch
    import paper_2605_16360_b200 as P
    M, K, N, bn, lw = 640, 256, 384, 128, 200
    g = torch.Generator(device="cuda").manual_seed(epi)
    a = torch.randn(M, K, device="cuda", generator=g)
    b = torch.randn(N, K, device="cuda", generator=g) / math.sqrt(K)
    bias = torch.randn(N, device="cuda", generator=g)
    pe = torch.randn(lw, N, device="cuda", generator=g)
    resid = torch.randn(M, N, device="cuda", generator=g)
    out = resid.clone() if epi == 3 else torch.zeros(M, N, device="cuda")
    P.check(_hooks()(gpu.h, a.data_ptr(), M, K, b.data_ptr(), N, 2, 2, bn, epi, bias.data_ptr(), pe.data_ptr(), lw,
                     out.data_ptr(), None))
    x = a.double() @ b.double().T + bias.double()
    gelu = lambda t: 0.5 * t * (1 + torch.erf(t / math.sqrt(2)))
    if epi == 1:
        want = x
    elif epi == 2:
        want = gelu(x)
    elif epi == 3:
        want = resid.double() + x
    else:
        rows = torch.arange(M, device="cuda") % lw
        want = gelu(x) + pe.double()[rows]
    err = (out.double() - want).abs().max().item()
    assert err <= 1e-5 * max(1.0, want.abs().max().item()), err


@pytest.mark.parametrize("nwin,Lw,heads", [(1, 128, 1), (2, 256, 8), (3, 200, 8), (2, 2048, 8), (1, 77, 2)])
def test_encoder_attention(gpu, nwin, Lw, heads):
    import torch
    import paper_2605_16360_b200 as P
    D = 64 * heads
    f = P.lib().pkv_test_attention
    f.restype = ctypes.c_int
    f.argtypes = [ctypes.c_void_p, ctypes.c_void_p] + [ctypes.c_int64] * 4 + [ctypes.c_void_p, ctypes.c_void_p]
    g = torch.Generator(device="cuda").manual_seed(Lw)
    qkv = torch.randn(nwin * Lw, 3 * D, device="cuda", generator=g) * 1.5
    out = torch.full((nwin * Lw, D), float("nan"), device="cuda")
    P.check(f(gpu.h, qkv.data_ptr(), nwin, Lw, D, heads, out.data_ptr(), None))
    x = _f16_round(qkv).view(nwin, Lw, 3, heads, 64)
    q, k, v = (x[:, :, i].permute(0, 2, 1, 3) for i in range(3))  # [nwin, heads, Lw, 64]
    a = torch.softmax((q @ k.transpose(-1, -2)) / 8.0, dim=-1)
    want = (a @ v).permute(0, 2, 1, 3).reshape(nwin * Lw, D)
    err = (out.double() - want).abs().max().item()
    assert err < 3e-3 * want.abs().max().item(), err


@pytest.mark.parametrize("M,K,N,na,nb,epi", [(512, 512, 512, 2, 2, 0), (1000, 768, 512, 2, 2, 4), (2048, 512, 1536, 2, 2, 1),
                                           (777, 512, 2048, 2, 2, 2), (640, 2048, 512, 2, 2, 3), (256, 64, 256, 1, 1, 0),
                                           (300, 512, 700, 2, 1, 0)])
def test_gemm_cta_pair(gpu, M, K, N, na, nb, epi):
    """cta_group::2 (256x256 tile over a CTA pair) == plain fp64 reference."""
    import torch
    import paper_2605_16360_b200 as P
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N)
    a = torch.randn(M, K, device="cuda", generator=g)
    b = torch.randn(N, K, device="cuda", generator=g) / math.sqrt(K)
    bias = torch.randn(N, device="cuda", generator=g)
    pe = torch.randn(333, N, device="cuda", generator=g)
    resid = torch.randn(M, N, device="cuda", generator=g)
    out = resid.clone() if epi == 3 else torch.zeros(M, N, device="cuda")
    P.check(_hooks()(gpu.h, a.data_ptr(), M, K, b.data_ptr(), N, na, nb, 512, epi, bias.data_ptr(), pe.data_ptr(), 333,
                     out.data_ptr(), None))
    x = _split_ref(a, na) @ _split_ref(b, nb).T + bias.double()
    gelu = lambda t: 0.5 * t * (1 + torch.erf(t / math.sqrt(2)))
    want = {0: x, 1: x, 2: gelu(x), 3: resid.double() + x, 4: gelu(x) + pe.double()[torch.arange(M, device="cuda") % 333]}[epi]
    err = (out.double() - want).abs().max().item()
    assert err <= 2e-5 * max(1.0, want.abs().max().item()), err
