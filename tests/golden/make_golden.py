"""Generates the committed golden fixtures in tests/golden/ from the REFERENCE
ITSELF: the unmodified /root/reference/proj sources compiled by oracle/Makefile
into oracle/_ref/libpkvref.so. Inputs are regenerated with the reference's own
Rng exactly as its unit tests do (proj/tests/test_pruning.cpp,
test_mapper.cpp). Run here (the container with /root/reference):

    make -C oracle && python tests/golden/make_golden.py [--slow]

The GPU box never runs this; it reads the .npz files.
"""
from __future__ import annotations

import argparse
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import pkv_oracle as O  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def pruning(ref: O.RefLib):
    g = {}
    # test_pruning.cpp:47-63 basic selections
    for name, vals, rho in [("basic", [3, 1, 2], 0.34), ("basic_all", [3, 1, 2], 1.0), ("tie", [0.3, 0.3, 0.1], 0.3),
                            ("loss_gt", [0.5, 0.1, 0.4, 0.2, 0.3], 0.4)]:
        bits, k = ref.topk_mask(np.array([[vals]], np.float64), rho)
        g[f"{name}_scores"] = np.array(vals, np.float64)
        g[f"{name}_rho"] = np.float64(rho)
        g[f"{name}_bits"] = bits.reshape(-1)
        g[f"{name}_k"] = np.int64(k)
    # test_pruning.cpp:65-82 exhaustive 3^8 alphabet, k = 1..8
    alphabet = np.array([0.1, 0.2, 0.3])
    codes = np.arange(6561)
    digits = np.stack([(codes // 3 ** i) % 3 for i in range(8)], axis=1)
    vecs = alphabet[digits]  # [6561, 8]
    ex_bits = np.zeros((8, 6561, 8), np.uint8)
    for k in range(1, 9):
        bits, kk = ref.topk_mask(vecs[:, None, :], k / 8.0)
        assert kk == k
        ex_bits[k - 1] = bits.reshape(6561, 8)
    g["exhaustive_vectors"] = vecs
    g["exhaustive_bits"] = ex_bits
    # test_pruning.cpp:84-98: 1000 length-32 tie-heavy vectors from Rng(99)
    rng = ref.rng(99)
    tv, tk, tb = [], [], []
    for _ in range(1000):
        v = [math.floor(rng.uniform(0.0, 8.0)) / 8.0 for _ in range(32)]
        k = 1 + rng.below(32)
        bits, kk = ref.topk_mask(np.array([[v]]), k / 32.0)
        assert kk == k
        tv.append(v)
        tk.append(k)
        tb.append(bits.reshape(-1))
    g["ties_vectors"] = np.array(tv)
    g["ties_k"] = np.array(tk, np.int64)
    g["ties_bits"] = np.array(tb, np.uint8)
    # test_pruning.cpp:100-113 affine invariance, Rng(5), [2,3,16] in [0,4), rho .25
    rng = ref.rng(5)
    av, aa, ac = [], [], []
    for _ in range(50):
        y = [rng.uniform(0.0, 4.0) for _ in range(2 * 3 * 16)]
        a = rng.uniform(0.1, 5.0)
        c = rng.uniform(-3.0, 3.0)
        av.append(y)
        aa.append(a)
        ac.append(c)
    g["affine_vectors"] = np.array(av).reshape(50, 2, 3, 16)
    g["affine_alpha"] = np.array(aa)
    g["affine_c"] = np.array(ac)
    g["affine_bits"] = np.stack([ref.topk_mask(v, 0.25)[0] for v in g["affine_vectors"]])
    # test_pruning.cpp:169-183 apply_mask: Rng(1) [1,1,1024] U[0,1)
    rng = ref.rng(1)
    big = np.array([rng.uniform(0.0, 1.0) for _ in range(1024)]).reshape(1, 1, 1024)
    bits, k = ref.topk_mask(big, 0.5)
    idx, dropped, per_head, total = ref.apply_mask(bits, k, 128, 2)
    g["apply_big_scores"] = big
    g["apply_big_idx"] = idx
    g["apply_big_bytes_per_head"] = np.int64(per_head)
    # Random fp32-representable scores at a realistic slice length with ±0.0,
    # subnormals and duplicate runs: [4, 3, 4096] at rho 0.2.
    r = np.random.RandomState(20260517)
    s = r.uniform(-1, 1, (4, 3, 4096)).astype(np.float32)
    s[0, 0, ::7] = 0.0
    s[0, 0, ::11] = -0.0
    s[0, 1, :100] = np.float32(1e-40)  # subnormal
    s[1, 2, :] = 0.25  # one all-equal slice
    s[2] = np.round(s[2] * 16) / 16  # heavy ties
    s = s.astype(np.float64)
    bits, k = ref.topk_mask(s, 0.2)
    idx, *_ = ref.apply_mask(bits, k, 128, 2)
    g["rand_scores"] = s.astype(np.float32)
    g["rand_bits"] = bits
    g["rand_idx"] = idx.astype(np.int32)
    g["rand_k"] = np.int64(k)
    np.savez_compressed(os.path.join(OUT, "pruning.npz"), **g)
    print("pruning.npz written")


def toy_geometry():
    return O.Geometry(4, 4, 2, 2, 8)  # test_mapper.cpp:19-27


def paper_config(**kw):
    return O.MapperConfig(**kw)


def mapper(ref: O.RefLib, slow: bool):
    g = {}
    # window offsets vectors (test_mapper.cpp:201-206)
    for i, (n, c, s) in enumerate([(12, 8, 4), (2048, 2048, 1024), (3072, 2048, 1024), (10, 4, 2), (13, 8, 4),
                                   (32768, 2048, 1024), (131072, 2048, 1024), (170000, 2048, 1024)]):
        g[f"win{i}_args"] = np.array([n, c, s], np.int64)
        g[f"win{i}_offsets"] = np.array(ref.window_offsets(n, c, s), np.int64)
    # layer pairing at the BASELINE geometries
    for name, (ll, ls) in {"llama": (32, 16), "qwen25": (28, 24), "qwen3": (64, 28), "tiny": (4, 2)}.items():
        geo = O.Geometry(ll, 8, ls, 8, 128)
        g[f"pair_{name}"] = np.array([ref.layer_pair(l, geo) for l in range(1, ll + 1)], np.int64)
    # PE slots
    g["pe_64_512"] = ref.sinusoidal_pe(64, 512)
    # Paper-width mapper (defaults, mapper.hpp:35-55) on small inputs: these are
    # the GPU-parity fixtures (the GPU path supports d_time % 64 == 0, d_head 64).
    cases = [
        # name, geometry, config kwargs, x shape (forward_full [B, Ls, Hs, N]), seed
        ("tiny_n256", O.Geometry(4, 8, 2, 4, 64), {}, (1, 2, 4, 256), 7),
        ("tiny_n200", O.Geometry(4, 8, 2, 4, 64), {}, (1, 2, 4, 200), 8),
        ("llama_n384_crop256", O.Geometry(32, 8, 16, 8, 128), {"crop_len": 256, "stride": 128}, (1, 16, 8, 384), 9),
        ("qwen25_n300", O.Geometry(28, 4, 24, 2, 128), {"crop_len": 128, "stride": 64}, (1, 24, 2, 300), 10),
        ("syn3_b2", O.Geometry(2, 8, 2, 4, 64), {"synthetic_heads": 3, "encoder_layers": 2}, (2, 2, 4, 128), 11),
    ]
    if slow:
        cases += [("tiny_full_n2048", O.Geometry(4, 8, 2, 4, 64), {}, (1, 2, 4, 2048), 12)]
    for name, geo, kw, shape, seed in cases:
        cfg = O.MapperConfig(**kw)
        t0 = time.time()
        rm = ref.mapper(geo, cfg, seed)
        x = np.random.RandomState(seed).uniform(0.0, 2.0, shape).astype(np.float32).astype(np.float64)
        y = rm.forward_full(x)
        g[f"{name}_geom"] = np.array(geo.as5(), np.int64)
        g[f"{name}_cfg"] = np.array(cfg.as12(), np.int64)
        g[f"{name}_seed"] = np.int64(seed)
        g[f"{name}_x"] = x.astype(np.float32)
        g[f"{name}_y"] = y
        print(f"  {name}: {time.time() - t0:.1f}s")
    np.savez_compressed(os.path.join(OUT, "mapper.npz"), **g)
    print("mapper.npz written")


def rng(ref: O.RefLib):
    r = ref.rng(12345)
    u = np.array([r.uniform(-0.5, 0.5) for _ in range(64)])
    r = ref.rng(777)
    nrm = np.array([r.normal() for _ in range(65)])
    r = ref.rng(31)
    b = np.array([r.below(17) for _ in range(64)], np.uint64)
    np.savez_compressed(os.path.join(OUT, "rng.npz"), uniform_12345=u, normal_777=nrm, below_31_17=b)
    print("rng.npz written")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--slow", action="store_true")
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    ref = O.RefLib()
    if a.only in ("", "rng"):
        rng(ref)
    if a.only in ("", "pruning"):
        pruning(ref)
    if a.only in ("", "mapper"):
        mapper(ref, a.slow)
