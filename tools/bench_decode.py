"""one decode step of the Llama-3.1-8B target (32 layers,
32 query / 8 KV heads, d 128) over the packed cache the pruner produced
(32k context; rho 0.1-0.5) vs the full cache: time (CUDA events, 20
iterations after 3 warm-ups), HBM GB/s against MEASURED_PEAKS.json. The
packed cache makes every decode step read rho of the bytes.

    python tools/bench_decode.py [--out profiles/r01_decode.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_16360_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out", default=None)
a = ap.parse_args()
L, Hq, Hkv, d, N = 32, 32, 8, 128, 32768
hbm = bench.peaks()[0]
ctx = P.Context(0)
st = torch.cuda.current_stream()
g = torch.Generator(device="cuda").manual_seed(0)
q = (torch.randn(L, Hq, d, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
rows = []
for rho in (None, 0.1, 0.2, 0.3, 0.5):
    K = N if rho is None else P.retention_count(rho, N)
    k = torch.randn(L, Hkv, K, d, device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn(L, Hkv, K, d, device="cuda", generator=g).to(torch.bfloat16)
    o = torch.empty(L, Hq, d, device="cuda")
    f = lambda: P.packed_decode_attention(q, k, v, ctx=ctx, stream=st, out=o)
    for _ in range(3):
        f()
    ms = bench.time_loop(f, 20, st)
    byts = 2 * L * Hkv * K * d * 2 + L * Hq * d * 2 + L * Hq * d * 4
    r = dict(rho=rho, K=K, ms=ms, gbs=byts / ms / 1e6, frac_hbm=byts / ms / 1e6 / hbm)
    rows.append(r)
    print(f"{'full' if rho is None else f'rho={rho:.1f}':9s} K={K:6d}  {ms:7.3f} ms  {r['gbs']:7.0f} GB/s  "
          f"{100 * r['frac_hbm']:.1f}% of {hbm:.0f} GB/s", flush=True)
    del k, v
if a.out:
    json.dump({"target": "Llama-3.1-8B decode (32L, 32Q/8KV, d128), 32k context", "hbm_peak_gbs": hbm,
               "points": rows}, open(a.out, "w"), indent=1)
