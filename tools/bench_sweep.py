"""BASELINE.json configs[4]: KV-budget sweep (rho 10-50% x ctx 8k-128k) on
Llama-3.1-8B target shapes (32 layers x 8 KV heads, head_dim 128, bf16): the
select + compaction regime, HBM-bound. Per point: select (radix Top-K ->
ascending indices, the library's choice of kernel, and each of the two select
kernels forced for comparison) and compaction (packed K/V gather) timed with CUDA events
on the launching stream through the C ABI with preallocated outputs (20 / 10
back-to-back launches queued behind a spin kernel, after 3 warm-ups; inputs >
L2 except the scores at 8k-16k, which the select reads once), algorithmic bytes per
SURVEY.md §8(d), fraction of MEASURED_PEAKS.json HBM bandwidth.

    python tools/bench_sweep.py [--out profiles/r01_sweep.json]
"""
import argparse
import ctypes
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
Ll, Hl, dt = 32, 8, 128
S = Ll * Hl
hbm = bench.peaks()[0]
ctx = P.Context(0)
_hook = P.lib().pkv_test_select_path
_hook.restype, _hook.argtypes = ctypes.c_int, [ctypes.c_int]
path = _hook
st = torch.cuda.current_stream()
rows = []
for N in (8192, 16384, 32768, 65536, 131072):
    g = torch.Generator(device="cuda").manual_seed(N)
    scores = torch.rand(S, N, device="cuda", generator=g)
    kt = torch.randint(-30000, 30000, (S, N, dt), device="cuda", dtype=torch.int16, generator=g).view(torch.bfloat16)
    vt = torch.randint(-30000, 30000, (S, N, dt), device="cuda", dtype=torch.int16, generator=g).view(torch.bfloat16)
    for rho in (0.1, 0.2, 0.3, 0.4, 0.5):
        K = P.retention_count(rho, N)
        ko = torch.empty(S, K, dt, dtype=torch.bfloat16, device="cuda")
        vo = torch.empty_like(ko)
        idx = torch.empty(S, K, dtype=torch.int32, device="cuda")
        L = P.lib()
        sel = lambda: P.check(L.pkv_topk_select(ctx.h, scores.data_ptr(), S, N, K, None, idx.data_ptr(),
                                                st.cuda_stream))
        sel()
        cmp = lambda: P.check(L.pkv_compact_kv(ctx.h, kt.data_ptr(), vt.data_ptr(), idx.data_ptr(), S, N, K, dt, 2,
                                               ko.data_ptr(), vo.data_ptr(), st.cuda_stream))
        for _ in range(3):
            sel()
            cmp()
        unit = lambda: P.check(L.pkv_select_compact(ctx.h, scores.data_ptr(), S, N, K, kt.data_ptr(), vt.data_ptr(),
                                                     dt, 2, idx.data_ptr(), ko.data_ptr(), vo.data_ptr(),
                                                     st.cuda_stream))
        for _ in range(3):
            unit()
        t_sel = bench.time_loop(sel, 20, st)
        t_cmp = bench.time_loop(cmp, 10, st)
        t_sc = bench.time_loop(unit, 10, st)  # pkv_select_compact: both kernels as one call
        alt = {}
        for mode, name in ((0, "register_cached_radix"), (1, "streaming")):
            prev = path(mode)  # force one select kernel (select.cu / select_stream.cu)
            sel()
            alt[name] = bench.time_loop(sel, 20, st)
            path(prev)
        c = dict(Ll=Ll, Hl=Hl, N=N, rho=rho, dt=dt)
        b_sel, b_cmp = bench.bytes_select(c), bench.bytes_compact(c)
        r = dict(N=N, rho=rho, K=K, select_ms=t_sel, compact_ms=t_cmp,
                 select_kernel_ms=alt,
                 select_gbs=b_sel / t_sel / 1e6, compact_gbs=b_cmp / t_cmp / 1e6,
                 combined_frac_hbm=(b_sel + b_cmp) / (t_sel + t_cmp) / 1e6 / hbm,
                 select_compact_ms=t_sc, select_compact_frac_hbm=(b_sel + b_cmp) / t_sc / 1e6 / hbm)
        rows.append(r)
        print(f"N={N:6d} rho={rho:.1f} K={K:6d}  select {t_sel * 1e3:6.1f} us (cached radix "
              f"{alt['register_cached_radix'] * 1e3:6.1f}, streaming {alt['streaming'] * 1e3:6.1f}) "
              f"{r['select_gbs']:5.0f} GB/s  compact {t_cmp:6.3f} ms {r['compact_gbs']:5.0f} GB/s  "
              f"select+compact {100 * r['combined_frac_hbm']:.1f}% of {hbm:.0f} GB/s; pkv_select_compact "
              f"{t_sc * 1e3:6.1f} us {100 * r['select_compact_frac_hbm']:.1f}%", flush=True)
        del ko, vo, idx
    del scores, kt, vt
    torch.cuda.empty_cache()
if a.out:
    json.dump({"hbm_peak_gbs": hbm, "target": "Llama-3.1-8B (32L, 8KV, d128) bf16", "points": rows},
              open(a.out, "w"), indent=1)
