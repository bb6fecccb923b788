"""Phase timing of the Top-K select (select.cu): the kernel stops after
phase PKV_SELECT_PROBE (1 load, 2 pass 0, 3 k-th key, 0 full) and is timed
as 20 back-to-back launches through the C ABI; run once per probe value and
for the legacy one-CTA-per-slice kernel (PKV_SELECT_LEGACY=1).

    python tools/probe_select.py            # driver: all probes, table
    python tools/probe_select.py --one      # one configuration (env-driven)
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SHAPES = [(256, 8192), (256, 32768), (256, 131072), (112, 170000)]


def one():
    import torch
    import bench
    import paper_2605_16360_b200 as P
    ctx = P.Context(0)
    st = torch.cuda.current_stream()
    L = P.lib()
    out = {}
    for S, n in SHAPES:
        for dist in ("uniform", "logits"):
            g = torch.Generator(device="cuda").manual_seed(n)
            s = torch.rand(S, n, device="cuda", generator=g) if dist == "uniform" else \
                torch.randn(S, n, device="cuda", generator=g) * 0.08 - 0.05
            k = P.retention_count(0.2, n)
            idx = torch.empty(S, k, dtype=torch.int32, device="cuda")
            f = lambda: P.check(L.pkv_topk_select(ctx.h, s.data_ptr(), S, n, k, None, idx.data_ptr(), st.cuda_stream))
            f()
            out[f"{S}x{n}/{dist}"] = bench.time_loop(f, 20, st) * 1e3
    print(json.dumps(out))


if __name__ == "__main__":
    if "--one" in sys.argv:
        one()
        sys.exit(0)
    rows = {}
    for name, env in [("legacy", {"PKV_SELECT_LEGACY": "1"}), ("load", {"PKV_SELECT_PROBE": "1"}),
                      ("pass0", {"PKV_SELECT_PROBE": "2"}), ("kth", {"PKV_SELECT_PROBE": "3"}), ("full", {})]:
        r = subprocess.run([sys.executable, __file__, "--one"], env={**os.environ, **env}, capture_output=True,
                           text=True)
        rows[name] = json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else r.stderr[-500:]
    keys = list(rows["full"].keys()) if isinstance(rows["full"], dict) else []
    print("us".ljust(22) + "".join(k.ljust(9) for k in rows))
    for key in keys:
        print(key.ljust(22) + "".join(f"{rows[c][key]:8.1f} " if isinstance(rows[c], dict) else "err      "
                                       for c in rows))
    json.dump(rows, open(os.path.join(ROOT, "gpurun_out", "probe_select.json"), "w"), indent=1)
