"""bench.py's JSON line contract on CPU: build_line over a synthetic run_ours
result carries every key the driver reads (metric/value/unit/n_gpus/steps/
warmup/ms_per_step/higher_is_better/scaling/vs_baseline/dtype/data/config,
roofline with the live in-step kernel time against the sustained peak, e2e with
the copied bytes, gpu_launches, clocks), and the numbers follow from the inputs."""
import argparse

import pytest

import bench


def _result(live=True):
    c = bench.CONFIGS["llama32k"]
    st = {"score_lse_ms": 118.0, "score_pool_ms": 52.0, "map_ms": 150.0, "select_ms": 0.04, "compact_ms": 0.28,
          "x_prefill_attn_causal_ms": 100.0, "x_score_pool_causal_ms": 31.0, "x_prune_with_prefill_lse_ms": 188.0}
    r = {"ms": 340.0, "shard": "none", "K": 6554, "stages": st, "clocks": {"sm_max_mhz": 1965.0, "reasons": []},
         "launches": 156, "e2e": {"ms": 345.0, "h2d": 6979321856, "d2h": 865757184}}
    if live:
        r["stages_live"] = {"score_lse": 135.0, "score_pool": 56.0, "map": 150.0, "select": 0.06, "compact": 0.3}
    return c, r


def _args():
    return argparse.Namespace(steps=20, warmup=3, config="llama32k", precision=3)


@pytest.mark.parametrize("live", [True, False])
def test_bench_line_contract(live):
    c, r = _result(live)
    line = bench.build_line(r, _args(), c, 1)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in line, k
    assert line["metric"] == bench.METRIC and line["unit"] == "tokens/s" and line["higher_is_better"] is True
    assert line["value"] == pytest.approx(c["N"] / 0.340)
    assert line["config"]["workload"] == "llama32k" and line["scaling"] == "weak" and line["n_gpus"] == 1
    roof = line["roofline"]
    assert roof["kernel"] == "score_lse" and roof["bound"] == "tensor" and roof["unit"] == "TFLOP/s"
    _, burst, sustained, _ = bench.peaks()
    t = 135.0 if live else 118.0
    assert roof["achieved"] == pytest.approx(bench.flops_score_pass(c) / (t * 1e-3) / 1e12)
    assert roof["peak"] == pytest.approx(sustained if live else burst)
    assert roof["frac"] == pytest.approx(roof["achieved"] / roof["peak"])
    e = line["e2e"]
    assert e["value"] == pytest.approx(c["N"] / 0.345) and e["unit"] == "tokens/s"
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert line["gpu_launches"] == 156
    assert ("stages_live_ms" in line) == live


def test_bench_line_strong_scaling_counts_one_context():
    c, r = _result()
    r["shard"] = "layer"
    line = bench.build_line(r, _args(), c, 4)
    assert line["scaling"] == "strong" and line["n_gpus"] == 4
    assert line["value"] == pytest.approx(c["N"] / 0.340)  # one context over 4 GPUs
    r["shard"] = "none"
    assert bench.build_line(r, _args(), c, 4)["value"] == pytest.approx(4 * c["N"] / 0.340)  # weak: 4 contexts
