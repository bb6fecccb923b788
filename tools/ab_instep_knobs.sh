# In-step A/B of the exponential-split knobs under the power cap: the whole bench
# step (device-resident, 10 timed steps) per setting, interleaved with the default
# so box drift shows. Output: gpurun_out/ab_instep.txt (ms_per_step, live stages).
set -u
out=gpurun_out/ab_instep.txt
: > $out
run() {  # label, env...
    label=$1; shift
    env "$@" timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_line.json 2> /dev/null
    python - "$label" >> $out <<'PY'
import json, sys
d = json.loads(open("gpurun_out/ab_line.json").read().strip().splitlines()[-1])
lv = d.get("stages_live_ms", {})
print(f"{sys.argv[1]:<14} step {d['ms_per_step']:7.2f} ms  lse {lv.get('score_lse', 0):6.1f}  pool {lv.get('score_pool', 0):5.1f}  "
      f"map {lv.get('map', 0):6.1f}  clock {d['clocks']['sm_mhz']}")
PY
}
run default PKV_POLY_PAIRS=10
run poly6 PKV_POLY_PAIRS=6
run poly14 PKV_POLY_PAIRS=14
run default PKV_POLY_PAIRS=10
run poly8 PKV_POLY_PAIRS=8
run poly12 PKV_POLY_PAIRS=12
run default PKV_POLY_PAIRS=10
run attn2 PKV_ATTN_POLY=2
run attn6 PKV_ATTN_POLY=6
run default PKV_POLY_PAIRS=10
