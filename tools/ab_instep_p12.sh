# Follow-up of tools/ab_instep_knobs.sh: PKV_POLY_PAIRS 12 vs the default 10, interleaved x4.
set -u
out=gpurun_out/ab_instep_p12.txt
: > $out
for i in 1 2 3 4; do
  for p in 10 12; do
    PKV_POLY_PAIRS=$p timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_line.json 2> /dev/null
    python - "poly$p" >> $out <<'PY'
import json, sys
d = json.loads(open("gpurun_out/ab_line.json").read().strip().splitlines()[-1])
lv = d.get("stages_live_ms", {})
print(f"{sys.argv[1]:<8} step {d['ms_per_step']:7.2f} ms  lse {lv.get('score_lse', 0):6.1f}  pool {lv.get('score_pool', 0):5.1f}  "
      f"map {lv.get('map', 0):6.1f}  clock {d['clocks']['sm_mhz']}")
PY
  done
done
