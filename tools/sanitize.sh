#!/bin/bash
# compute-sanitizer over the GPU path: memcheck,
# racecheck (shared-memory hazards incl. the mbarrier/TMEM pipelines'
# smem staging), synccheck and initcheck on the whole-path smoke (score ->
# map -> select -> compact through pkv_pruner_run), memcheck additionally on
# the tiny-config pruner / scoring / kernel / decode parity tests.
# Logs: gpurun_out/sanitizer_<tool>.log (summaries copied to profiles/).
set -u
OUT=${1:-gpurun_out}
mkdir -p "$OUT"
CS="compute-sanitizer --print-limit 50 --error-exitcode 9"
SMOKE="python -c 'import __graft_entry__ as g; g.smoke()'"
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
  echo "== $tool: smoke" > "$OUT/sanitizer_$tool.log"
  eval timeout 480 $CS --tool $tool $extra $SMOKE >> "$OUT/sanitizer_$tool.log" 2>&1
  echo "exit=$?" >> "$OUT/sanitizer_$tool.log"
done
echo "== memcheck: parity tests" >> "$OUT/sanitizer_memcheck.log"
timeout 900 $CS --tool memcheck python -m pytest -q -x tests/test_pruner_gpu.py tests/test_score_gpu.py \
  tests/test_kernels_gpu.py tests/test_decode_gpu.py tests/test_select_f64_gpu.py >> "$OUT/sanitizer_memcheck.log" 2>&1
echo "exit=$?" >> "$OUT/sanitizer_memcheck.log"
# round 2 additions: GPU training, mapper precision mode 6 (e4m3 corrections), the streaming select
echo "== memcheck: training / mode 6 / streaming select" >> "$OUT/sanitizer_memcheck.log"
timeout 900 $CS --tool memcheck python -m pytest -q -x tests/test_train_gpu.py tests/test_select_compact_gpu.py \
  "tests/test_mapper_gpu.py::test_fp16f8_mode_small_and_multiwindow" >> "$OUT/sanitizer_memcheck.log" 2>&1
echo "exit=$?" >> "$OUT/sanitizer_memcheck.log"
