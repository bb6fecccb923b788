# Encoder attention kernel times (one Llama/32k layer) under ncu for the default kernel, the
# no-exponential timing probe and the polynomial splits, after the attention kernel tests.
# Usage (on the GPU box): bash tools/time_attn_modes.sh  -> gpurun_out/attn_modes.log
t() { echo "== $1" >> gpurun_out/attn_modes.log; env $1 timeout 300 ncu --metrics gpu__time_duration.sum,smsp__cycles_elapsed.avg.per_second --clock-control none -k regex:attn_kernel -c 4 python tools/time_attn_clocked.py 2>&1 | grep -E "gpu__time_duration|cycles_elapsed" | tail -2 >> gpurun_out/attn_modes.log; }
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -k attention >> gpurun_out/attn_modes.log 2>&1
t PKV_ATTN_MODE=0
t PKV_ATTN_MODE=1
t PKV_ATTN_POLY=2
t PKV_ATTN_POLY=6
