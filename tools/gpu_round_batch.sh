set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score_lse_kernel -s 4 -c 1 -o gpurun_out/ncu_lse python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_lse.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sel_stream_kernel -s 2 -c 1 -o gpurun_out/ncu_sel python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_sel.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:compact_kv_kernel -s 2 -c 1 -o gpurun_out/ncu_compact python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_compact.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score_pool_kernel -s 4 -c 1 -o gpurun_out/ncu_pool python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_pool.log 2>&1
ls -la gpurun_out
