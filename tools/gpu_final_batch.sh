# Round-end evidence on one B200: the GPU suite, smoke, the default bench line, the
# mode-6 bench line, the reference arm and the extra legs (tools/gpu_final_batch.sh;
# outputs under gpurun_out/).
set -x
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/final_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo smoke_exit=$? >> gpurun_out/final_smoke.log
timeout 600 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
timeout 600 python bench.py --precision 6 --no-cpu-baseline > gpurun_out/final_bench_p6.json 2> gpurun_out/final_bench_p6.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err
timeout 900 python bench.py --extras --steps 5 --no-cpu-baseline > gpurun_out/final_bench_extras.json 2> gpurun_out/final_bench_extras.err
