#!/bin/bash
# One GPU-box pass: GPU tests, smoke, the bench line, the reference arm, the
# ncu launch list of the bench command and one full capture of the round-2
# kernels (tools/ncu_targets.py). Outputs under gpurun_out/.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.txt 2>&1; echo "TESTS_EXIT=$?" >> gpurun_out/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "SMOKE_EXIT=$?" >> gpurun_out/smoke.txt
timeout 600 python bench.py > gpurun_out/bench_line.json 2> gpurun_out/bench_err.txt; echo "BENCH_EXIT=$?" >> gpurun_out/bench_err.txt
timeout 600 python tools/config_sweep.py > gpurun_out/config_sweep.jsonl 2> gpurun_out/sweep_err.txt
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_plain.log 2>&1 &&
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
timeout 300 python tools/ncu_targets.py > gpurun_out/targets_plain.log 2>&1 &&
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k 'regex:tridiag_reduce|tridiag_bisect|tridiag_vectors|chol_panel|gram_stream_kernel|gram_mode0|gram_mid|proj2_kernel|quad_|field_stat|field_apply' \
  -c 40 -o gpurun_out/r2_targets python tools/ncu_targets.py > gpurun_out/ncu_targets.log 2>&1
echo done
