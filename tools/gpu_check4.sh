#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.txt 2>&1; echo "TESTS_EXIT=$?" >> gpurun_out/gpu_tests.txt
timeout 600 python tools/config_sweep.py > gpurun_out/config_sweep.jsonl 2> gpurun_out/sweep_err.txt
timeout 300 python tools/stream_breakdown.py c2 c3 c4 c5 > gpurun_out/stream_breakdown.txt 2>&1
timeout 600 python tools/shape_sweep.py > gpurun_out/shape_sweep.jsonl 2> gpurun_out/shape_sweep_err.txt
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick_err.txt
echo done
