#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.txt 2>&1; echo "TESTS_EXIT=$?" >> gpurun_out/gpu_tests.txt
timeout 600 python tools/shape_sweep.py > gpurun_out/shape_sweep.jsonl 2> gpurun_out/shape_sweep_err.txt
timeout 300 python tools/bht_breakdown.py c5 > gpurun_out/bht_c5.txt 2>&1
timeout 300 python tools/stream_trace.py c3 > gpurun_out/trace_c3.txt 2>&1
timeout 300 python tools/stream_trace.py c2 > gpurun_out/trace_c2.txt 2>&1
timeout 300 python tools/stream_trace.py c4 > gpurun_out/trace_c4.txt 2>&1
HTR_TIMELINE=1 timeout 300 python tools/stream_overhead.py 12 c3 > gpurun_out/overhead_c3.txt 2>&1
timeout 600 python tools/config_sweep.py > gpurun_out/config_sweep.jsonl 2> gpurun_out/sweep_err.txt
echo done
