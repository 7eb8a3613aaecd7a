#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "pair_projection or config5 or config1 or streaming_gram or mode0_gram" > gpurun_out/gpu_tests_d.txt 2>&1; echo "TESTS_EXIT=$?" >> gpurun_out/gpu_tests_d.txt
timeout 300 python tools/bht_breakdown.py c5 > gpurun_out/bht_c5.txt 2>&1
timeout 300 python tools/stream_breakdown.py c3+30 c3 > gpurun_out/stream_breakdown_c3g.txt 2>&1
echo done
