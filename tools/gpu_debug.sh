#!/bin/bash
set -u
mkdir -p gpurun_out
for i in 0 1 2 3 4 5 6 7; do
  timeout 200 python -X faulthandler -m pytest tests/test_gpu_parity.py -x -q -o faulthandler_timeout=90 -k "balanced4_fused_tail_cases and dims$i-" > gpurun_out/dbg_$i.txt 2>&1; echo "EXIT=$?" >> gpurun_out/dbg_$i.txt
done
echo done
