#!/bin/bash
set -u
mkdir -p gpurun_out
K='regex:^(fused3|tail3|tail4|quad|gram|tridiag|chol|proj2|gemm|rank_rule|sumsq|sum_partials|basis_defect|take_columns|expand|decode2|cholqr2|orthonormalize|pair_project|mode_small|pad_axis|fill|unfold|field|permute|posdef|jacobi|diff_sumsq)'
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "balanced4 or config3 or leading_modes or adaptive or stream_random" > gpurun_out/t4_tests.txt 2>&1; echo "EXIT=$?" >> gpurun_out/t4_tests.txt
timeout 600 python -m pytest tests/test_gpu_stream.py tests/test_gpu_multirank.py -x -q > gpurun_out/t4_tests2.txt 2>&1; echo "EXIT=$?" >> gpurun_out/t4_tests2.txt
timeout 300 python tools/stream_breakdown.py c2 c3 c4 c5 > gpurun_out/stream_breakdown.txt 2>&1
timeout 300 python tools/bht_breakdown.py c1 > gpurun_out/bht_c1.txt 2>&1
timeout 300 python tools/bht_breakdown.py c5 > gpurun_out/bht_c5.txt 2>&1
timeout 300 python tools/config_sweep.py --configs c2,c3 > gpurun_out/sweep_c23.jsonl 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_plain.log 2>&1 &&
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
timeout 300 python tools/ncu_targets_update.py > gpurun_out/targets_plain.log 2>&1 &&
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k 'regex:^(fused3|tail3|tail4|quad|field|expand|decode2)' \
  -c 40 -o gpurun_out/r2_update_targets python tools/ncu_targets_update.py > gpurun_out/ncu_targets.log 2>&1
echo done
