#!/bin/bash
# One GPU-box pass (gpurun -- 'bash tools/gpu_check.sh'): GPU tests, smoke,
# the bench line, the per-config and per-shape sweeps, the ncu launch list of
# the bench command (this library's kernels only) and full captures of the
# BHT-l2r and skip-update kernels. Outputs under gpurun_out/; the summaries
# committed under profiles/ are made from them with tools/ncu_multi_summary.py.
set -u
mkdir -p gpurun_out
K='regex:^(fused3|tail3|tail4|quad|gram|tridiag|chol|proj2|gemm|rank_rule|sumsq|sum_partials|basis_defect|take_columns|expand|decode2|cholqr2|orthonormalize|pair_project|mode_small|pad_axis|fill|unfold|field|permute|posdef|jacobi|diff_sumsq|splitk|sym_mirror)'
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.txt 2>&1; echo "TESTS_EXIT=$?" >> gpurun_out/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "SMOKE_EXIT=$?" >> gpurun_out/smoke.txt
timeout 600 python bench.py > gpurun_out/bench_line.json 2> gpurun_out/bench_err.txt; echo "BENCH_EXIT=$?" >> gpurun_out/bench_err.txt
timeout 600 python tools/config_sweep.py > gpurun_out/config_sweep.jsonl 2> gpurun_out/sweep_err.txt
timeout 600 python tools/shape_sweep.py > gpurun_out/shape_sweep.jsonl 2> gpurun_out/shape_sweep_err.txt
timeout 300 python tools/stream_breakdown.py c2 c3 c4 c5 > gpurun_out/stream_breakdown.txt 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_plain.log 2>&1 &&
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
timeout 300 python tools/ncu_targets.py c5 c1 > gpurun_out/targets_plain.log 2>&1 &&
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k 'regex:^(tridiag_reduce|tridiag_bisect|tridiag_vectors|chol_panel|gram_stream|gram_mode0|gram_mid|proj2|gemm_fast)' \
  -c 40 -o /tmp/r2_targets python tools/ncu_targets.py c5 c1 > gpurun_out/ncu_targets.log 2>&1
# (the reports are summarised here: gpurun brings back at most 64 MiB)
python tools/ncu_multi_summary.py /tmp/r2_targets.ncu-rep > gpurun_out/r2_bht_kernels_ncu_summary.txt 2>&1
for k in gram_stream tridiag_reduce tridiag_vectors proj2; do
  echo "== $k" >> gpurun_out/r2_bht_kernels_ncu_lines.txt
  python tools/ncu_lines.py /tmp/r2_targets.ncu-rep $k 12 >> gpurun_out/r2_bht_kernels_ncu_lines.txt 2>&1
done
timeout 300 python tools/ncu_targets_update.py > gpurun_out/targets_update_plain.log 2>&1 &&
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k 'regex:^(fused3|tail3|tail4|quad|field|expand|decode2)' \
  -c 40 -o /tmp/r2_update_targets python tools/ncu_targets_update.py > gpurun_out/ncu_update_targets.log 2>&1
python tools/ncu_multi_summary.py /tmp/r2_update_targets.ncu-rep > gpurun_out/r2_update_kernels_ncu_summary.txt 2>&1
for k in fused3_kernel tail3_kernel tail4_kernel quad_stream; do
  echo "== $k" >> gpurun_out/r2_update_kernels_ncu_lines.txt
  python tools/ncu_lines.py /tmp/r2_update_targets.ncu-rep $k 12 >> gpurun_out/r2_update_kernels_ncu_lines.txt 2>&1
done
echo done
