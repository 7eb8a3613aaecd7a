#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 1500 python tools/full_parity.py c5 --batches 40 --compare all > gpurun_out/full_parity_c5.jsonl 2> gpurun_out/full_parity_c5_err.txt; echo "EXIT=$?" >> gpurun_out/full_parity_c5_err.txt
timeout 600 python tools/full_parity.py c4 --batches 10 --compare all > gpurun_out/full_parity_c4.jsonl 2> gpurun_out/full_parity_c4_err.txt; echo "EXIT=$?" >> gpurun_out/full_parity_c4_err.txt
echo done
