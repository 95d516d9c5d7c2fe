#!/bin/bash
# full GPU test suite with parity counts collected (tag = output prefix)
mkdir -p gpurun_out
tag=${1:-t1}
nproc > gpurun_out/${tag}_nproc.txt
rm -f gpurun_out/${tag}_parity_counts.jsonl
PARITY_LOG=gpurun_out/${tag}_parity_counts.jsonl timeout 2400 python -m pytest tests -q -m gpu -x -rs --durations=15 > gpurun_out/${tag}_gpu_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_gpu_tests.log
