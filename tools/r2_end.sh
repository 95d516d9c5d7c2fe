#!/bin/bash
# the driver's round-end sequence on one GPU: smoke, full GPU suite, default bench, reference arm
mkdir -p gpurun_out
tag=${1:-e1}
bash tools/r2_final.sh $tag
PARITY_LOG=gpurun_out/${tag}_parity_counts.jsonl timeout 2400 python -m pytest tests -q -m gpu -x -rs > gpurun_out/${tag}_gpu_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_gpu_tests.log
