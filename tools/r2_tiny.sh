#!/bin/bash
# one-launch small-batch path: c1 / c2 bench lines, then the full GPU suite (tag = prefix)
mkdir -p gpurun_out
tag=${1:-y1}
for cfg in c1 c2; do
  timeout 300 python bench.py --config $cfg --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/${tag}_bench_$cfg.json 2> gpurun_out/${tag}_bench_$cfg.err
done
PARITY_LOG=gpurun_out/${tag}_parity_counts.jsonl timeout 2400 python -m pytest tests -q -m gpu -x -rs > gpurun_out/${tag}_gpu_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_gpu_tests.log
