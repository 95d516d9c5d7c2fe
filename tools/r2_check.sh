#!/bin/bash
# bench lines c3 (ARGMAX, SAMPLE), c1, c2 and the full GPU suite (tag = prefix)
mkdir -p gpurun_out
tag=${1:-k1}
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_c3.json 2> gpurun_out/${tag}_c3.err
timeout 300 python bench.py --select sample --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_c3s.json 2> gpurun_out/${tag}_c3s.err
for cfg in c1 c2; do
  timeout 300 python bench.py --config $cfg --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_$cfg.json 2> gpurun_out/${tag}_$cfg.err
done
if [ "$2" != "notests" ]; then
PARITY_LOG=gpurun_out/${tag}_parity_counts.jsonl timeout 2400 python -m pytest tests -q -m gpu -x -rs > gpurun_out/${tag}_gpu_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_gpu_tests.log
fi
