#!/bin/bash
# c3 chunk-count sweep (CTAs per unit of the statistics pass; tag = prefix)
mkdir -p gpurun_out
tag=${1:-cs}
for cs in 0 2 4 8 16; do
  timeout 300 python bench.py --cluster-size $cs --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_cs$cs.json 2>/dev/null
  timeout 300 python bench.py --select sample --cluster-size $cs --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_s_cs$cs.json 2>/dev/null
done
