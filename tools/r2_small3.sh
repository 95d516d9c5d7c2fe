#!/bin/bash
mkdir -p gpurun_out
tag=${1:-sc3}
for cfg in c1 c2; do
for cs in 1 2 4 8 16; do
  timeout 300 python bench.py --config $cfg --cluster-size $cs --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --traffic off > gpurun_out/${tag}_C${cs}_${cfg}.json 2> gpurun_out/${tag}_C${cs}_${cfg}.err
done
done
echo done
