#!/bin/bash
# small-config latency: chunk-count sweep for c1 / c2 and their launch lists (tag = prefix)
mkdir -p gpurun_out
tag=${1:-m1}
for cfg in c1 c2; do
  for cs in 0 1 2 4 8 16; do
    echo "$cfg cs=$cs $(timeout 300 python bench.py --config $cfg --cluster-size $cs --steps 50 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; a=json.loads(sys.stdin.read()); print(a["ms_per_step"]*1e3, a["roofline"]["kernel_us"])')" >> gpurun_out/${tag}_sweep.txt
  done
done
for cfg in c1 c2; do
  timeout 300 ncu --target-processes all --metrics gpu__time_duration.sum --clock-control none -k regex:cosine -c 12 --csv --log-file gpurun_out/${tag}_launches_$cfg.csv python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
echo done
