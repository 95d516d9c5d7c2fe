#!/bin/bash
# c1 / c2: one-launch (tiny_kernel) vs split path (--cluster-size forces it) and ncu of tiny_kernel
mkdir -p gpurun_out
tag=${1:-y2}
for cfg in c1 c2; do
  for cs in 0 1 4 16; do
    echo "$cfg cs=$cs $(timeout 300 python bench.py --config $cfg --cluster-size $cs --steps 50 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; a=json.loads(sys.stdin.read()); print(a["ms_per_step"]*1e3, a["gpu_launches"], a["roofline"]["kernel_us"])')" >> gpurun_out/${tag}_sweep.txt
  done
done
timeout 300 ncu --target-processes all --metrics gpu__time_duration.sum --clock-control none -k regex:"tiny|stats|decide|resample" -c 20 --csv --log-file gpurun_out/${tag}_launches_c1.csv python bench.py --config c1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_ncu1.log 2>&1
timeout 600 ncu --target-processes all --set full --import-source on --clock-control none -k regex:tiny -s 3 -c 1 -o gpurun_out/${tag}_tiny_c1 python bench.py --config c1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_ncu2.log 2>&1
echo done
