#!/bin/bash
# ncu launch lists (durations, DRAM bytes) of one call per config (tag = prefix)
mkdir -p gpurun_out
tag=${1:-n1}
N='timeout 600 ncu --target-processes all --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:stats_kernel|decide|resample|tiny_kernel|tree_|shard_|fuse_|sample_ --csv'
for cfg in c3 c4 c2 c1; do
  $N -c 12 --log-file gpurun_out/${tag}_launches_$cfg.csv python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --traffic off > gpurun_out/${tag}_ncu_$cfg.log 2>&1
done
$N -c 12 --log-file gpurun_out/${tag}_launches_c3_sample.csv python bench.py --select sample --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --traffic off > /dev/null 2>&1
$N -c 40 --log-file gpurun_out/${tag}_launches_c4_lazy.csv python bench.py --config c4 --lazy --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --traffic off > /dev/null 2>&1
