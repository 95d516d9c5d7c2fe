#!/bin/bash
# every single-GPU bench line of DESIGN §8 and the launch lists (tag = prefix)
mkdir -p gpurun_out
tag=${1:-a1}
B="timeout 600 python bench.py"
$B > gpurun_out/${tag}_c3.json 2> gpurun_out/${tag}_c3.err
$B --select sample --no-cpu-baseline > gpurun_out/${tag}_c3_sample.json 2>/dev/null
$B --weights point --no-cpu-baseline > gpurun_out/${tag}_c3_point.json 2>/dev/null
$B --lazy --no-cpu-baseline > gpurun_out/${tag}_c3_lazy.json 2>/dev/null
$B --config c4 --no-cpu-baseline > gpurun_out/${tag}_c4.json 2>/dev/null
$B --config c4 --lazy --no-cpu-baseline > gpurun_out/${tag}_c4_lazy.json 2>/dev/null
$B --config c2 --steps 50 --no-cpu-baseline > gpurun_out/${tag}_c2.json 2>/dev/null
$B --config c1 --steps 50 --no-cpu-baseline > gpurun_out/${tag}_c1.json 2>/dev/null
$B --config c5 --no-cpu-baseline > gpurun_out/${tag}_c5.json 2>/dev/null
N="timeout 600 ncu --target-processes all --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"stats_kernel|decide|resample|tiny_kernel|tree_|shard_|fuse_|sample_" --csv"
$N -c 12 --log-file gpurun_out/${tag}_launches_c3.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --traffic off > /dev/null 2>&1
$N -c 12 --log-file gpurun_out/${tag}_launches_c3_sample.csv python bench.py --select sample --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --traffic off > /dev/null 2>&1
$N -c 12 --log-file gpurun_out/${tag}_launches_c4.csv python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --traffic off > /dev/null 2>&1
$N -c 12 --log-file gpurun_out/${tag}_launches_c2.csv python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --traffic off > /dev/null 2>&1
$N -c 12 --log-file gpurun_out/${tag}_launches_c1.csv python bench.py --config c1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --traffic off > /dev/null 2>&1
echo done > gpurun_out/${tag}_done.txt
