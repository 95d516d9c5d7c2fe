#!/bin/bash
mkdir -p gpurun_out
tag=${1:-c5p}
timeout 300 python tools/c5_vgroup_prof.py 4 > gpurun_out/${tag}_run.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"stats_kernel|shard_|resample" -c 40 --csv --log-file gpurun_out/${tag}_launches.csv python tools/c5_vgroup_prof.py 4 > gpurun_out/${tag}_ncu.log 2>&1
