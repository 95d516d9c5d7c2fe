#!/bin/bash
mkdir -p gpurun_out
tag=${1:-sc1}
for cfg in c1 c2 c3; do
  timeout 300 python bench.py --config $cfg --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --traffic off > gpurun_out/${tag}_${cfg}.json 2> gpurun_out/${tag}_${cfg}.err
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -c 12 -k regex:"stats_kernel|decide_kernel|resample_kernel" --csv --log-file gpurun_out/${tag}_ncu_c2.csv python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --traffic off > gpurun_out/${tag}_ncu_c2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -c 12 -k regex:"stats_kernel|decide_kernel|resample_kernel" --csv --log-file gpurun_out/${tag}_ncu_c1.csv python bench.py --config c1 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --traffic off > gpurun_out/${tag}_ncu_c1.log 2>&1
echo done
