#!/bin/bash
mkdir -p gpurun_out
tag=${1:-cs1}
for cs in 4 8 16; do
  timeout 300 python bench.py --config c3 --cluster-size $cs --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --traffic off > gpurun_out/${tag}_C${cs}_c3.json 2> gpurun_out/${tag}_C${cs}_c3.err
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:stats_kernel -s 3 -c 1 -o gpurun_out/${tag}_stats_c3 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --traffic off > gpurun_out/${tag}_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:resample_kernel -s 3 -c 1 -o gpurun_out/${tag}_resample_c3 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --traffic off > gpurun_out/${tag}_ncu2.log 2>&1
echo done
