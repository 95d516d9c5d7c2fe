#!/bin/bash
# end-of-round profiles: launch lists of one call per config and --set full captures of the
# c3 statistics and resample kernels and the c2 one-launch kernel (tag = prefix)
mkdir -p gpurun_out
tag=${1:-p}
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k one_launch > gpurun_out/${tag}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_tests.log
bash tools/r2_ncu_lists.sh ${tag}
F='timeout 900 ncu --target-processes all --set full --import-source on --clock-control none'
$F -k regex:stats_kernel -s 3 -c 1 -o gpurun_out/${tag}_stats_c3 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --traffic off > gpurun_out/${tag}_full1.log 2>&1
$F -k regex:resample_kernel -s 3 -c 1 -o gpurun_out/${tag}_resample_c3 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --traffic off > gpurun_out/${tag}_full2.log 2>&1
$F -k regex:tiny_kernel -s 3 -c 1 -o gpurun_out/${tag}_tiny_c2 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --traffic off > gpurun_out/${tag}_full3.log 2>&1
for r in stats_c3 resample_c3 tiny_c2; do
  ncu -i gpurun_out/${tag}_$r.ncu-rep --page raw --csv > gpurun_out/${tag}_${r}_raw.csv 2>/dev/null
done
echo done > gpurun_out/${tag}_done.txt
