#!/bin/bash
# Round-2 experiment: parity of the single-launch verify kernel, occupancy 6 vs 5, ncu bytes.
mkdir -p gpurun_out
tag=${1:-e2}
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/${tag}_parity.log 2>&1
echo "parity rc=$?" >> gpurun_out/${tag}_parity.log
for r in 1 2; do
  timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --traffic off > gpurun_out/${tag}_occ6_$r.json 2> gpurun_out/${tag}_occ6_$r.err
  COSINE_EXP_OCC5=1 timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --traffic off > gpurun_out/${tag}_occ5_$r.json 2> gpurun_out/${tag}_occ5_$r.err
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:verify_kernel -c 3 --csv --log-file gpurun_out/${tag}_ncu_occ6.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --traffic off > gpurun_out/${tag}_ncu6.log 2>&1
COSINE_EXP_OCC5=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:verify_kernel -c 3 --csv --log-file gpurun_out/${tag}_ncu_occ5.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --traffic off > gpurun_out/${tag}_ncu5.log 2>&1
echo done
