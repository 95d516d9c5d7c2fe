#!/bin/bash
mkdir -p gpurun_out
tag=${1:-e10}
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/${tag}_parity.log 2>&1
echo "parity rc=$?" >> gpurun_out/${tag}_parity.log
COSINE_EXP_PAIR=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/${tag}_parityP.log 2>&1
echo "parityP rc=$?" >> gpurun_out/${tag}_parityP.log
for r in 1 2; do
for cfg in c3 c2; do
  timeout 300 python bench.py --config $cfg --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --traffic off > gpurun_out/${tag}_base_${cfg}_$r.json 2> gpurun_out/${tag}_base_${cfg}.err
  COSINE_EXP_PAIR=1 timeout 300 python bench.py --config $cfg --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --traffic off > gpurun_out/${tag}_pair_${cfg}_$r.json 2> gpurun_out/${tag}_pair_${cfg}.err
done
done
for v in base pair; do
  if [ $v = pair ]; then export COSINE_EXP_PAIR=1; else unset COSINE_EXP_PAIR; fi
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 12 -k regex:"stats_kernel|decide_kernel|resample_kernel" --csv --log-file gpurun_out/${tag}_ncu_$v.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --traffic off > gpurun_out/${tag}_ncu_$v.log 2>&1
done
echo done
