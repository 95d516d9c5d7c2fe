#!/bin/bash
mkdir -p gpurun_out
tag=${1:-e7}
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/${tag}_parity.log 2>&1
echo "parity rc=$?" >> gpurun_out/${tag}_parity.log
for occ in 5 6; do
  if [ $occ = 5 ]; then export COSINE_EXP_OCC5=1; else unset COSINE_EXP_OCC5; fi
  for C in 0 8; do
    TRACE_C=$C timeout 300 python tools/trace_verify.py c3 gpurun_out/${tag}_trace_C${C}_o${occ}.pt > gpurun_out/${tag}_trace_C${C}_o${occ}.json 2>&1
    timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --traffic off --cluster-size $C > gpurun_out/${tag}_C${C}_o${occ}.json 2> gpurun_out/${tag}_C${C}_o${occ}.err
  done
done
export COSINE_EXP_OCC5=1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:verify_kernel -c 2 --csv --log-file gpurun_out/${tag}_ncu_o5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --traffic off > gpurun_out/${tag}_ncu5.log 2>&1
echo done
