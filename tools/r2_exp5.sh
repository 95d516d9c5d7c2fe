#!/bin/bash
mkdir -p gpurun_out
tag=${1:-e5}
for C in 2 4 8; do
  for occ in 5 6; do
    if [ $occ = 5 ]; then export COSINE_EXP_OCC5=1; else unset COSINE_EXP_OCC5; fi
    TRACE_C=$C timeout 300 python tools/trace_verify.py c3 gpurun_out/${tag}_trace_C${C}_o${occ}.pt > gpurun_out/${tag}_trace_C${C}_o${occ}.json 2>&1
    timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --traffic off --cluster-size $C > gpurun_out/${tag}_C${C}_o${occ}.json 2> gpurun_out/${tag}_C${C}_o${occ}.err
  done
done
echo done
