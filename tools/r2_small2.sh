#!/bin/bash
mkdir -p gpurun_out
tag=${1:-sc2}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_entrypoints.py -q -x > gpurun_out/${tag}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_tests.log
for m in 0 1; do
for cfg in c1 c2 c3; do
  COSINE_EXP_MERGED=$m timeout 300 python bench.py --config $cfg --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --traffic off > gpurun_out/${tag}_m${m}_${cfg}.json 2> gpurun_out/${tag}_m${m}_${cfg}.err
done
done
echo done
