#!/bin/bash
mkdir -p gpurun_out
tag=${1:-e9}
export COSINE_EXP_OCC5=1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/${tag}_parity.log 2>&1
echo "parity rc=$?" >> gpurun_out/${tag}_parity.log
COSINE_EXP_SPLIT3=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/${tag}_parity3.log 2>&1
echo "parity3 rc=$?" >> gpurun_out/${tag}_parity3.log
for r in 1 2; do
for cfg in c3 c2; do
  timeout 300 python bench.py --config $cfg --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --traffic off > gpurun_out/${tag}_C0_o5_${cfg}_$r.json 2> gpurun_out/${tag}_C0_o5_${cfg}.err
  COSINE_EXP_SPLIT3=1 timeout 300 python bench.py --config $cfg --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --traffic off > gpurun_out/${tag}_C0_s3_${cfg}_$r.json 2> gpurun_out/${tag}_C0_s3_${cfg}.err
done
done
TRACE_C=0 timeout 300 python tools/trace_verify.py c3 gpurun_out/${tag}_trace_C0_o5.pt > gpurun_out/${tag}_trace_C0_o5.json 2>&1
COSINE_EXP_SPLIT3=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 12 -k regex:"stats_kernel|decide_kernel|resample_kernel" --csv --log-file gpurun_out/${tag}_ncu_s3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --traffic off > gpurun_out/${tag}_ncu_s3.log 2>&1
echo done
