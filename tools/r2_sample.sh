#!/bin/bash
mkdir -p gpurun_out
tag=${1:-sm1}
PARITY_LOG=gpurun_out/${tag}_parity_counts.jsonl timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_entrypoints.py -q -x > gpurun_out/${tag}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_tests.log
for sel in argmax sample; do
  timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --traffic off --select $sel > gpurun_out/${tag}_bench_${sel}.json 2> gpurun_out/${tag}_bench_${sel}.err
done
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --traffic off --weights point > gpurun_out/${tag}_bench_point.json 2> gpurun_out/${tag}_bench_point.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 9 -k regex:"stats_kernel|decide_kernel|resample_kernel" --csv --log-file gpurun_out/${tag}_ncu_sample.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --traffic off --select sample > gpurun_out/${tag}_ncu_sample.log 2>&1
echo done
