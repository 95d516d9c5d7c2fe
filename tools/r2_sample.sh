#!/bin/bash
# SAMPLE-selection parity tests and the SAMPLE bench line (tag = output prefix)
mkdir -p gpurun_out
tag=${1:-s1}
PARITY_LOG=gpurun_out/${tag}_parity_counts.jsonl timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_entrypoints.py -q -x -k "sample or select or chunking or ragged" > gpurun_out/${tag}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_tests.log
timeout 600 python bench.py --select sample --steps 20 --warmup 5 > gpurun_out/${tag}_bench_sample.json 2> gpurun_out/${tag}_bench_sample.err
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${tag}_bench_argmax.json 2> gpurun_out/${tag}_bench_argmax.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:cosine -c 40 --csv --log-file gpurun_out/${tag}_launches.csv python bench.py --select sample --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo done
