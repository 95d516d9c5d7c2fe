#!/bin/bash
mkdir -p gpurun_out
tag=${1:-s2}
G=$(nvidia-smi -L | wc -l)
for sl in 1 2 4 8; do
  COSINE_EXP_SLICES=$sl NCCL_DEBUG=WARN timeout 600 python bench.py --config c5 --gpus $G --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --traffic off --watchdog 400 > gpurun_out/${tag}_bench_c5_n${G}_sl${sl}.json 2> gpurun_out/${tag}_bench_c5_n${G}_sl${sl}.err
done
echo done
