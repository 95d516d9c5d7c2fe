#!/bin/bash
# ncu --set full capture of one launch of a kernel of bench.py (args: tag kernel-regex bench-args...)
tag=$1; kre=$2; shift 2
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$kre" -s 3 -c 1 \
  -o gpurun_out/$tag -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --traffic off "$@" \
  > gpurun_out/$tag.log 2>&1
echo "ncu rc=$?" >> gpurun_out/$tag.log
