#!/bin/bash
# the driver's round-end commands (one GPU): smoke, the default bench line, the reference arm
mkdir -p gpurun_out
tag=${1:-f1}
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/${tag}_smoke.log
start=$(date +%s)
timeout 1200 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
echo "bench rc=$? seconds=$(( $(date +%s) - start ))" >> gpurun_out/${tag}_bench.err
start=$(date +%s)
timeout 1200 python bench.py --impl reference > gpurun_out/${tag}_ref.json 2> gpurun_out/${tag}_ref.err
echo "ref rc=$? seconds=$(( $(date +%s) - start ))" >> gpurun_out/${tag}_ref.err
nproc > gpurun_out/${tag}_nproc.txt
