#!/bin/bash
mkdir -p gpurun_out
tag=${1:-e3}
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/${tag}_parity.log 2>&1
echo "parity rc=$?" >> gpurun_out/${tag}_parity.log
timeout 300 python tools/trace_verify.py c3 gpurun_out/${tag}_trace_c3.pt > gpurun_out/${tag}_trace_c3.json 2>&1
COSINE_EXP_OCC5=1 timeout 300 python tools/trace_verify.py c3 gpurun_out/${tag}_trace_c3_occ5.pt > gpurun_out/${tag}_trace_c3_occ5.json 2>&1
timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --traffic off > gpurun_out/${tag}_occ6.json 2> gpurun_out/${tag}_occ6.err
COSINE_EXP_OCC5=1 timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --traffic off > gpurun_out/${tag}_occ5.json 2> gpurun_out/${tag}_occ5.err
echo done
