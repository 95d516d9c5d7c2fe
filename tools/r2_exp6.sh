#!/bin/bash
mkdir -p gpurun_out
tag=${1:-e6}
export COSINE_EXP_OCC5=1
for C in 4 8; do
  TRACE_C=$C timeout 300 python tools/trace_verify.py c3 gpurun_out/${tag}_trace_C${C}_o5.pt > gpurun_out/${tag}_trace_C${C}_o5.json 2>&1
done
echo done
