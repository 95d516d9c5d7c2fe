#!/bin/bash
# latency traces of the one-launch kernel (tools/tiny_trace.py), cooperative and not (tag = prefix)
mkdir -p gpurun_out
tag=${1:-tr}
out=gpurun_out/${tag}.txt
: > $out
for v in "" noncoop; do
  for cfg in c1 c2; do
    TRACE_VARIANT=$v timeout 300 python tools/tiny_trace.py run $cfg >> $out 2>&1
    TRACE_VARIANT=$v timeout 300 python tools/tiny_trace.py run $cfg noflush >> $out 2>&1
  done
done
