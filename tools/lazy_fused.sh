#!/bin/bash
run() { timeout 300 env "$@" python bench.py --lazy --steps 30 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$*', round(d['value']), round(d['ms_per_step']*1000,1))"; }
run COSINE_LAZY_FUSED=1
run COSINE_LAZY_FUSED=0
run COSINE_LAZY_FUSED=1
