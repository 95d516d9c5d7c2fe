#!/bin/bash
run() { timeout 300 env "$@" python bench.py --lazy --steps 30 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$*', round(d['value']), round(d['ms_per_step']*1000,1))"; }
run COSINE_LAZY_SPAN0=2 COSINE_LAZY_SPAN=2
run COSINE_LAZY_SPAN0=1 COSINE_LAZY_SPAN=2
run COSINE_LAZY_SPAN0=3 COSINE_LAZY_SPAN=2
run COSINE_LAZY_SPAN0=1 COSINE_LAZY_SPAN=3
run COSINE_LAZY_SPAN0=2 COSINE_LAZY_SPAN=3
