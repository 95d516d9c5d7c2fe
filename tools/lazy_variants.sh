#!/bin/bash
# lazy-mode round shapes on c3 (experiments)
run() { timeout 300 env "$@" python bench.py --lazy --steps 30 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$*', round(d['value']), round(d['ms_per_step']*1000,1), d['gpu_launches'], round(d['roofline']['achieved']))"; }
run COSINE_LAZY_C=8 COSINE_LAZY_SPAN=1
run COSINE_LAZY_C=16 COSINE_LAZY_SPAN=1
run COSINE_LAZY_C=16 COSINE_LAZY_SPAN=2
run COSINE_LAZY_C=8 COSINE_LAZY_SPAN=2
run COSINE_LAZY_C=16 COSINE_LAZY_SPAN=3
