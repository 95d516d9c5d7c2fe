#!/bin/bash
# timing variants of the c3 step (experiments; results on stdout)
run() { timeout 300 env "$@" python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$*', round(d['value']), round(d['ms_per_step']*1000,1), round(d['roofline']['kernel_us'],1), d['gpu_launches'])"; }
run A=1
run COSINE_NOFUSE=1
