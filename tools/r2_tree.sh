#!/bin/bash
# tree (c4) benches and the tree / lazy GPU tests (tag = prefix)
mkdir -p gpurun_out
tag=${1:-t1}
timeout 300 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_c4.json 2>/dev/null
timeout 300 python bench.py --config c4 --lazy --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_c4_lazy.json 2>/dev/null
timeout 900 python -m pytest tests/test_gpu_tree.py tests/test_gpu_lazy.py tests/test_gpu_tree_select.py -q -x > gpurun_out/${tag}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_tests.log
