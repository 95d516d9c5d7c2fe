#!/bin/bash
mkdir -p gpurun_out
tag=${1:-d2}
G=$(nvidia-smi -L | wc -l)
NCCL_DEBUG=WARN timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$G --master-addr=127.0.0.1 --master-port=29541 bench.py --gpus $G --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --traffic off --watchdog 150 > gpurun_out/${tag}_direct.json 2> gpurun_out/${tag}_direct.err
echo "direct rc=$?" >> gpurun_out/${tag}_direct.err
NCCL_DEBUG=WARN timeout 300 python bench.py --gpus $G --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --traffic off --watchdog 150 > gpurun_out/${tag}_self.json 2> gpurun_out/${tag}_self.err
echo "self rc=$?" >> gpurun_out/${tag}_self.err
