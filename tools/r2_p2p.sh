#!/bin/bash
mkdir -p gpurun_out
tag=${1:-p2}
G=$(nvidia-smi -L | wc -l)
nvidia-smi topo -m > gpurun_out/${tag}_topo.txt 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$G --master-addr=127.0.0.1 --master-port=29533 tools/shard_check.py --c5 --out gpurun_out/${tag}_shard_check_g${G}.json > gpurun_out/${tag}_shard_check_g${G}.log 2>&1
echo "shard_check rc=$?" >> gpurun_out/${tag}_shard_check_g${G}.log
for r in 1 2; do
for ex in auto nccl; do NCCL_DEBUG=WARN timeout 600 python bench.py --config c5 --gpus $G --exchange $ex --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --traffic off --watchdog 400 > gpurun_out/${tag}_bench_c5_n${G}_${ex}_$r.json 2> gpurun_out/${tag}_bench_c5_n${G}_${ex}_$r.err; done
done
echo done
