#!/bin/bash
# multi-GPU checks on a G-GPU box: sharded parity over NCCL (incl. c5 full size), bench c3 weak
# scaling and c5 strong scaling at N=1 and N=G (bench self-launches its ranks)
mkdir -p gpurun_out
tag=${1:-m2}
G=$(nvidia-smi -L | wc -l)
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$G --master-addr=127.0.0.1 --master-port=29533 tools/shard_check.py --c5 --out gpurun_out/${tag}_shard_check_g${G}.json > gpurun_out/${tag}_shard_check_g${G}.log 2>&1
echo "shard_check rc=$?" >> gpurun_out/${tag}_shard_check_g${G}.log
for cfg in c3 c5; do
  timeout 600 python bench.py --config $cfg --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --traffic off > gpurun_out/${tag}_bench_${cfg}_n1.json 2> gpurun_out/${tag}_bench_${cfg}_n1.err
  NCCL_DEBUG=WARN timeout 600 python bench.py --config $cfg --gpus $G --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --traffic off --watchdog 400 > gpurun_out/${tag}_bench_${cfg}_n${G}.json 2> gpurun_out/${tag}_bench_${cfg}_n${G}.err
done
echo done
