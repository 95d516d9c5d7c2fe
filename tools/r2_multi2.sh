#!/bin/bash
# multi-GPU round check: sharded parity (c5 full size), GPU shard tests, bench c3 weak scaling
# and c5 (both exchanges) at N=1 and N=G (tag = prefix)
mkdir -p gpurun_out
tag=${1:-m}
G=$(nvidia-smi -L | wc -l)
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$G --master-addr=127.0.0.1 --master-port=29533 tools/shard_check.py --c5 --out gpurun_out/${tag}_shard_check_g${G}.json > gpurun_out/${tag}_shard_check_g${G}.log 2>&1
echo "shard_check rc=$?" >> gpurun_out/${tag}_shard_check_g${G}.log
timeout 1200 python -m pytest tests/test_gpu_vocab_shard.py -q -rs > gpurun_out/${tag}_shard_tests_g${G}.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_shard_tests_g${G}.log
B="timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --traffic off"
$B > gpurun_out/${tag}_c3_n1.json 2>/dev/null
NCCL_DEBUG=WARN $B --gpus $G --watchdog 400 > gpurun_out/${tag}_c3_n${G}.json 2> gpurun_out/${tag}_c3_n${G}.err
$B --config c5 > gpurun_out/${tag}_c5_n1.json 2>/dev/null
for ex in auto nccl; do
  NCCL_DEBUG=WARN $B --config c5 --gpus $G --exchange $ex --watchdog 400 > gpurun_out/${tag}_c5_n${G}_${ex}.json 2> gpurun_out/${tag}_c5_n${G}_${ex}.err
done
echo done > gpurun_out/${tag}_done.txt
