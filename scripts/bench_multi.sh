#!/bin/bash
# End-of-round bench lines at n = 2 and 4 (configs 2, 4, 5; config 2 also with NCCL_ALGO=Ring for
# the dense baseline), each JSON line into gpurun_out/bench_n<n>_c<config>[_ring].json
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for n in ${NS:-2 4}; do
  for c in 2 4 5; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n --steps 30 --warmup 5 --config $c \
      > gpurun_out/bench_n${n}_c${c}.log 2>&1
    grep '^{' gpurun_out/bench_n${n}_c${c}.log | tail -1 > gpurun_out/bench_n${n}_c${c}.json
    echo "n=$n c=$c $(python -c "import json; d=json.load(open('gpurun_out/bench_n${n}_c${c}.json')); print(d['ms_per_step'], d['value'])" 2>&1 | tail -1)"
  done
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n --steps 30 --warmup 5 --config 2 --nccl-algo ring \
    > gpurun_out/bench_n${n}_c2_ring.log 2>&1
  grep '^{' gpurun_out/bench_n${n}_c2_ring.log | tail -1 > gpurun_out/bench_n${n}_c2_ring.json
  echo "n=$n c=2 ring $(python -c "import json; d=json.load(open('gpurun_out/bench_n${n}_c2_ring.json')); print(d['ms_per_step'], d['value'])" 2>&1 | tail -1)"
done
