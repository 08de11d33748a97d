#!/bin/bash
# Multi-GPU parity matrix (scripts/multi_gpu_check.py) at n = $1 GPUs for every gather mode; raw
# JSON lines land in gpurun_out/multi_n<n>_<mode>.json (commit them under profiles/round2/).
#   gpurun --gpus 2 -- 'bash scripts/multi_gpu_suite.sh 2'
n=${1:-2}
mkdir -p gpurun_out
rc=0
for mode in push nccl multicast; do
  args=""
  [ $mode = nccl ] && args="--gather nccl"
  [ $mode = multicast ] && args="--multicast"
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 1000)) scripts/multi_gpu_check.py $args \
    > gpurun_out/multi_n${n}_${mode}.log 2>&1
  r=$?
  grep '^{' gpurun_out/multi_n${n}_${mode}.log | tail -1 > gpurun_out/multi_n${n}_${mode}.json
  echo "n=$n mode=$mode rc=$r $(python -c "import json,sys; d=json.load(open('gpurun_out/multi_n${n}_${mode}.json')); print('ok' if d['ok'] else 'FAIL', d['gather_modes'], [k for k,v in d['results'].items() if not v['passed']])" 2>&1)"
  [ $r -ne 0 ] && rc=$r
done
exit $rc
