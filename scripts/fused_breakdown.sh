#!/bin/bash
# Fused push + reconstruction at n = world size, VGG-19 bucket, clean L2: normal, no push/wait,
# push without wait, the staged path (push-gather kernel + reconstruction), and n = 1.
#   bash scripts/fused_breakdown.sh 2      (on a box with >= 2 GPUs)
cd "$(dirname "$0")/.."
n=${1:-2}
run() {
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 \
    --master-port $2 scripts/fused_probe.py 2>&1 | grep '^{'
}
for d in 0 1 2; do TAG_FUSED_DEBUG=$d run $n $((29600 + d)); done
TAG_NO_FUSE=1 run $n 29610
run 1 29611
# reconstruction alone, operands in the symmetric window (push) vs cudaMalloc (nccl)
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
  --master-port 29620 scripts/recon_window_probe.py 2>&1 | grep '^{'
TAG_GATHER=nccl timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
  --master-addr 127.0.0.1 --master-port 29621 scripts/recon_window_probe.py 2>&1 | grep '^{'
TAG_GATHER=nccl run $n 29622
