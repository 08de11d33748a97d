#!/bin/bash
# Fused exchange + reconstruction at n = world size, VGG-19 bucket, clean L2 (scripts/fused_probe.py):
# the product kernel; diagnostics variants (scripts/build_variant.sh): no push / no wait
# (EXP_FUSED_DBG=1), push without the arrival wait (=2), the staged path (EXP_NO_FUSE=1); the
# ncclAllGather mode; and n = 1. Build the variants first:
#   for d in 1 2 3; do scripts/build_variant.sh dbg$d -DEXP_FUSED_DBG=$d; done
#   scripts/build_variant.sh nofuse -DEXP_NO_FUSE=1
#   bash scripts/fused_breakdown.sh 2      (on a box with >= 2 GPUs)
cd "$(dirname "$0")/.."
n=${1:-2}
run() {
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 \
    --master-port $2 scripts/fused_probe.py ${@:3} 2>&1 | grep '^{'
}
run $n 29600
for v in dbg1 dbg2 nofuse; do TAG_LIB_PATH=build_exp/libtag_$v.so run $n $((29601 + RANDOM % 100)) --label $v; done
run $n 29710 --gather nccl
run 1 29711
