#!/bin/bash
# Fused push + reconstruction A/B at n = 2 and 4 on one box (scripts/fused_probe.py, VGG bucket):
# the product library against every diagnostics build under build_exp/, alternating, 3 rounds.
cd "$(dirname "$0")/.."
for i in 1 2 3; do
  for v in product $(ls build_exp | sed -n 's/^libtag_\(.*\)\.so$/\1/p'); do
    lib=""; [ $v != product ] && lib=build_exp/libtag_$v.so
    for n in ${NS:-2 4}; do
      TAG_LIB_PATH=$lib timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
        --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) scripts/fused_probe.py \
        --label $v 2>/dev/null | grep "^{" | cut -c1-160
    done
  done
done
