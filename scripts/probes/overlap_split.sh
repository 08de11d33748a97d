#!/bin/bash
# run overlap_split_probe.py at n = $1 for the product library (no overlap arm) and every capped
# diagnostics build under build_exp/
cd "$(dirname "$0")/../.."
n=${1:-4}
for v in product $(ls build_exp | sed -n 's/^libtag_\(.*\)\.so$/\1/p'); do
  lib=""; [ $v != product ] && lib=build_exp/libtag_$v.so
  TAG_LIB_PATH=$lib timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
    --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) scripts/probes/overlap_split_probe.py \
    --label $v 2>&1 | grep '^{'
done
