#!/bin/bash
# Fused-exchange schedule sweep at n = $1: the product kernel vs every diagnostics variant under
# build_exp/ (scripts/build_variant.sh: EXP_R0 = rounds the push units skip, EXP_PUSH_CTAS,
# EXP_PUSH_NT, ...), VGG-19 bucket, scripts/fused_probe.py.
cd "$(dirname "$0")/.."
n=${1:-2}
shift
for v in product $(ls build_exp | sed -n 's/^libtag_\(.*\)\.so$/\1/p' | grep -v '^dbg'); do
  lib=""; [ $v != product ] && lib=build_exp/libtag_$v.so
  TAG_LIB_PATH=$lib timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
    --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) scripts/fused_probe.py --label $v "$@" 2>&1 | grep '^{'
done
