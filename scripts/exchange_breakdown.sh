#!/bin/bash
# Fused-exchange phase breakdown at n = $1 (VGG-19 bucket): the product kernel, the diagnostics
# variants under build_exp/ (see scripts/fused_breakdown.sh), and the %globaltimer phase stamps of
# the dbg3 variant (push stores issued, CTA barrier, system-scope fence, local add, last CTA's
# publish, first arrival wait satisfied, end).
cd "$(dirname "$0")/.."
n=${1:-2}
bash scripts/r0_sweep.sh $n
TAG_LIB_PATH=build_exp/libtag_dbg3.so ITERS=6 timeout 300 python -m torch.distributed.run --nnodes=1 \
  --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) \
  scripts/fused_probe.py --label dbg3 2>&1 | grep "fused dbg" | tail -$((2 * n))
