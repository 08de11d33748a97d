#!/bin/bash
# BERT-L E2 bucket (bench --config 5, n = 1): the product kernel against every diagnostics
# variant under build_exp/; prints step us and the HBM roofline fraction (two runs each).
cd "$(dirname "$0")/.."
for v in product $(ls build_exp | sed -n 's/^libtag_\(.*\)\.so$/\1/p'); do
  lib=""; [ $v != product ] && lib=build_exp/libtag_$v.so
  for i in 1 2; do
    echo "$v $(TAG_LIB_PATH=$lib timeout 300 python bench.py --config 5 --steps 30 --warmup 5 --no-cpu-baseline --no-virtual 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['ms_per_step'], d['roofline']['frac'])")"
  done
done
