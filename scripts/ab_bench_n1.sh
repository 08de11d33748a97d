#!/bin/bash
# n = 1 bench A/B on one box: the product library against the builds under build_exp/, alternating
cd "$(dirname "$0")/.."
for i in 1 2 3; do
  for v in product $(ls build_exp | sed -n 's/^libtag_\(.*\)\.so$/\1/p'); do
    lib=""; [ $v != product ] && lib=build_exp/libtag_$v.so
    echo "$v $(TAG_LIB_PATH=$lib timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-virtual 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'])")"
  done
done
