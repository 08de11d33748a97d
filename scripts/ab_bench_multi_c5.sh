#!/bin/bash
# BERT-L E2 bucket (bench --config 5) at n = 2 and 4: the product library against every build
# under build_exp/, alternating, two rounds; prints ms_per_step per variant.
cd "$(dirname "$0")/.."
for i in 1 2; do
  for v in product $(ls build_exp | sed -n 's/^libtag_\(.*\)\.so$/\1/p'); do
    lib=""; [ $v != product ] && lib=build_exp/libtag_$v.so
    for n in ${NS:-2 4}; do
      echo "$v n=$n $(TAG_LIB_PATH=$lib timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
        --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n --steps 20 \
        --warmup 5 --config ${CFG:-5} 2>/dev/null | grep '^{' | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline'].get('recon_only_us'))")"
    done
  done
done
