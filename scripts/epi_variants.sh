#!/bin/bash
# fc6 reconstruction at virtual n = 8 (K = 256) and n = 1 (K = 32), bf16 and fp32 dW: the product
# kernel against every diagnostics variant under build_exp/ (scripts/build_variant.sh).
cd "$(dirname "$0")/.."
for v in product $(ls build_exp | sed -n 's/^libtag_\(.*\)\.so$/\1/p'); do
  lib=""; [ $v != product ] && lib=build_exp/libtag_$v.so
  for nv in 8 1; do
    for out in bf16 f32; do
      echo "$v $(TAG_LIB_PATH=$lib timeout 120 python scripts/recon_time.py --layer fc6 --n $nv --out $out)"
    done
  done
done
