#!/bin/bash
# Where the time of the CTA-pair reconstruction goes (fc6, virtual n = 8, K = 256): the shipped
# kernel against diagnostic builds whose epilogue does progressively less.
#   build here:  for v in 1 2 3 4; do scripts/build_variant.sh epi$v -DEXP_EPI_MODE=$v; done
#                scripts/build_variant.sh w16 -DEXP_EPI_WARPS=16
#   run on a GPU box:  bash scripts/epi_decompose.sh
#   EXP_EPI_MODE 2 = MMA + operand feed only, 4 = + TMEM reads, 1 = + smem transpose (no global
#   stores), 0 = shipped, 3 = TMEM -> direct 16-B stores (no smem); w16 = 16 epilogue warps.
#   TAG_RECON_NO3D=1 loads each operand as 2-D 64-column boxes instead of one 3-D box.
cd "$(dirname "$0")/.."
for lib in "" build_exp/libtag_epi2.so build_exp/libtag_epi4.so build_exp/libtag_epi1.so \
           build_exp/libtag_epi3.so build_exp/libtag_w16.so; do
  for out in bf16 f32; do
    TAG_LIB_PATH=$lib timeout 120 python scripts/recon_time.py --layer fc6 --n 8 --out $out
  done
done
for out in bf16 f32; do
  TAG_RECON_NO3D=1 timeout 120 python scripts/recon_time.py --layer fc6 --n 8 --out $out
done
