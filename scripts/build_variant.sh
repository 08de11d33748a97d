#!/bin/bash
# Build an experimental libtag variant with extra nvcc defines for recon_tc.cu:
#   scripts/build_variant.sh <name> -DSTAGES_PAIR=9 ...   -> build_exp/libtag_<name>.so
# Load it with TAG_LIB_PATH=build_exp/libtag_<name>.so (sweeps only; never the product path).
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
csrc=$root/paper_2302_06126_b200/csrc
nccl=/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl
mkdir -p "$root/build_exp"
make -C "$csrc" -s
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC,-fvisibility=hidden \
  --expt-relaxed-constexpr -I$nccl/include -I$root/include -I$csrc "$@" -c "${SRC:-$csrc/recon_tc.cu}" -o "$root/build_exp/recon_tc_$name.o"
objs=""
for o in api recon_simt pack_sgd push_gather bias select ilp; do objs="$objs $csrc/$o.o"; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$root/build_exp/libtag_$name.so" $objs \
  "$root/build_exp/recon_tc_$name.o" -cudart static -L$nccl/lib -l:libnccl.so.2 -Xlinker -rpath,$nccl/lib
echo "built build_exp/libtag_$name.so"
