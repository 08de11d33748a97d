#!/bin/bash
# Build a diagnostics variant of libtag with extra nvcc defines (the EXP_* knobs of recon_tc.cu,
# api.cu, push_gather.cu — e.g. -DEXP_FUSED_DBG=3, -DEXP_NO_FUSE=1, -DEXP_RECON_BN=256, -DEXP_R0=4):
#   scripts/build_variant.sh <name> -DEXP_...=...   -> build_exp/libtag_<name>.so
# Load it with TAG_LIB_PATH=build_exp/libtag_<name>.so (sweeps only; never the product path).
# The product build (make -C paper_2302_06126_b200/csrc) sets none of these.
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
csrc=$root/paper_2302_06126_b200/csrc
nccl=${NCCL_HOME:-/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl}
out=$root/build_exp/$name
mkdir -p "$out"
make -C "$csrc" -s NCCL_HOME=$nccl
objs=""
for f in api recon_tc recon_simt pack_sgd push_gather bias; do
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC,-fvisibility=hidden \
    --expt-relaxed-constexpr -I$nccl/include -I$root/include -I$csrc "$@" -c "$csrc/$f.cu" -o "$out/$f.o" &
  objs="$objs $out/$f.o"
done
wait
objs="$objs $csrc/select.o $csrc/ilp.o"
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$root/build_exp/libtag_$name.so" $objs \
  -cudart static -L$nccl/lib -l:libnccl.so.2 -Xlinker -rpath,$nccl/lib
echo "built build_exp/libtag_$name.so"
