cd /root/repo
for i in 1 2 3; do for v in old product; do
lib=""; [ $v = old ] && lib=build_exp/libtag_old.so
for n in 2 4; do TAG_LIB_PATH=$lib timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) scripts/fused_probe.py --label $v 2>/dev/null | grep "^{" | cut -c1-140; done; done; done
