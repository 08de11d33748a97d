cd /root/repo
for n in 2 4; do for c in 1 3; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n --steps 30 --warmup 5 --config $c > gpurun_out/bench_n${n}_c${c}.log 2>&1
grep '^{' gpurun_out/bench_n${n}_c${c}.log | tail -1 > gpurun_out/bench_n${n}_c${c}.json; echo "n=$n c=$c $(tail -c 300 gpurun_out/bench_n${n}_c${c}.log | head -c 200)"
done; done
