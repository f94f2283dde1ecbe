set -x
N=2
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
for W in llama3-70b-fsdp llama3-8b-tp-sp gpt2-1.3b-dp; do
timeout 1500 $TR --master-port 29621 bench.py --gpus $N --workload $W --steps 16 --out gpurun_out/r2g_n${N}_$W.json > gpurun_out/r2g_n${N}_$W.log 2>&1; echo "bench $W exit $?"
done
