set -x
N=4
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
for W in gpt2-1.3b-dp llama3-8b-tp-sp llama3-70b-fsdp mixtral-8x7b-ep; do
timeout 1500 $TR --master-port 29631 bench.py --gpus $N --workload $W --steps 20 --out gpurun_out/r2h_n${N}_$W.json > gpurun_out/r2h_n${N}_$W.log 2>&1; echo "bench $W exit $?"
done
