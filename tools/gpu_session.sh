set -x
N=2
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
for W in gpt2-1.3b-dp llama3-8b-tp-sp llama3-70b-fsdp mixtral-8x7b-ep; do
timeout 900 $TR --master-port 29561 tools/counter_profile.py --workload $W --out gpurun_out/r2_counters_n${N}_$W.json > gpurun_out/r2_counters_n${N}_$W.log 2>&1; echo "counters $W exit $?"
timeout 1200 $TR --master-port 29562 bench.py --gpus $N --workload $W --steps 20 --out gpurun_out/r2_final_n${N}_$W.json > gpurun_out/r2_final_n${N}_$W.log 2>&1; echo "bench $W exit $?"
done
