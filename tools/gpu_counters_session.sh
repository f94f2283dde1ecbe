# Counter profiles (CUPTI PM sampling) of every workload with the final
# kernels, at N = 4 and N = 2 on one 4-GPU box, for tools/counter_fit.py.
set -x
for N in ${NS:-4 2}; do
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
for W in gpt2-1.3b-dp llama3-8b-tp-sp llama3-70b-fsdp mixtral-8x7b-ep; do
timeout 1200 $TR --master-port 2979$N tools/counter_profile.py --workload $W --one-hop 2 --out gpurun_out/cnt_n${N}_$W.json > gpurun_out/cnt_n${N}_$W.log 2>&1; echo "counters n $N $W exit $?"
done
done
