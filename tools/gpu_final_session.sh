# Final bench lines: every workload at N = 4 and N = 2 on one 4-GPU box,
# REPS repeats (each repeat is a fresh bench process with its own search).
set -x
TAG=${TAG:-r2k}
for REP in $(seq 1 ${REPS:-2}); do
for N in ${NS:-4 2}; do
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
for W in gpt2-1.3b-dp llama3-8b-tp-sp llama3-70b-fsdp mixtral-8x7b-ep; do
timeout 1500 $TR --master-port 2975$N bench.py --gpus $N --workload $W --steps 20 --out gpurun_out/${TAG}_rep${REP}_n${N}_$W.json > gpurun_out/${TAG}_rep${REP}_n${N}_$W.log 2>&1; echo "bench rep $REP n $N $W exit $?"
done
done
done
