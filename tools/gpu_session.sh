# Repeat of the N=2 bench lines with the final kernels (run-to-run variation).
TR2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532"
for W in gpt2-1.3b-dp llama3-8b-tp-sp llama3-70b-fsdp mixtral-8x7b-ep; do
timeout 900 $TR2 bench.py --gpus 2 --workload $W --steps 10 --out gpurun_out/rep2_n2_$W.json > gpurun_out/rep2_n2_$W.log 2>&1; echo "n2 $W exit $?"
done
