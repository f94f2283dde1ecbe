# Repeat of the N=4 bench lines with the final kernels (run-to-run variation).
TR4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531"
for W in gpt2-1.3b-dp llama3-8b-tp-sp llama3-70b-fsdp mixtral-8x7b-ep; do
timeout 900 $TR4 bench.py --gpus 4 --workload $W --steps 10 --out gpurun_out/rep2_n4_$W.json > gpurun_out/rep2_n4_$W.log 2>&1; echo "n4 $W exit $?"
done
