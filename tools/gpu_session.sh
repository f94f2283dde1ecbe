# Final round-1 evidence with the final kernels: contention profile, then bench lines at N=4, N=2, N=1.
TR4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531"
TR2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532"
timeout 1200 $TR4 tools/contention_profile.py --out gpurun_out/contention_profile_n4_v2.json > gpurun_out/contention_profile_n4_v2.log 2>&1; echo "profile exit $?"
for W in gpt2-1.3b-dp llama3-8b-tp-sp llama3-70b-fsdp mixtral-8x7b-ep; do
timeout 900 $TR4 bench.py --gpus 4 --workload $W --steps 10 --out gpurun_out/v2_n4_$W.json > gpurun_out/v2_n4_$W.log 2>&1; echo "n4 $W exit $?"
done
for W in gpt2-1.3b-dp llama3-8b-tp-sp llama3-70b-fsdp mixtral-8x7b-ep; do
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $TR2 bench.py --gpus 2 --workload $W --steps 10 --out gpurun_out/v2_n2_$W.json > gpurun_out/v2_n2_$W.log 2>&1; echo "n2 $W exit $?"
done
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --out gpurun_out/v2_n1.json > gpurun_out/v2_n1.log 2>&1; echo "n1 exit $?"
