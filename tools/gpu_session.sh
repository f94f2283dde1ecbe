set -x
N=2
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 1200 python -m pytest tests/test_coll_multigpu.py -q -m gpu -k "2-nvls]" -s 2>&1 | grep -E "MISMATCH|mp_coll_check|passed|failed" | head
for W in gpt2-1.3b-dp llama3-8b-tp-sp llama3-70b-fsdp mixtral-8x7b-ep; do
timeout 1500 $TR --master-port 29611 bench.py --gpus $N --workload $W --steps 20 --out gpurun_out/r2f_n${N}_$W.json > gpurun_out/r2f_n${N}_$W.log 2>&1; echo "bench $W exit $?"
timeout 900 $TR --master-port 29612 tools/counter_profile.py --workload $W --out gpurun_out/r2c_n${N}_$W.json > gpurun_out/r2c_n${N}_$W.log 2>&1; echo "counters $W exit $?"
done
