set -x
timeout 1500 python -m pytest tests/test_coll_multigpu.py -q -m gpu -k "2" -s 2>&1 | grep -E "MISMATCH|mp_coll_check|passed|failed|Error|error" | head -40
TR2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for W in gpt2-1.3b-dp llama3-70b-fsdp; do
timeout 900 $TR2 --master-port 29541 bench.py --gpus 2 --workload $W --steps 10 --out gpurun_out/r2b_n2_$W.json > gpurun_out/r2b_n2_$W.log 2>&1; echo "n2 $W exit $?"
done
