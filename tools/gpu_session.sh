set -x
N=4
timeout 2400 python -m pytest tests/test_coll_multigpu.py -q -m gpu -k "4" -s 2>&1 | grep -E "MISMATCH|mp_coll_check|tolerance|passed|failed" | head -30
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
for W in mixtral-8x7b-ep llama3-8b-tp-sp gpt2-1.3b-dp llama3-70b-fsdp; do
timeout 1200 $TR --master-port 29591 bench.py --gpus $N --workload $W --steps 12 --sm-partition 0 --ablations 0 --out gpurun_out/r2_p0_n${N}_$W.json > gpurun_out/r2_p0_n${N}_$W.log 2>&1; echo "bench p0 $W exit $?"
done
timeout 1200 $TR --master-port 29592 bench.py --gpus $N --workload mixtral-8x7b-ep --steps 12 --a2a-tma 1 --ablations 0 --out gpurun_out/r2_tma_n${N}_mixtral-8x7b-ep.json > gpurun_out/r2_tma_n${N}_mixtral.log 2>&1; echo "bench tma exit $?"
