# Switch-kernel barrier rework: parity at n = 4 first, then phases and the
# bench on the comm-heavy workloads.
set -x
N=${N:-4}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests/test_coll_multigpu.py -m gpu -x -q > gpurun_out/bar_mp_n$N.log 2>&1; echo "mp parity rc $?"
tail -3 gpurun_out/bar_mp_n$N.log
LAGOM_PHASE_STAMPS=1 timeout 600 $TR --master-port 29731 tools/nvls_phases.py --sizes 1M,4M,25M,64M,256M --colls AR,AG,RS --configs 8:512,16:512,64:128,4:512 --out gpurun_out/phases3_n$N.jsonl > gpurun_out/phases3_n$N.log 2>&1; echo "phases rc $?"
for W in ${WL:-llama3-8b-tp-sp gpt2-1.3b-dp}; do
timeout 1500 $TR --master-port 29741 bench.py --gpus $N --workload $W --steps 20 --out gpurun_out/bar_n${N}_$W.json > gpurun_out/bar_n${N}_$W.log 2>&1; echo "bench $W exit $?"
done
