set -x
timeout 1500 python -m pytest tests/test_coll_multigpu.py -q -m gpu -k "one_hop and 2" -s 2>&1 | grep -E "MISMATCH|mp_coll_check|tolerance|passed|failed" | head -20
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for W in llama3-8b-tp-sp llama3-70b-fsdp; do for H in 0 2; do
timeout 1200 $TR --master-port 29571 bench.py --gpus 2 --workload $W --steps 12 --one-hop $H --ablations 0 --out gpurun_out/r2_oh${H}_n2_$W.json > gpurun_out/r2_oh${H}_n2_$W.log 2>&1; echo "bench $W $H exit $?"
done; done
