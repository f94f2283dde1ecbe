# One-hop TMA AllGather / pull ReduceScatter: parity at n = 2 and 4, rates,
# then FSDP and TP-SP at N = 2 with one_hop = 2 vs 0.
set -x
timeout 1500 python -m pytest tests/test_coll_multigpu.py -m gpu -x -q -k "one_hop or bench_sizes" > gpurun_out/oh_mp.log 2>&1; echo "mp parity rc $?"
tail -3 gpurun_out/oh_mp.log
for N in 2 4; do
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 600 $TR --master-port 2976$N tools/coll_sweep.py --nvls 1 --sizes 25M,64M,256M,1G --colls AG,RS --configs 8:512:2M:0:1,16:512:2M:0:1,24:640:2M:0:1,32:640:2M:0:1 --batch 5 --reps 3 --nccl 1 --out gpurun_out/oh_scan0_n$N.jsonl > gpurun_out/oh_scan0_n$N.log 2>&1; echo "scan0 rc $?"
timeout 600 $TR --master-port 2977$N tools/coll_sweep.py --nvls 1 --one-hop 1 --sizes 25M,64M,256M,1G --colls AG,RS --configs 8:512:2M:0:1,16:512:2M:0:1,24:640:2M:0:1,32:640:2M:0:1 --batch 5 --reps 3 --nccl 0 --out gpurun_out/oh_scan1_n$N.jsonl > gpurun_out/oh_scan1_n$N.log 2>&1; echo "scan1 rc $?"
done
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for W in llama3-70b-fsdp llama3-8b-tp-sp; do
for OH in 2 0; do
timeout 1500 $TR --master-port 29781 bench.py --gpus 2 --workload $W --steps 20 --one-hop $OH --out gpurun_out/oh${OH}_n2_$W.json > gpurun_out/oh${OH}_n2_$W.log 2>&1; echo "bench $W one_hop $OH exit $?"
done
done
