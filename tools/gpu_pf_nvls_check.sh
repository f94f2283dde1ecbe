# L2 prefetch in the switch / one-hop kernels that read locally: parity, then
# the co-resident one-hop and A2A rates at n = 2 and 4.
set -x
timeout 1500 python -m pytest tests/test_coll_multigpu.py -m gpu -x -q > gpurun_out/pfn_mp.log 2>&1; echo "mp parity rc $?"
tail -3 gpurun_out/pfn_mp.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 400 $TR --master-port 29811 tools/coll_sweep.py --nvls 1 --one-hop 1 --sizes 64M,1G --colls AG,RS --configs 64:128:2M:0:1,64:128:512K:0:1,32:256:2M:0:1,64:256:2M:0:1,16:128:2M:0:1 --batch 5 --reps 3 --nccl 0 --out gpurun_out/pfn_co_scan1_n2.jsonl > gpurun_out/pfn_co_scan1.log 2>&1; echo "scan rc $?"
for N in 2 4; do
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 400 $TR --master-port 2982$N tools/coll_sweep.py --nvls 1 --sizes 64M,256M --colls AG,A2A --configs 64:128:2M:0:1,32:256:2M:0:1,8:512:2M:0:1 --batch 5 --reps 3 --nccl 1 --out gpurun_out/pfn_a2a_n$N.jsonl > gpurun_out/pfn_a2a_n$N.log 2>&1; echo "a2a scan $N rc $?"
done
