# TMA one-hop kernels with the local share on the LSU warps: parity, rates,
# FSDP at N = 2.
set -x
timeout 1500 python -m pytest tests/test_coll_multigpu.py -m gpu -x -q > gpurun_out/tl_mp.log 2>&1; echo "mp parity rc $?"
tail -3 gpurun_out/tl_mp.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 400 $TR --master-port 29831 tools/coll_sweep.py --nvls 1 --one-hop 1 --sizes 64M,1G --colls AG,RS,A2A --configs 8:512:2M:0:1,16:512:2M:0:1,24:640:2M:0:1,32:640:2M:0:1 --batch 5 --reps 3 --nccl 0 --out gpurun_out/tl_scan_n2.jsonl > gpurun_out/tl_scan_n2.log 2>&1; echo "scan2 rc $?"
TR4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 400 $TR4 --master-port 29832 tools/coll_sweep.py --nvls 1 --sizes 64M,256M --colls A2A --configs 8:512:2M:0:1,16:512:2M:0:1 --batch 5 --reps 3 --nccl 0 --out gpurun_out/tl_scan_n4.jsonl > gpurun_out/tl_scan_n4.log 2>&1; echo "scan4 rc $?"
if grep -q "passed" gpurun_out/tl_mp.log && ! grep -q "failed" gpurun_out/tl_mp.log; then
for REP in 1 2; do
timeout 1500 $TR --master-port 29833 bench.py --gpus 2 --workload llama3-70b-fsdp --steps 20 --out gpurun_out/tl_rep${REP}_n2_llama3-70b-fsdp.json > gpurun_out/tl_rep${REP}_n2_fsdp.log 2>&1; echo "bench fsdp rep $REP exit $?"
done
fi
