TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531"
timeout 900 python -m pytest tests/test_coll_multigpu.py -x -q -s > gpurun_out/mgpu.log 2>&1; echo "mgpu exit $?"; grep "mp_coll_check:\|MISMATCH\|passed\|failed" gpurun_out/mgpu.log | head -20
LAGOM_BIG=1 LAGOM_NVLS=1 timeout 600 $TR tests/mp_coll_check.py > gpurun_out/mgpu_big.log 2>&1; echo "big exit $?"; grep "mp_coll_check:\|MISMATCH" gpurun_out/mgpu_big.log | head
for T in 0 1; do
LAGOM_A2A_TMA=$T timeout 400 $TR tools/coll_sweep.py --nvls 1 --nccl $T --sizes 64M,256M --colls A2A --configs 2:64:1M:0:1,4:64:1M:0:1,4:256:1M:0:1,8:256:1M:0:1,8:640:1M:0:1,16:640:1M:0:1 --out gpurun_out/a2a_direct_t$T.jsonl > gpurun_out/a2a_direct_t$T.log 2>&1; echo "sweep $T exit $?"
done
timeout 900 $TR bench.py --gpus 4 --workload mixtral-8x7b-ep --steps 6 --out gpurun_out/bench_n4_mixtral.json > gpurun_out/bench_n4_mixtral.log 2>&1; echo "bench exit $?"; tail -c 300 gpurun_out/bench_n4_mixtral.log
