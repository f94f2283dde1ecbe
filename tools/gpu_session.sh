TR2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532"
timeout 900 python -m pytest tests/test_coll_multigpu.py -x -q -s -k "2" > gpurun_out/mgpu2.log 2>&1; echo "mgpu exit $?"; grep "mp_coll_check:\|MISMATCH\|passed\|failed" gpurun_out/mgpu2.log | head
LAGOM_BIG=1 LAGOM_NVLS=1 timeout 600 $TR2 tests/mp_coll_check.py > gpurun_out/mgpu_big2.log 2>&1; echo "big exit $?"; grep "mp_coll_check:\|MISMATCH" gpurun_out/mgpu_big2.log | head
for W in llama3-70b-fsdp llama3-8b-tp-sp; do
timeout 900 $TR2 bench.py --gpus 2 --workload $W --steps 8 --out gpurun_out/fin2_n2_$W.json > gpurun_out/fin2_n2_$W.log 2>&1; echo "bench $W exit $?"
done
