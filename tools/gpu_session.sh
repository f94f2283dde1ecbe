# TMA/LSU split copy steps: parity with shares forced, then 2-GPU sweep over shares.
LAGOM_TMA_SHARE_PUSH=900 LAGOM_TMA_SHARE_LOCAL=360 timeout 900 python -m pytest tests/test_coll_gpu.py -x -q > gpurun_out/pytest_split.log 2>&1; echo "pytest split exit $?"; tail -2 gpurun_out/pytest_split.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531"
for S in 0 400 900 2000; do
LAGOM_TMA_SHARE_PUSH=$S LAGOM_TMA_SHARE_LOCAL=$((S*2/5)) timeout 400 $TR tools/coll_sweep.py --nccl 0 --sizes 64M,256M --colls A2A,AG \
    --configs 8:128:1M:0,8:512:1M:0,8:640:2M:0,32:640:4M:0 --out gpurun_out/split_$S.jsonl > gpurun_out/split_$S.log 2>&1; echo "sweep $S exit $?"
done
