set -x
nvidia-smi topo -m | head -8
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 2951$N bench.py --gpus $N --steps 5 --warmup 3 --out gpurun_out/bench$N.json > gpurun_out/bench$N.log 2>&1; echo "bench$N exit $?"
grep metric gpurun_out/bench$N.log | cut -c1-2500
done
timeout 600 python -m pytest tests/test_coll_multigpu.py -q -m gpu -x > gpurun_out/pytest_mgpu.log 2>&1; echo "pytest mgpu exit $?"; tail -3 gpurun_out/pytest_mgpu.log
