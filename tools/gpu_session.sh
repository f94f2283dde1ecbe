set -x
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29511 tools/coll_sweep.py --sizes 64M,512M --out gpurun_out/sweep2.jsonl > gpurun_out/sweep2.log 2>&1; echo "sweep exit $?"
grep 512 gpurun_out/sweep2.log | cut -c1-200
