set -x
timeout 600 python bench.py --steps 5 --warmup 3 --out gpurun_out/bench1.json > gpurun_out/bench1.log 2>&1; echo "bench1 exit $?"
tail -c 3000 gpurun_out/bench1.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 5 --warmup 3 --out gpurun_out/bench2.json > gpurun_out/bench2.log 2>&1; echo "bench2 exit $?"
tail -c 3000 gpurun_out/bench2.log
