N=4
timeout 420 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus $N --steps 8 --warmup 3 --out gpurun_out/bench4_full.json > gpurun_out/bench4_full.log 2>&1; echo "bench exit $?"
