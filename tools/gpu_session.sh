for N in 2 4; do
LAGOM_TRACE=0 timeout 420 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 2953$N bench.py --gpus $N --steps 8 --warmup 3 --out gpurun_out/bench$N.json > gpurun_out/bench$N.log 2>&1; echo "bench$N exit $?"
grep metric gpurun_out/bench$N.log | cut -c1-3500
done
