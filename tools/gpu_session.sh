N=4
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29571 tools/contention_profile.py --out gpurun_out/fitted_params_n4.json > gpurun_out/cprof4.log 2>&1; echo "cprof exit $?"
tail -c 2500 gpurun_out/cprof4.log
