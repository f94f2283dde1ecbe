TR4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531"
timeout 1500 $TR4 tools/contention_profile.py --out gpurun_out/contention_profile_n4.json > gpurun_out/contention_profile_n4.log 2>&1; echo "profile exit $?"; tail -c 1500 gpurun_out/contention_profile_n4.log
