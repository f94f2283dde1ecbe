TR4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531"
timeout 1200 $TR4 tools/contention_profile.py --out gpurun_out/contention_profile_n4_v3.json > gpurun_out/contention_profile_n4_v3.log 2>&1; echo "profile exit $?"; tail -c 300 gpurun_out/contention_profile_n4_v3.log
