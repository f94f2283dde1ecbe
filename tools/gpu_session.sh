TR4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531"
S='T:8:512:2M|T:8:512:2M T:8:512:2M|T:64:640:4M T:4:128:64K|T:64:640:4M T:4:512:1M|T:64:640:4M T:3:128:64K|T:64:640:4M T:2:256:64K|T:64:640:4M'
timeout 900 $TR4 tools/fixed_configs.py --sets $S --steps 8 --out gpurun_out/fixed_n4_gpt2.jsonl > gpurun_out/fixed_n4_gpt2.log 2>&1; echo "gpt2 exit $?"
timeout 900 $TR4 tools/fixed_configs.py --workload llama3-8b-tp-sp --sets $S --steps 6 --out gpurun_out/fixed_n4_tp.jsonl > gpurun_out/fixed_n4_tp.log 2>&1; echo "tp exit $?"
