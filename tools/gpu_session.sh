S='T:1:256:1M|T:64:640:4M T:2:256:1M|T:64:640:4M T:3:256:1M|T:64:640:4M T:4:256:1M|T:64:640:4M T:8:512:2M|T:8:512:2M T:2:256:1M|T:16:640:4M'
timeout 600 python tools/fixed_configs.py --sets $S --steps 5 --out gpurun_out/fixed_n1.jsonl > gpurun_out/fixed_n1.log 2>&1; echo "res1 exit $?"
timeout 600 python tools/fixed_configs.py --sets $S --steps 5 --sm-reserve 0 --out gpurun_out/fixed_n1.jsonl > gpurun_out/fixed_n1_nores.log 2>&1; echo "res0 exit $?"
