N=4
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29711 tools/contention_profile.py --out gpurun_out/cprof_final_n4.json > gpurun_out/cprof_final_n4.log 2>&1; echo "cprof exit $?"
for N in 4 2; do
for W in gpt2-1.3b-dp llama3-8b-tp-sp llama3-70b-fsdp mixtral-8x7b-ep; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 2972$N bench.py --gpus $N --steps 8 --warmup 3 --workload $W --params gpurun_out/cprof_final_n4.json --out gpurun_out/final_n${N}_$W.json > gpurun_out/final_n${N}_$W.log 2>&1; echo "$N $W exit $?"
python - <<PY
import json
d=json.load(open("gpurun_out/final_n${N}_$W.json"))["line"]
t=d["config"]["tune"]
print("N=$N $W", "lagom", round(d["value"],2), "nccl", round(d["nccl_default_ms"],2), "x", round(d["speedup_vs_nccl_default"],3), "start", t["start"], t["picks"][:2], "slow", round(d["compute"]["slowdown"],3), round(d["compute"]["slowdown_nccl"],3), "roof", round(d["roofline"]["frac"],3))
PY
done; done
