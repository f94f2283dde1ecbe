timeout 600 python bench.py --steps 6 --warmup 3 --out gpurun_out/bench1_default.json > gpurun_out/bench1_default.log 2>&1; echo "bench1 exit $?"
grep metric gpurun_out/bench1_default.log | cut -c1-600
N=2
for W in gpt2-1.3b-dp llama3-70b-fsdp llama3-8b-tp-sp mixtral-8x7b-ep; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29691 bench.py --gpus $N --steps 6 --warmup 3 --workload $W --out gpurun_out/bench2n_$W.json > gpurun_out/bench2n_$W.log 2>&1; echo "$W exit $?"
python - <<PY
import json
d=json.load(open("gpurun_out/bench2n_$W.json"))["line"]
t=d["config"]["tune"]
print("$W", "lagom", round(d["value"],2), "nccl", round(d["nccl_default_ms"],2), "x", round(d["speedup_vs_nccl_default"],3), "start", t["start"], t["picks"][:3], "slow", round(d["compute"]["slowdown"],3), round(d["compute"]["slowdown_nccl"],3))
PY
done
