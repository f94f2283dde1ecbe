timeout 600 python -m pytest tests -m gpu -q -x --timeout 200 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest $?"; tail -2 gpurun_out/pytest_gpu.log
N=4
for W in gpt2-1.3b-dp llama3-8b-tp-sp llama3-70b-fsdp mixtral-8x7b-ep; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29601 bench.py --gpus $N --steps 6 --warmup 3 --workload $W --out gpurun_out/bench4_$W.json > gpurun_out/bench4_$W.log 2>&1; echo "$W exit $?"
python - <<PY
import json
d=json.load(open("gpurun_out/bench4_$W.json"))["line"]
t=d["config"]["tune"]
print("$W", "lagom", round(d["value"],2), "nccl", round(d["nccl_default_ms"],2), "x", round(d["speedup_vs_nccl_default"],3), "seed", round(d["lagom_kernels_nccl_seed_ms"],2), "start", t["start"], {k:(round(sorted(v["Z_select"])[1]/1e3,2) if v["Z_select"] else None, v["calls"]) for k,v in t["others"].items()}, t["picks"], "slow", round(d["compute"]["slowdown"],3), round(d["compute"]["slowdown_nccl"],3), "roof", round(d["roofline"]["achieved"],1))
PY
done
