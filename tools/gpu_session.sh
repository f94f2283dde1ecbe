N=4
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29671 tools/contention_profile.py --out gpurun_out/cprof_nvls_n4.json > gpurun_out/cprof_nvls_n4.log 2>&1; echo "cprof exit $?"
tail -c 1500 gpurun_out/cprof_nvls_n4.log
for W in llama3-70b-fsdp llama3-8b-tp-sp gpt2-1.3b-dp mixtral-8x7b-ep; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29681 bench.py --gpus $N --steps 6 --warmup 3 --workload $W --params gpurun_out/cprof_nvls_n4.json --out gpurun_out/bench4n_$W.json > gpurun_out/bench4n_$W.log 2>&1; echo "$W exit $?"
python - <<PY
import json
d=json.load(open("gpurun_out/bench4n_$W.json"))["line"]
t=d["config"]["tune"]
print("$W", "lagom", round(d["value"],2), "nccl", round(d["nccl_default_ms"],2), "x", round(d["speedup_vs_nccl_default"],3), "seed", round(d["lagom_kernels_nccl_seed_ms"],2), "start", t["start"], {k:(round(sorted(v["Z_select"])[1]/1e3,2) if v["Z_select"] else None, v["calls"]) for k,v in t["others"].items()}, t["picks"], "slow", round(d["compute"]["slowdown"],3), round(d["compute"]["slowdown_nccl"],3), "roof", round(d["roofline"]["achieved"],1))
PY
done
