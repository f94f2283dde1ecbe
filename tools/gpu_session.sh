timeout 900 python -m pytest tests/test_coll_gpu.py tests/test_engine_gpu.py -m gpu -q --timeout 600 -p no:cacheprovider -k "misaligned or zero_count or exhaustive or tune_and_replay or cli" > gpurun_out/pytest_new.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_new.log
python - <<'PY'
import json, time
from paper_2602_20656_b200 import _lagom_py as L
w = L.gen("fsdp", layers=2, seed=7)
t0 = time.perf_counter(); c = json.loads(L.oracle(w, "", 10**8)); t1 = time.perf_counter()
g = json.loads(L.oracle_gpu(w, "", 10**8, 0)); t2 = time.perf_counter()
g = json.loads(L.oracle_gpu(w, "", 10**8, 0)); t3 = time.perf_counter()
print("points", c["evaluations"], "cpu_s", round(t1-t0,3), "gpu_s(first)", round(t2-t1,3), "gpu_s", round(t3-t2,3), "identical", c == g)
PY
