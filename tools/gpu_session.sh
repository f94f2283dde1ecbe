set -x
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15
timeout 600 python bench.py --steps 10 --warmup 3 --out gpurun_out/bench_n1.json > gpurun_out/bench_n1.log 2>&1; echo "bench rc $?"
tail -c 3000 gpurun_out/bench_n1.log
