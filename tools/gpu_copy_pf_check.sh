# single-rank copy prefetch (one-CTA form): tests, rates, bench
set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "single_rank or local or copy" > gpurun_out/cp_pytest.log 2>&1; echo "pytest rc $?"
tail -2 gpurun_out/cp_pytest.log
for CFG in "1 64" "2 128" "64 128" "8 512"; do
set -- $CFG
timeout 120 python tools/coll_kernel_run.py --coll AR --ranks 1 --count 13107200 --nc $1 --nt $2 --chunk 2M --iters 20 >> gpurun_out/cp_rates.log 2>&1
done
cat gpurun_out/cp_rates.log
timeout 1200 python bench.py --out gpurun_out/cp_n1_gpt2-1.3b-dp.json > gpurun_out/cp_bench.log 2>&1; echo "bench rc $?"
tail -c 300 gpurun_out/cp_bench.log
