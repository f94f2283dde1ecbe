# L2 prefetch in the single-rank copy: correctness, rate with / without, bench.
set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "single_rank or local or copy" > gpurun_out/pf_pytest.log 2>&1; echo "pytest rc $?"
tail -2 gpurun_out/pf_pytest.log
for PF in 0 1; do
for CFG in "64 128" "32 128" "64 256" "8 512"; do
set -- $CFG
for CNT in 13107200 134217728; do
LAGOM_COPY_PREFETCH=$PF timeout 120 python tools/coll_kernel_run.py --coll AR --ranks 1 --count $CNT --nc $1 --nt $2 --chunk 2M --iters 20 >> gpurun_out/pf_rates_$PF.log 2>&1
done; done; done
cat gpurun_out/pf_rates_0.log gpurun_out/pf_rates_1.log
timeout 1200 python bench.py --out gpurun_out/pf_n1_gpt2-1.3b-dp.json > gpurun_out/pf_bench.log 2>&1; echo "bench rc $?"
tail -c 300 gpurun_out/pf_bench.log
