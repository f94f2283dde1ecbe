# What the driver runs at round end on one B200: smoke(), the GPU tests, the
# default bench line (and the reference arm).
set -x
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/fin_smoke.log 2>&1; echo "smoke rc $?"
tail -2 gpurun_out/fin_smoke.log
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/fin_pytest.log 2>&1; echo "pytest rc $?"
tail -2 gpurun_out/fin_pytest.log
timeout 1200 python bench.py --out gpurun_out/fin_n1_gpt2-1.3b-dp.json > gpurun_out/fin_bench.log 2>&1; echo "bench rc $?"
tail -c 600 gpurun_out/fin_bench.log
timeout 1200 python bench.py --impl reference > gpurun_out/fin_ref.log 2>&1; echo "ref rc $?"
tail -c 400 gpurun_out/fin_ref.log
