set -x
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py --steps 10 --warmup 3 --out gpurun_out/att_n1.json > gpurun_out/att_n1.log 2>&1; echo "bench rc $?"; tail -c 300 gpurun_out/att_n1.log
