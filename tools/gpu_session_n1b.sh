# N=1: the driver's GPU test suite, the bench's ncu launch list with its own
# default search, and ncu --set full of the tuned copy (NC 64, NT 128).
set -x
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/n1b_pytest.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/n1b_pytest.log
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 900 $CMD > gpurun_out/n1b_plain.log 2>&1 && \
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/n1b_launches.csv $CMD > gpurun_out/n1b_ncu_launch.log 2>&1; echo "ncu launches rc $?"
K="python tools/coll_kernel_run.py --coll AR --ranks 1 --count 13107200 --nc 64 --nt 128 --chunk 2M --iters 5"
timeout 300 $K && timeout 900 ncu --set full --clock-control none --import-source on -k regex:local_copy -s 2 -c 2 -o gpurun_out/prof_copy_n1_nc64 $K > gpurun_out/n1b_ncu_full.log 2>&1; echo "ncu full rc $?"
