# ncu of the final single-rank copy (with the L2 prefetch), at the bench's pick.
set -x
K="python tools/coll_kernel_run.py --coll AR --ranks 1 --count 13107200 --nc 64 --nt 128 --chunk 2M --iters 5"
timeout 300 $K && timeout 900 ncu --set full --clock-control none --import-source on -k regex:local_copy -s 2 -c 2 -o gpurun_out/prof_copy_n1_nc64_pf $K > gpurun_out/ncu_pf.log 2>&1; echo "ncu full rc $?"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 900 $CMD > gpurun_out/n1c_plain.log 2>&1 && \
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/n1c_launches.csv $CMD > gpurun_out/n1c_ncu_launch.log 2>&1; echo "ncu launches rc $?"
