# Round-2 N=1 evidence: the bench line, its ncu launch list, and one ncu
# --set full capture of the dominant collective kernel at the bench's picks.
set -x
timeout 1200 python bench.py --steps 20 --warmup 5 --out gpurun_out/r2f_n1_gpt2-1.3b-dp.json > gpurun_out/r2f_n1.log 2>&1; echo "bench rc $?"
tail -c 400 gpurun_out/r2f_n1.log
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --start nccl-default --budget 8"
timeout 900 $CMD > gpurun_out/plain_n1.log 2>&1 && \
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_n1.csv $CMD > gpurun_out/ncu_launch_n1.log 2>&1; echo "ncu launches rc $?"
K="python tools/coll_kernel_run.py --coll AR --ranks 1 --count 13107200 --nc 8 --nt 512 --chunk 2M --iters 5"
timeout 300 $K && timeout 900 ncu --set full --clock-control none --import-source on -k regex:local_copy -s 2 -c 2 -o gpurun_out/prof_copy_n1_nc8 $K > gpurun_out/ncu_full_n1.log 2>&1; echo "ncu full rc $?"
K2="python tools/coll_kernel_run.py --coll AR --ranks 1 --count 13107200 --nc 64 --nt 128 --chunk 2M --iters 5"
timeout 300 $K2 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:local_copy -s 2 -c 2 -o gpurun_out/prof_copy_n1_nc64 $K2 > gpurun_out/ncu_full_n1b.log 2>&1; echo "ncu full2 rc $?"
