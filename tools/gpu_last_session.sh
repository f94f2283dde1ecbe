# N = 4 bench lines with the final bench (two repeats), then the counter
# profiles of every workload at N = 4 and N = 2 with the final kernels.
set -x
NS=4 TAG=r2p REPS=2 bash tools/gpu_final_session.sh
NS="4 2" bash tools/gpu_counters_session.sh
