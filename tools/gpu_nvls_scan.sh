# NVLS kernel rates vs size on one box: back-to-back launches (--batch), so
# the rows show the kernels' own rate without launch latency or rank skew.
# Lagom TREE (in-switch) at several NC / NT, NCCL default, NCCL_ALGO=NVLS.
set -x
N=${N:-4}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
SZ=${SZ:-1M,4M,16M,25M,64M,256M}
CF=${CF:-8:512:2M:0:1,16:512:2M:0:1,32:512:2M:0:1,64:128:2M:0:1,64:256:2M:0:1,8:640:2M:0:1,4:512:2M:0:1}
timeout 900 $TR --master-port 29711 tools/coll_sweep.py --nvls 1 --sizes $SZ --colls ${COLLS:-AR,AG,RS} --configs $CF --batch 20 --reps 5 --nccl 1 --out gpurun_out/nvls_scan_n$N.jsonl > gpurun_out/nvls_scan_n$N.log 2>&1; echo "scan rc $?"
NCCL_ALGO=NVLS timeout 600 $TR --master-port 29712 tools/coll_sweep.py --nvls 1 --lagom 0 --sizes $SZ --colls ${COLLS:-AR,AG,RS} --batch 20 --reps 5 --out gpurun_out/nvls_scan_ncclnvls_n$N.jsonl > gpurun_out/nvls_scan_ncclnvls_n$N.log 2>&1; echo "nccl nvls rc $?"
tail -3 gpurun_out/nvls_scan_n$N.log gpurun_out/nvls_scan_ncclnvls_n$N.log
