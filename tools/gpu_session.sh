timeout 1200 python -m pytest tests/test_coll_multigpu.py -x -q -s > gpurun_out/mgpu4.log 2>&1; echo "mgpu exit $?"; grep "mp_coll_check:\|MISMATCH\|passed\|failed" gpurun_out/mgpu4.log | head -12
