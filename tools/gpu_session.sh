timeout 600 python tools/sanitize_colls.py > gpurun_out/san_plain.log 2>&1; echo "plain exit $?"; tail -1 gpurun_out/san_plain.log
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_colls.py > gpurun_out/memcheck.log 2>&1; echo "memcheck exit $?"
grep -E "ERROR SUMMARY|sanitize_colls|Invalid|error" gpurun_out/memcheck.log | head -10
