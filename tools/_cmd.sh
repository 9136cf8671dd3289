T=gpurun_out/r02v; mkdir -p $T
timeout 600 python tools/sanitize_cases.py > $T/plain.log 2>&1; echo "plain rc=$?"; cat $T/plain.log | tail -16
timeout 1500 compute-sanitizer --tool memcheck --leak-check no python tools/sanitize_cases.py > $T/memcheck.log 2>&1; echo "memcheck rc=$?"; tail -5 $T/memcheck.log
