T=gpurun_out/r02z; mkdir -p $T
nproc > $T/nproc.txt; free -g >> $T/nproc.txt
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 1800 -s -p no:cacheprovider > $T/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $T/pytest.log; grep -E "full|every query" $T/pytest.log | head
