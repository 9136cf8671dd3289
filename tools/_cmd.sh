T=gpurun_out/r02ag; mkdir -p $T
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "bucketed or cfg5" > $T/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $T/pytest.log
for r in 1 2; do timeout 300 python tools/time_paths.py 5 5 2>&1 | grep -E " eval|step" | sed "s/^/r$r /"; done
