T=gpurun_out/r02t; mkdir -p $T
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 > $T/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $T/pytest.log
