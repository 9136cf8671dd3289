T=gpurun_out/r02q; mkdir -p $T
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 > $T/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 $T/pytest.log
