T=gpurun_out/r02d; mkdir -p $T
timeout 300 python tools/time_paths.py 4 20 2>&1 | tee $T/tp4.log
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_parity.py -q -x --timeout 600 > $T/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 $T/pytest.log
