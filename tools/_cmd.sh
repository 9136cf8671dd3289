T=gpurun_out/r02g; mkdir -p $T
timeout 2400 python -m pytest tests -m gpu -q --timeout 1500 > $T/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $T/pytest_gpu.log
bash tools/gpu_ncu.sh r02g
