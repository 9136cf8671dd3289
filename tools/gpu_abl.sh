mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ablation.py -q -x --timeout 600 > gpurun_out/pytest_abl.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_abl.log
timeout 900 python bench.py --ablation > gpurun_out/ablation.log 2>&1; echo "ablation rc=$?"; tail -c 600 gpurun_out/ablation.log
