# usage: bash tools/gpu_dev.sh [CFGS] -- all GPU tests (not slow) + quick path timings
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m "gpu and not slow" -q -x --timeout 300 > gpurun_out/pytest_dev.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/pytest_dev.log
for c in ${1:-2 3 1}; do timeout 300 python tools/time_paths.py $c 20 2>&1 | tail -6; done
