# usage: bash tools/gpu_fused.sh [CFGS] -- fused + build GPU tests, quick path timings
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_parity.py -q -x --timeout 300 -k "fused or build_all or cfg2 or cfg3 or cfg1" > gpurun_out/pytest_fused.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/pytest_fused.log
for c in ${1:-2 3 1}; do timeout 300 python tools/time_paths.py $c 20 2>&1 | tail -6; done
FLUSH=w timeout 300 python tools/time_paths.py 2 20 2>&1 | tail -6
