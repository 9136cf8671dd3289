# usage: bash tools/gpu_quick.sh "CFGS"  -- gpu tests (not slow) + short benches
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m "gpu and not slow" -q -x --timeout 120 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
for c in $1; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg$c.log 2>&1; echo "bench cfg$c rc=$?"
  python tools/summ.py gpurun_out/bench_cfg$c.log
done
