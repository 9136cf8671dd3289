# usage: bash tools/gpu_r02.sh [TAG] -- round-2 check on a B200: smoke, all GPU tests, the default
# bench line (cfg4 fp64), every other config, the reference arm.  Logs under gpurun_out/<TAG>/.
T=gpurun_out/${1:-r02}; mkdir -p $T
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $T/gpu.txt 2>&1
python __graft_entry__.py smoke > $T/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 ${PYTEST_K:+-k "$PYTEST_K"} > $T/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 $T/pytest_gpu.log
timeout 600 python bench.py > $T/bench_default.log 2>&1; echo "bench rc=$?"; python tools/summ.py $T/bench_default.log
for c in ${CFGS:-2 3 1 5}; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > $T/bench_cfg$c.log 2>&1; echo "bench cfg$c rc=$?"; python tools/summ.py $T/bench_cfg$c.log; done
if [ -z "$NOREF" ]; then timeout 600 python bench.py --impl reference > $T/bench_reference.log 2>&1; echo "ref rc=$?"; tail -c 300 $T/bench_reference.log; fi
