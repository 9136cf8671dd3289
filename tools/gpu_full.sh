# usage: bash tools/gpu_full.sh -- round-end style evidence: all GPU tests, bench (default), reference arm,
# ncu launch list of the bench, ncu --set full of cfg2's build + eval kernels
mkdir -p gpurun_out
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > gpurun_out/clocks_before.csv
timeout 300 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench_default.log
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.log 2>&1; echo "ref rc=$?"; tail -c 800 gpurun_out/bench_reference.log
for c in 1 3 4 5; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_cfg$c.log 2>&1; echo "bench cfg$c rc=$?"; python tools/summ.py gpurun_out/bench_cfg$c.log; done
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/launch_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
python tools/prof.py 2 4 > gpurun_out/prof_plain_2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:k1_|k_eval" -s 2 -c 2 -o gpurun_out/prof_cfg2 -f python tools/prof.py 2 4 > gpurun_out/ncu_cfg2.log 2>&1; echo "ncu full rc=$?"
