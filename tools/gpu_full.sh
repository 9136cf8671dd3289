# usage: bash tools/gpu_full.sh TAG -- round evidence on a B200 (gpurun), part A: smoke, every bench
# line (default cfg4 with cpu_baseline + e2e; cfg1/2/3/5; cfg3 shared knots), the reference arm, the
# ncu launch list of the default bench (one ncu per call: part B is tools/gpu_ncu.sh).
T=gpurun_out/${1:-r02}; mkdir -p $T
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $T/gpu.txt 2>&1
python __graft_entry__.py smoke > $T/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $T/bench_cfg4.log 2>&1; echo "bench default rc=$?"; python tools/summ.py $T/bench_cfg4.log
for c in 1 2 3 5; do timeout 600 python bench.py --config $c --steps 30 --warmup 5 > $T/bench_cfg$c.log 2>&1; echo "bench cfg$c rc=$?"; python tools/summ.py $T/bench_cfg$c.log; done
timeout 600 python bench.py --config 3 --steps 30 --warmup 5 --x-shared --no-cpu-baseline > $T/bench_cfg3_xshared.log 2>&1; echo "bench cfg3 xshared rc=$?"
timeout 900 python bench.py --impl reference > $T/bench_reference.log 2>&1; echo "ref rc=$?"; tail -c 300 $T/bench_reference.log
timeout 900 python bench.py --ablation > $T/ablation.log 2>&1; echo "ablation rc=$?"
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $T/launch_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $T/launches_cfg4.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $T/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
