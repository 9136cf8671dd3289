T=gpurun_out/r02r; mkdir -p $T
timeout 600 python bench.py --config 3 --steps 20 --warmup 5 --no-cpu-baseline > $T/bench_cfg3.log 2>&1; echo "rc=$?"; python tools/summ.py $T/bench_cfg3.log
timeout 600 python bench.py --config 3 --steps 20 --warmup 5 --x-shared > $T/bench_cfg3_xshared.log 2>&1; echo "rc=$?"; python tools/summ.py $T/bench_cfg3_xshared.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $T/bench_cfg4.log 2>&1; echo "rc=$?"; python tools/summ.py $T/bench_cfg4.log
