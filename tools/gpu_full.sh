# usage: bash tools/gpu_full.sh -- round evidence: smoke, all GPU tests, bench (default + every config),
# reference arm, ncu launch list of the default bench, ncu --set full of cfg2's build/eval/fused kernels
# and of cfg3's / cfg4's build and eval kernels
mkdir -p gpurun_out
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"; tail -c 400 gpurun_out/bench_default.log
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.log 2>&1; echo "ref rc=$?"
for c in 1 3 4 5; do timeout 400 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_cfg$c.log 2>&1; echo "bench cfg$c rc=$?"; done
python tools/summ.py gpurun_out/bench_default.log; for c in 1 3 4 5; do python tools/summ.py gpurun_out/bench_cfg$c.log; done
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/launch_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
python tools/prof.py 2 3 > gpurun_out/pp_2.log 2>&1 && python tools/prof_fused.py 2 3 > gpurun_out/ppf_2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:k1_|k_eval" -s 2 -c 2 -o gpurun_out/prof_cfg2 -f python tools/prof.py 2 3 > gpurun_out/ncu_cfg2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:k_fused" -s 1 -c 1 -o gpurun_out/prof_fused_cfg2 -f python tools/prof_fused.py 2 3 > gpurun_out/ncu_fused_cfg2.log 2>&1; echo "ncu full rc=$?"
for c in 3 4; do python tools/prof.py $c 3 > gpurun_out/pp_$c.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:k1_|k_tile|k_eval" -s 2 -c 2 -o gpurun_out/prof_cfg$c -f python tools/prof.py $c 3 > gpurun_out/ncu_cfg$c.log 2>&1; echo "ncu cfg$c rc=$?"; done
# the paper's quality checks and the control-point / division sweep
mkdir -p gpurun_out/export/r01
timeout 600 python tools/precision_report.py gpurun_out/export/r01/precision_report.json > gpurun_out/precision.log 2>&1; echo "precision rc=$?"
timeout 900 python bench.py --ablation > gpurun_out/ablation.log 2>&1; echo "ablation rc=$?"
grep '^{' gpurun_out/ablation.log > gpurun_out/export/r01/ablation_sweep.jsonl
# summaries + bench lines into gpurun_out/export (copied back); keep only cfg2's full report
python tools/save_profiles.py r01 gpurun_out/export > gpurun_out/export.log 2>&1; echo "export rc=$?"
rm -f gpurun_out/prof_fused_cfg2.ncu-rep gpurun_out/prof_cfg3.ncu-rep gpurun_out/prof_cfg4.ncu-rep
du -sh gpurun_out
