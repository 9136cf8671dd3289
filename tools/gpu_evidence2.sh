# usage: bash tools/gpu_evidence2.sh TAG -- part B of the round evidence on a B200 (after tools/gpu_full.sh):
# the whole GPU test suite, the precision report, the §8(d) counter capture of every config's timed
# kernels (tools/gpu_steps.sh) and the --set full captures of the top kernels (tools/gpu_ncu.sh).
T=gpurun_out/${1:-r02g}; mkdir -p $T
timeout 2400 python -m pytest tests -m gpu -q --timeout 1500 > $T/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $T/pytest_gpu.log
timeout 600 python tools/precision_report.py $T/precision_report.json > $T/precision.log 2>&1; echo "precision rc=$?"
bash tools/gpu_steps.sh ${1:-r02g}s
bash tools/gpu_ncu.sh ${1:-r02g}n
