# usage: bash tools/gpu_prof_fused.sh "CFGS" -- ncu full capture of the fused kernel per config
mkdir -p gpurun_out
for C in $1; do
  python tools/prof_fused.py $C 3 > gpurun_out/prof_plain_f$C.log 2>&1 || { echo "plain run failed $C"; tail gpurun_out/prof_plain_f$C.log; exit 1; }
done
for C in $1; do
  ncu --set full --clock-control none --import-source on -k "regex:k_fused" -s 1 -c 1 -o gpurun_out/prof_fused_cfg$C -f python tools/prof_fused.py $C 3 > gpurun_out/ncu_fused_cfg$C.log 2>&1
  echo "ncu $C rc=$?"
done
