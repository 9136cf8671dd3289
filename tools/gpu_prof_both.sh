# usage: bash tools/gpu_prof_both.sh "CFGS" -- ncu full capture: separate eval kernel + fused kernel per config
mkdir -p gpurun_out
for C in $1; do
  python tools/prof.py $C 3 > gpurun_out/pp_$C.log 2>&1 || { echo "plain run failed $C"; tail gpurun_out/pp_$C.log; exit 1; }
  python tools/prof_fused.py $C 3 > gpurun_out/ppf_$C.log 2>&1 || { echo "plain fused run failed $C"; tail gpurun_out/ppf_$C.log; exit 1; }
done
for C in $1; do
  ncu --set full --clock-control none --import-source on -k "regex:k_eval|k1_" -s 2 -c 2 -o gpurun_out/prof_cfg$C -f python tools/prof.py $C 3 > gpurun_out/ncu_cfg$C.log 2>&1; echo "ncu sep $C rc=$?"
  ncu --set full --clock-control none --import-source on -k "regex:k_fused" -s 1 -c 1 -o gpurun_out/prof_fused_cfg$C -f python tools/prof_fused.py $C 3 > gpurun_out/ncu_fused_cfg$C.log 2>&1; echo "ncu fused $C rc=$?"
done
