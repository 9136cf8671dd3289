# usage: bash tools/gpu_prof3.sh "CFGS" REGEX -- ncu full capture (2nd iteration's kernels matching REGEX) per config
mkdir -p gpurun_out
for C in $1; do
  python tools/prof.py $C 4 > gpurun_out/prof_plain_$C.log 2>&1 || { echo "plain run failed $C"; tail gpurun_out/prof_plain_$C.log; exit 1; }
done
for C in $1; do
  ncu --set full --clock-control none --import-source on -k "regex:$2" -s 2 -c 2 -o gpurun_out/prof_cfg$C -f python tools/prof.py $C 4 > gpurun_out/ncu_cfg$C.log 2>&1
  echo "ncu $C rc=$?"
done
