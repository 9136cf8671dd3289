# usage: bash tools/gpu_prof.sh CFG  -- ncu full capture of every kernel of one build+eval (2nd iteration)
mkdir -p gpurun_out
C=$1
python tools/prof.py $C 2 > gpurun_out/prof_plain_$C.log 2>&1 && \
ncu --set full --clock-control none --import-source on -s 2 -c 4 -o gpurun_out/prof_cfg$C -f python tools/prof.py $C 2 > gpurun_out/ncu_cfg$C.log 2>&1
echo "ncu rc=$?"
tail -3 gpurun_out/ncu_cfg$C.log
