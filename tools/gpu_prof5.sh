mkdir -p gpurun_out
python tools/prof.py 5 2 > gpurun_out/pp_5.log 2>&1 || { tail gpurun_out/pp_5.log; exit 1; }
ncu --set full --clock-control none --import-source on -k "regex:records|k_tile|k4_top" -s 4 -c 5 -o gpurun_out/prof_cfg5 -f python tools/prof.py 5 2 > gpurun_out/ncu_cfg5.log 2>&1; echo "ncu rc=$?"
