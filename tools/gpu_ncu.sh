# usage: bash tools/gpu_ncu.sh TAG -- part B of the round evidence: ONE ncu --set full capture over the
# timed kernels of cfg2, cfg4 and cfg5 (tools/prof.py, one process each; --target-processes all).
T=gpurun_out/${1:-r02}; mkdir -p $T
cat > $T/top.sh <<'EOS'
set -e
python tools/prof.py 2 1
python tools/prof.py 4 1
python tools/prof.py 5 1
EOS
bash $T/top.sh > $T/top_plain.log 2>&1 && \
ncu --target-processes all --set full --clock-control none --import-source on \
    -k regex:"k1_thomas_half|k_eval_curvewarp|k_build_eval_warp|k_tile|k_eval_sorted|k_bucket_eval|k_bucket_scatter|k_bucket_gather" \
    -c 18 -o $T/top -f bash $T/top.sh > $T/ncu_top.log 2>&1; echo "ncu full rc=$?"; tail -2 $T/ncu_top.log
# summaries travel back (gpurun_out is capped at 64 MiB): metrics per kernel + stall hot spots
python tools/ncu_summary.py $T/top.ncu-rep --json $T/ncu_full_top.json > $T/ncu_full_top.txt 2>&1
python tools/ncu_hotspots.py $T/top.ncu-rep 20 > $T/ncu_full_top_hotspots.txt 2>&1
rm -f $T/top.ncu-rep; ls -la $T
