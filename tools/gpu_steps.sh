# usage: bash tools/gpu_steps.sh TAG -- one ncu capture (§8(d) counters) of every config's timed
# kernels (tools/prof_steps.sh: the bench step, the split build, the split eval; one process per
# config), parsed here by tools/traffic_capture.py into profiles/<round>/ncu_steps.json and
# profiles/traffic.json (what bench.py reports as roofline.traffic).
T=gpurun_out/${1:-r02s}; mkdir -p $T
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_write.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,smsp__inst_executed_pipe_fp64.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio,smsp__average_warp_latency_issue_stalled_short_scoreboard.ratio,smsp__average_warp_latency_issue_stalled_math_pipe_throttle.ratio,smsp__average_warp_latency_issue_stalled_barrier.ratio,launch__registers_per_thread
bash tools/prof_steps.sh > $T/plain.log 2>&1; echo "plain rc=$?"
ncu --target-processes all --metrics $M --clock-control none -k regex:"k_|k1_|k4_" --csv --log-file $T/steps.csv bash tools/prof_steps.sh > $T/ncu.log 2>&1; echo "ncu rc=$?"; tail -3 $T/ncu.log; wc -l $T/steps.csv
