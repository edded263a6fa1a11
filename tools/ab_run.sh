# scratch (development aid): ncu of the FFMA conv, default vs libmdh_b200_alt.so
ALT=$PWD/paper_2405_05118_b200/libmdh_b200_alt.so
M="smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,gpu__time_duration.sum,smsp__average_warp_latency_issue_stalled_dispatch_stall.ratio,smsp__average_warp_latency_issue_stalled_not_selected.ratio,smsp__average_warp_latency_issue_stalled_math_pipe_throttle.ratio,smsp__average_warp_latency_issue_stalled_short_scoreboard.ratio,smsp__average_warp_latency_issue_stalled_wait.ratio,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fmalite_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fmalite.avg.pct_of_peak_sustained_active"
for v in "" "MDHB_LIB=$ALT"; do
  echo "== $v"
  env $v timeout 300 ncu --metrics $M --clock-control none -k regex:ffma_conv_tma -c 2 python tools/profile_routines.py mcc_nhwc 2>&1 | grep -E "ffma_conv_tma|smsp__|sm__|gpu__" | head -40
done
