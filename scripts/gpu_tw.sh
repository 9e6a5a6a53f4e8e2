# trace kernel CTA width experiment (option trace_warps) + ncu metrics per variant
mkdir -p gpurun_out
for tw in 8 16 32 8; do TRACE_WARPS=$tw PROBE_REPS=7 timeout 300 python scripts/probe_ab.py >> gpurun_out/tw.jsonl 2>> gpurun_out/tw.err; done
for tw in 8 32; do
TRACE_WARPS=$tw PROBE_REPS=1 timeout 600 ncu --clock-control none -k regex:k_ray_policy2 -s 1 -c 1 --metrics gpu__time_duration.sum,sm__inst_executed.sum,l1tex__t_sector_hit_rate.pct,lts__t_sector_hit_rate.pct,smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio,smsp__average_warp_latency_issue_stalled_wait.ratio,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,lts__t_sectors_srcunit_tex_op_read.sum --csv python scripts/probe_ab.py > gpurun_out/tw_ncu_$tw.csv 2>&1
done
echo DONE
