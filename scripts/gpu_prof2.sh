NCU=/usr/local/cuda/bin/ncu
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,launch__grid_size,launch__registers_per_thread,launch__occupancy_limit_registers,sm__throughput.avg.pct_of_peak_sustained_elapsed
timeout 900 $NCU --profile-from-start off --cache-control none --metrics $M --clock-control none --csv --log-file gpurun_out/r1_vcycle_metrics.csv python scripts/profile_ops.py vcycle > gpurun_out/prof_vc.log 2>&1; echo "ncu rc=$?"
tail -2 gpurun_out/prof_vc.log
