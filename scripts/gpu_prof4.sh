NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r1z_launches_c3.csv python scripts/profile_ops.py step > gpurun_out/p1.log 2>&1; echo "step rc=$?"
timeout 900 $NCU --profile-from-start off --set full --import-source on --clock-control none -o gpurun_out/r1z_c3_kernels python scripts/profile_ops.py kernels > gpurun_out/p2.log 2>&1; echo "kernels rc=$?"
timeout 900 $NCU --profile-from-start off --set full --import-source on --clock-control none -o gpurun_out/r1z_c3_kernels_mixed python scripts/profile_ops.py kernels --mixed > gpurun_out/p3.log 2>&1; echo "mixed rc=$?"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size
timeout 900 $NCU --profile-from-start off --cache-control none --metrics $M --clock-control none --csv --log-file gpurun_out/r1z_vcycle_warm_c3.csv python scripts/profile_ops.py vcycle > gpurun_out/p4.log 2>&1; echo "vcycle rc=$?"
ls -la gpurun_out | grep r1z
