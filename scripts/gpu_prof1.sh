NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r1_launches_c3.csv python scripts/profile_ops.py step > gpurun_out/prof_step.log 2>&1; echo "step rc=$?"
tail -3 gpurun_out/prof_step.log
timeout 900 $NCU --profile-from-start off --set full --import-source on --clock-control none -o gpurun_out/r1_c3_kernels python scripts/profile_ops.py kernels > gpurun_out/prof_kernels.log 2>&1; echo "kernels rc=$?"
tail -3 gpurun_out/prof_kernels.log
ls -la gpurun_out/
