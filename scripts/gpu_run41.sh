# Current-code evidence: launch list of one C3 step + full capture of the fine kernels; Vanka parity.
python __graft_entry__.py build
timeout 900 python -m pytest tests/test_gpu_vanka.py -q > gpurun_out/gpu_t41.log 2>&1; echo "vanka tests rc=$?"; tail -1 gpurun_out/gpu_t41.log
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r1s_launches_c3.csv python scripts/profile_ops.py step > gpurun_out/p1.log 2>&1; echo "step rc=$?"
timeout 900 $NCU --profile-from-start off --set full --import-source on --clock-control none -o gpurun_out/r1s_c3_kernels python scripts/profile_ops.py kernels > gpurun_out/p2.log 2>&1; echo "kernels rc=$?"
ls -la gpurun_out | grep r1s
