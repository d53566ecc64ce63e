python __graft_entry__.py build
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --profile-from-start off -k regex:k_ns --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r1s_ns_kernels.csv python scripts/profile_ns.py ns_step > gpurun_out/p_ns3.log 2>&1; echo "ns kernels rc=$?"
