python __graft_entry__.py build
timeout 1500 python -m pytest tests/test_gpu_vanka.py tests/test_gpu_ns.py -q -k "vanka" > gpurun_out/gpu_t50.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/gpu_t50.log
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r1s_c4ns_sweeps6.csv python scripts/profile_ns.py c4ns_sweep > gpurun_out/p_c4f.log 2>&1; echo "c4ns sweeps rc=$?"
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool memcheck python scripts/sanitize_next.py 2>&1 | grep -E "SUMMARY|ok$"; echo memcheck
