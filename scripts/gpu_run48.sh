python __graft_entry__.py build
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --profile-from-start off --set full --import-source on -k regex:k_vanka --clock-control none -o gpurun_out/r1s_vanka_full python scripts/profile_ns.py c4ns_sweep > gpurun_out/p_v.log 2>&1; echo "rc=$?"
