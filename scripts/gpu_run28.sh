# Vanka kernel v2 (multi-patch warps, interleaved inverse layout): parity, bench; ncu of NS step and C4 sweeps.
python __graft_entry__.py build
timeout 1500 python -m pytest tests/test_gpu_vanka.py -q > gpurun_out/gpu_vanka.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/gpu_vanka.log
timeout 900 python bench.py --config c4ns --steps 3 --vanka --no-cpu-baseline > gpurun_out/bench_c4ns_vanka.json 2> gpurun_out/bench_c4ns_vanka.err; echo "bench c4ns vanka rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_c4ns_vanka.json')); print(d['value'], d['config']['lin_its'], d['time_step'])"
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r1r_ns_step_launches.csv python scripts/profile_ns.py ns_step > gpurun_out/p_ns.log 2>&1; echo "ns step rc=$?"
timeout 600 $NCU --profile-from-start off --set full --import-source on --clock-control none -k regex:k_ns -o gpurun_out/r1r_ns_kernels python scripts/profile_ns.py ns_step > gpurun_out/p_ns2.log 2>&1; echo "ns kernels rc=$?"
timeout 600 $NCU --profile-from-start off --set full --import-source on --clock-control none -o gpurun_out/r1r_c4ns_sweeps python scripts/profile_ns.py c4ns_sweep > gpurun_out/p_c4.log 2>&1; echo "c4ns sweeps rc=$?"
ls -la gpurun_out | grep r1r
