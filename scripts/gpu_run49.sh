python __graft_entry__.py build
timeout 1500 python -m pytest tests/test_gpu_vanka.py tests/test_gpu_ns.py -q -k "vanka" > gpurun_out/gpu_t49.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/gpu_t49.log
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r1s_c4ns_sweeps5.csv python scripts/profile_ns.py c4ns_sweep > gpurun_out/p_c4e.log 2>&1; echo "c4ns sweeps rc=$?"
timeout 900 python bench.py --config c4ns --steps 3 --vanka --no-cpu-baseline > gpurun_out/bench_c4ns_vanka.json 2> gpurun_out/bench_c4ns_vanka.err; echo "bench c4ns vanka rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_c4ns_vanka.json')); print(d['value'], d['time_step'])"
timeout 900 python bench.py --config ns --steps 20 --no-cpu-baseline > gpurun_out/bench_ns.json 2> gpurun_out/bench_ns.err; echo "bench ns rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_ns.json')); print(d['ms_per_step'], d['vanka_pressure']['ms_per_step'])"
