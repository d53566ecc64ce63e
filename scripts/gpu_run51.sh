# Transfer kernels: the < UB tail entries as one batch. Full suite, bench, kernel times.
python __graft_entry__.py build
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/gpu_tests.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_c3.json')); print(d['value'], d['e2e']['value'], d['vcycle_only']['ms'], d['vcycle_only']['frac'], d['vcycle_levels']['ms'])"
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r1s_kernels_c3.csv python scripts/profile_ops.py kernels > gpurun_out/p2.log 2>&1; echo "kernels rc=$?"
