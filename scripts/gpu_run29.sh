# Full -m gpu suite, smoke, default bench, NS step with the Vanka pressure smoother.
python __graft_entry__.py build
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -8 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py --config ns --steps 20 --vanka --omega 0.8 --no-cpu-baseline > gpurun_out/bench_ns_vanka.json 2> gpurun_out/bench_ns_vanka.err; echo "bench ns vanka rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_ns_vanka.json')); print(d['ms_per_step'], d['config']['pressure_gmres_per_step'], d['table_ns_split_ms_per_step'])"
timeout 900 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_c3.json')); print(d['value'], d['e2e']['value'], d['vcycle_only'], d['roofline']['frac'], d['gpu_launches'], d['clocks'])"
