# Final verification of this session's code: full -m gpu suite, smoke, default bench.
python __graft_entry__.py build
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -4 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_c3.json')); print(d['value'], d['e2e']['value'], d['vcycle_only']['ms'], d['vcycle_only']['frac'], d['roofline']['frac'], d['spmv_hbm']['frac'], d['mixed_precision']['value'], d['gpu_launches'], d['clocks'])"
