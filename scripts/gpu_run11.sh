timeout 900 python -m pytest tests/test_gpu_mixed.py -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/gpu_tests.log
timeout 900 python bench.py --steps 10 --no-cpu-baseline --precision mixed > gpurun_out/bench_c3_mixed.json 2> gpurun_out/bench_c3_mixed.err; echo "bench mixed rc=$?"
cat gpurun_out/bench_c3_mixed.json | python -c "import json,sys; d=json.load(sys.stdin); print(d['value'], d['solve_ms'], d['vcycle_only'], d['roofline']['frac'], d['roofline']['avg_launch_ms'])"
