timeout 1500 python -m pytest tests -x -q -m gpu --deselect tests/test_gpu_fullsize.py > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/gpu_tests.log
for i in 1 2 3; do timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "coarse_tail" 2>&1 | tail -1; done
timeout 900 python bench.py --steps 10 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_c3.json')); print(d['value'], d['solve_ms'], d['vcycle_only']['ms'], d['mixed_precision']['value'])"
