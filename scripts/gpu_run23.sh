python paper_2405_05047_b200/build.py
timeout 1500 python -m pytest tests -x -q -m gpu --deselect tests/test_gpu_fullsize.py > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/gpu_tests.log
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q -m gpu -k e6 > gpurun_out/gpu_full_e6.log 2>&1; echo "full e6 rc=$?"
tail -3 gpurun_out/gpu_full_e6.log
timeout 900 python bench.py --config e6 --steps 10 > gpurun_out/bench_e6.json 2> gpurun_out/bench_e6.err; echo "bench e6 rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_e6.json')); print('e6', round(d['value'],1), round(d['solve_ms'],2), d['config']['iterations_per_solve'], round(d['vcycle_only']['ms'],3), round(d['vcycle_only']['frac'],3), round(d['roofline']['frac'],3), round(d['spmv_hbm']['frac'],3), d['mixed_precision']['value'], d['cpu_baseline']['value'])"
