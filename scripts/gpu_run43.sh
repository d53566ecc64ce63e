python __graft_entry__.py build
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -k "td_l10" > gpurun_out/gpu_t43.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gpu_t43.log
timeout 900 python bench.py --config td_l10 --steps 10 > gpurun_out/bench_td_l10.json 2> gpurun_out/bench_td_l10.err; echo "bench td_l10 rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_td_l10.json')); print(d['value'], d['solve_ms'], d['config']['iterations_per_solve'], d['vcycle_only']['ms'], d['vcycle_only']['frac'], d['paper_context'], d['cpu_baseline']['solve'], d['mixed_precision']['solve_ms'])"
timeout 900 python bench.py --config e6 --steps 10 > gpurun_out/bench_e6.json 2> gpurun_out/bench_e6.err; echo "bench e6 rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_e6.json')); print(d['value'], d['solve_ms'], d['config']['iterations_per_solve'], d['paper_context'], d['cpu_baseline']['solve'])"
