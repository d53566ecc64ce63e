python __graft_entry__.py build
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -k "e6_edge or e6_vertex" > gpurun_out/gpu_t45.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gpu_t45.log
for cfg in e6_edge e6_vertex; do
timeout 900 python bench.py --config $cfg --steps 10 > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err; echo "bench $cfg rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_$cfg.json')); print(d['value'], d['solve_ms'], d['config']['iterations_per_solve'], d['vcycle_only']['ms'], d['paper_context'], d['cpu_baseline']['solve'], d['mixed_precision']['solve_ms'])"
done
