for cfg in c2 c4 c5; do
timeout 1200 python bench.py --config $cfg --steps 10 > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err; echo "bench $cfg rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_$cfg.json')); print('$cfg', round(d['value'],1), round(d['solve_ms'],2), d['config']['iterations_per_solve'], round(d['vcycle_only']['ms'],3), round(d['vcycle_only']['frac'],3), round(d['roofline']['frac'],3), round(d['spmv_hbm']['frac'],3), d['mixed_precision']['value'] if d['mixed_precision'] else None, d['cpu_baseline']['value'])"
done
