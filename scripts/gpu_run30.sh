# Fused small-level mean projection: Neumann + NS parity, NS bench (Jacobi + Vanka pressure smoother).
python __graft_entry__.py build
timeout 1500 python -m pytest tests/test_gpu_neumann.py tests/test_gpu_ns.py -q > gpurun_out/gpu_ns.log 2>&1; echo "tests rc=$?"
tail -4 gpurun_out/gpu_ns.log
timeout 900 python bench.py --config ns --steps 20 > gpurun_out/bench_ns.json 2> gpurun_out/bench_ns.err; echo "bench ns rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_ns.json')); print(d['ms_per_step'], d['config']['pressure_gmres_per_step'], d['table_ns_split_ms_per_step'], d['vanka_pressure'], d['gpu_launches'])"
timeout 900 python bench.py --config pres --steps 10 --no-cpu-baseline --no-mixed > gpurun_out/bench_pres.json 2> gpurun_out/bench_pres.err; echo "bench pres rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_pres.json')); print(d['value'], d['solve_ms'], d['config']['iterations_per_solve'], d['vcycle_only'])"
