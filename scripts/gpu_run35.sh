# No copy-back after pre-smoothing; k_ns_div / Vanka clamped loads: full -m gpu suite, initcheck probe, bench.
python __graft_entry__.py build
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -4 gpurun_out/gpu_tests.log
CS=/usr/local/cuda/bin/compute-sanitizer
for args in "ns graphs" "ch graphs"; do
timeout 600 $CS --tool initcheck --print-limit 2 python scripts/initcheck_probe.py $args > gpurun_out/initprobe.log 2>&1; echo "initcheck $args rc=$?"
grep -E "SUMMARY" gpurun_out/initprobe.log
done
timeout 900 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_c3.json')); print(d['value'], d['e2e']['value'], d['vcycle_only'], d['roofline']['frac'], d['mixed_precision']['value'], d['clocks'])"
timeout 900 python bench.py --config ns --steps 20 --no-cpu-baseline > gpurun_out/bench_ns.json 2> gpurun_out/bench_ns.err; echo "bench ns rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_ns.json')); print(d['ms_per_step'], d['table_ns_split_ms_per_step'], d['vanka_pressure']['ms_per_step'])"
timeout 900 python bench.py --config c4ns --steps 3 --vanka --no-cpu-baseline > gpurun_out/bench_c4ns_vanka.json 2> gpurun_out/bench_c4ns_vanka.err; echo "bench c4ns vanka rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_c4ns_vanka.json')); print(d['value'], d['time_step'], d['roofline']['avg_launch_ms'])"
timeout 900 python bench.py --config c4ns --steps 3 > gpurun_out/bench_c4ns.json 2> gpurun_out/bench_c4ns.err; echo "bench c4ns rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_c4ns.json')); print(d['value'], d['time_step'], d['e2e'])"
