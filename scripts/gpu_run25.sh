# Newton (C4 per SURVEY §8(d)): parity tests, re-run of update/NS tests, smoke, c4ns bench line.
python __graft_entry__.py build
timeout 1500 python -m pytest tests/test_gpu_newton.py tests/test_gpu_update.py tests/test_gpu_ns.py -x -q > gpurun_out/gpu_newton.log 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/gpu_newton.log
timeout 900 python bench.py --config c4ns --steps 3 > gpurun_out/bench_c4ns.json 2> gpurun_out/bench_c4ns.err; echo "bench rc=$?"
tail -5 gpurun_out/bench_c4ns.err; head -c 2500 gpurun_out/bench_c4ns.json
