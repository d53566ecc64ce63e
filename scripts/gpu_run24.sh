# Round-1 re-entry check: build, full -m gpu suite, smoke, default bench.
set -x
python __graft_entry__.py build
cat MEASURED_PEAKS.json > gpurun_out/measured_peaks.json 2>/dev/null
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "bench rc=$?"
cat gpurun_out/bench_c3.json | head -c 3000
