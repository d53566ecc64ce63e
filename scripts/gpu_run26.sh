# Newton (C4 per SURVEY §8(d)) parity incl. inexact Newton, c4ns and ns bench lines.
python __graft_entry__.py build
timeout 1500 python -m pytest tests/test_gpu_newton.py -x -q > gpurun_out/gpu_newton.log 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/gpu_newton.log
timeout 900 python bench.py --config c4ns --steps 3 > gpurun_out/bench_c4ns.json 2> gpurun_out/bench_c4ns.err; echo "bench c4ns rc=$?"
tail -3 gpurun_out/bench_c4ns.err; head -c 1800 gpurun_out/bench_c4ns.json; echo
timeout 900 python bench.py --config ns --steps 20 > gpurun_out/bench_ns.json 2> gpurun_out/bench_ns.err; echo "bench ns rc=$?"
tail -3 gpurun_out/bench_ns.err; head -c 2500 gpurun_out/bench_ns.json
