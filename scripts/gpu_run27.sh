# Vanka smoother parity, Newton parity, c4ns with Vanka vs block-Jacobi.
python __graft_entry__.py build
timeout 1500 python -m pytest tests/test_gpu_vanka.py tests/test_gpu_newton.py -q > gpurun_out/gpu_vanka.log 2>&1; echo "tests rc=$?"
tail -25 gpurun_out/gpu_vanka.log
timeout 900 python bench.py --config c4ns --steps 3 --vanka --no-cpu-baseline > gpurun_out/bench_c4ns_vanka.json 2> gpurun_out/bench_c4ns_vanka.err; echo "bench c4ns vanka rc=$?"
tail -3 gpurun_out/bench_c4ns_vanka.err; head -c 1800 gpurun_out/bench_c4ns_vanka.json; echo
