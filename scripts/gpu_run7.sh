python paper_2405_05047_b200/build.py
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/gpu_tests.log
timeout 900 python bench.py --config c5 --steps 5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "bench c5 rc=$?"
cat gpurun_out/bench_c5.json; tail -3 gpurun_out/bench_c5.err
timeout 600 python bench.py --config c4 --steps 10 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench c4 rc=$?"
cat gpurun_out/bench_c4.json; tail -3 gpurun_out/bench_c4.err
