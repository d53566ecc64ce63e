python paper_2405_05047_b200/build.py
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -4 gpurun_out/gpu_tests.log
timeout 900 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "bench rc=$?"
cat gpurun_out/bench_c3.json; tail -2 gpurun_out/bench_c3.err
timeout 900 /usr/local/cuda/bin/ncu --profile-from-start off --cache-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r1c_launches_warm.csv python scripts/profile_ops.py step > gpurun_out/prof_step.log 2>&1; echo "ncu rc=$?"
