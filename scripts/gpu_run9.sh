timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -6 gpurun_out/gpu_tests.log
