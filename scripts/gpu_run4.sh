python paper_2405_05047_b200/build.py
timeout 1200 python -m pytest tests/test_gpu_distributed.py -x -q -m gpu > gpurun_out/gpu_dist.log 2>&1; echo "dist rc=$?"
tail -30 gpurun_out/gpu_dist.log
timeout 1200 python -m pytest tests -x -q -m gpu --deselect tests/test_gpu_distributed.py > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/gpu_tests.log
