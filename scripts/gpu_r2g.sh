#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2g_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_distributed.py tests/test_gpu_ipc.py tests/test_gpu_mixed.py tests/test_gpu_update.py -x -q > gpurun_out/r2g_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2g_pytest.log
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-mixed"
timeout 900 $B > gpurun_out/r2g_c3.json 2> gpurun_out/r2g_c3.err
MGB200_KS4_SLICES=2000 timeout 900 $B > gpurun_out/r2g_c3_ks2l4.json 2> gpurun_out/r2g_c3_ks2l4.err
MGB200_KS2_SLICES=4096 MGB200_KS4_SLICES=256 timeout 900 $B > gpurun_out/r2g_c3_ks8.json 2> gpurun_out/r2g_c3_ks8.err
timeout 900 $B --config c2 > gpurun_out/r2g_c2.json 2> gpurun_out/r2g_c2.err
timeout 900 $B --config c5 > gpurun_out/r2g_c5.json 2> gpurun_out/r2g_c5.err
