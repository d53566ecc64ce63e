#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2h_build.log 2>&1
python paper_2405_05047_b200/build.py --variant /tmp/lib_minb0.so -DMGB200_KS_MINB=0 >> gpurun_out/r2h_build.log 2>&1 &
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_distributed.py tests/test_gpu_ipc.py tests/test_gpu_mixed.py tests/test_gpu_update.py tests/test_gpu_bench_contract.py -x -q > gpurun_out/r2h_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2h_pytest.log
wait
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-mixed"
for rep in 1 2; do
  timeout 900 $B > gpurun_out/r2h_c3_new_$rep.json 2> gpurun_out/r2h_c3_new_$rep.err
  MGB200_LIB=/tmp/lib_minb0.so timeout 900 $B > gpurun_out/r2h_c3_minb0_$rep.json 2> gpurun_out/r2h_c3_minb0_$rep.err
done
timeout 900 $B --config c2 > gpurun_out/r2h_c2_new.json 2> gpurun_out/r2h_c2_new.err
MGB200_LIB=/tmp/lib_minb0.so timeout 900 $B --config c2 > gpurun_out/r2h_c2_minb0.json 2> gpurun_out/r2h_c2_minb0.err
timeout 900 $B --config c5 > gpurun_out/r2h_c5_new.json 2> gpurun_out/r2h_c5_new.err
