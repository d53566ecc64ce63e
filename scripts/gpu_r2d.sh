#!/bin/bash
# round 2: full GPU suite with the SELL-C transfers, ncu of the new transfer
# kernels (and the old ones for comparison), C3 bench.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2d_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2d_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2d_pytest.log
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:"k_tsell|k_transfer" -o gpurun_out/r2d_tsell python scripts/profile_ops.py kernels --config c3 > gpurun_out/r2d_ncu.log 2>&1
MGB200_TSELL=0 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off -k regex:"k_tsell|k_transfer" --csv python scripts/profile_ops.py kernels --config c3 > gpurun_out/r2d_ncu_old.csv 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-solve > gpurun_out/r2d_c3.json 2> gpurun_out/r2d_c3.err
MGB200_TSELL=0 timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-mixed > gpurun_out/r2d_c3_old.json 2> gpurun_out/r2d_c3_old.err
