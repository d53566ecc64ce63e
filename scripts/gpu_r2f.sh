#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2f_build.log 2>&1
timeout 900 python scripts/tune_tsell.py c3 > gpurun_out/r2f_tune_c3.txt 2>&1
timeout 900 python scripts/tune_tsell.py c5 > gpurun_out/r2f_tune_c5.txt 2>&1
timeout 600 python scripts/tune_tsell.py c2 > gpurun_out/r2f_tune_c2.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:"k_sell_apply" -o gpurun_out/r2f_level4 python scripts/profile_ops.py kernels --config c3 --level 4 > gpurun_out/r2f_ncu4.log 2>&1
MGB200_TSELL_R=2,1 timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-mixed > gpurun_out/r2f_c3.json 2> gpurun_out/r2f_c3.err
MGB200_TSELL_R=2,1 MGB200_MGS_ALT=0 timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-mixed > gpurun_out/r2f_c3_noalt.json 2> gpurun_out/r2f_c3_noalt.err
