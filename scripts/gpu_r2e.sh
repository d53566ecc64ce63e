#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2e_build.log 2>&1
timeout 600 python scripts/tune_tsell.py c3 > gpurun_out/r2e_tune_c3.txt 2>&1
timeout 600 python scripts/tune_tsell.py c5 > gpurun_out/r2e_tune_c5.txt 2>&1
timeout 600 python scripts/tune_tsell.py c2 > gpurun_out/r2e_tune_c2.txt 2>&1
