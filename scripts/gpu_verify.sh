#!/bin/bash
# Verification at HEAD on one B200: build, GPU suite, smoke, default bench line and secondaries.
# usage: scripts/gpu_verify.sh TAG [configs...]
TAG=${1:-v}; shift
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { echo build failed; tail gpurun_out/${TAG}_build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
tail -3 gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${TAG}_smoke.log 2>&1
tail -1 gpurun_out/${TAG}_smoke.log
for cfg in "$@"; do
  timeout 1500 python bench.py --config $cfg > gpurun_out/${TAG}_$cfg.json 2> gpurun_out/${TAG}_$cfg.err
  head -c 600 gpurun_out/${TAG}_$cfg.json; echo
done
