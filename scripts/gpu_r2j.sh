#!/bin/bash
# PDL A/B (same box) + GPU suite without the slow full-size tests
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2j_build.log 2>&1
timeout 1800 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/r2j_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2j_pytest.log
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-mixed"
for cfg in c1 c2 e6_vertex td_l10 ns c3; do
  for pdl in 1 0; do
    MGB200_PDL=$pdl timeout 900 $B --config $cfg > gpurun_out/r2j_${cfg}_pdl$pdl.json 2> gpurun_out/r2j_${cfg}_pdl$pdl.err
  done
done
