#!/bin/bash
# Same-box A/B: bench lines of several configs with build/libmgb200_base.so (A) and the
# in-tree library (B), plus optional env variants of B.
# usage: scripts/gpu_ab.sh TAG "cfg1 cfg2 ..." ["ENV=1 ENV2=2" ...]
TAG=$1; CFGS=$2; shift 2
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-mixed --no-orth-side"
summ() { python -c "
import json,sys
try:
  d=json.loads(open('$1').read().strip().splitlines()[-1])
  print('%-28s %-10s value %9.2f  ms %8.3f  vcycle %8.4f ms frac %.3f  e2e %s' % ('$2', '$3', d['value'], d['ms_per_step'], d['vcycle_only']['ms'], d['vcycle_only']['frac'], round(d['e2e']['value'],2)))
except Exception as e: print('$2 $3 failed', e)
"; }
for cfg in $CFGS; do
  for rep in 1 2; do
    MGB200_LIB=$PWD/build/libmgb200_base.so timeout 900 $B --config $cfg > gpurun_out/${TAG}_${cfg}_A$rep.json 2> gpurun_out/${TAG}_${cfg}_A$rep.err
    summ gpurun_out/${TAG}_${cfg}_A$rep.json $cfg A$rep
    timeout 900 $B --config $cfg > gpurun_out/${TAG}_${cfg}_B$rep.json 2> gpurun_out/${TAG}_${cfg}_B$rep.err
    summ gpurun_out/${TAG}_${cfg}_B$rep.json $cfg B$rep
    i=0
    for v in "$@"; do
      i=$((i+1))
      env $v timeout 900 $B --config $cfg > gpurun_out/${TAG}_${cfg}_V$i$rep.json 2> gpurun_out/${TAG}_${cfg}_V$i$rep.err
      summ gpurun_out/${TAG}_${cfg}_V$i$rep.json $cfg "V$i:$v"
    done
  done
done
