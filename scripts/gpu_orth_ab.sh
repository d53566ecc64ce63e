#!/bin/bash
# Same-box A/B of the DCGS2 kernel implementations (MGB200_DCGS_KERNEL = ws | reg | tma):
# bench lines with the orthogonalisation side line (MGS headline, DCGS2 side).
# usage: scripts/gpu_orth_ab.sh TAG "cfgs" "kernels"
TAG=$1; CFGS=$2; KS=${3:-"ws reg"}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-mixed"
for cfg in $CFGS; do for rep in 1 2; do for k in $KS; do
  MGB200_DCGS_KERNEL=$k timeout 900 $B --config $cfg > gpurun_out/${TAG}_${cfg}_${k}$rep.json 2> gpurun_out/${TAG}_${cfg}_${k}$rep.err
  python -c "
import json; d=json.loads(open('gpurun_out/${TAG}_${cfg}_${k}$rep.json').read().strip().splitlines()[-1]); o=d['orth_other']
print('%-8s %-4s mgs %9.2f %8.3f ms | dcgs2 %9.2f %8.3f ms its %s' % ('$cfg', '$k', d['value'], d['ms_per_step'], o['value'], o['solve_ms'], o['iterations_per_solve']))"
done; done; done
