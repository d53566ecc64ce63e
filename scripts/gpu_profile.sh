#!/bin/bash
# ncu captures of one config (run only after the same command exited 0 without ncu):
#   TAG_CFG_launches.csv : launch list of one bench step (cold cache, serialised)
#   TAG_CFG_warm.csv     : the same with --cache-control none (warm)
#   TAG_CFG_full.ncu-rep : --set full of the finest-level kernels (sweep, residual, SpMV, R, P)
# usage: scripts/gpu_profile.sh TAG CFG [what...]   what in {launches, warm, full}
TAG=$1; CFG=$2; shift 2
WHAT=${*:-launches warm full}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv"
for w in $WHAT; do
  case $w in
    launches) MGB200_GMRES_LOOP=host timeout 900 ncu $M --log-file gpurun_out/${TAG}_${CFG}_launches.csv python scripts/profile_ops.py step --config $CFG > gpurun_out/${TAG}_${CFG}_launches.log 2>&1 ;;
    warm) MGB200_GMRES_LOOP=host timeout 900 ncu $M --cache-control none --log-file gpurun_out/${TAG}_${CFG}_warm.csv python scripts/profile_ops.py step --config $CFG > gpurun_out/${TAG}_${CFG}_warm.log 2>&1 ;;
    full) timeout 1200 ncu --set full --import-source on --clock-control none --profile-from-start off -o gpurun_out/${TAG}_${CFG}_full python scripts/profile_ops.py kernels --config $CFG > gpurun_out/${TAG}_${CFG}_full.log 2>&1 ;;
  esac
  echo "$w rc=$?"
done
