#!/bin/bash
# ncu launch list of exactly the timed steps of the default bench command (MGB200_PROFILE_TIMED
# opens the profiler range around the timed loop; the GMRES cycle runs one graph per Arnoldi
# step so its kernels are visible to ncu -- the same kernels as the conditional cycle graph).
# usage: scripts/gpu_launchlist.sh TAG [bench args...]
TAG=$1; shift
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
MGB200_PROFILE_TIMED=1 MGB200_GMRES_LOOP=host timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/${TAG}_bench_timed_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-mixed --no-orth-side "$@" > gpurun_out/${TAG}_bench_under_ncu.log 2>&1
echo "ncu rc=$?"
