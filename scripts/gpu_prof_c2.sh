#!/bin/bash
# C2 (latency-bound small config): launch list of one graph-free V-cycle and --set full of the
# finest-level kernels.  usage: scripts/gpu_prof_c2.sh TAG [config]
TAG=${1:-p}; CFG=${2:-c2}
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/${TAG}_${CFG}_vcycle.csv python scripts/profile_ops.py vcycle --config $CFG > gpurun_out/${TAG}_vc.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -o gpurun_out/${TAG}_${CFG}_full python scripts/profile_ops.py kernels --config $CFG > gpurun_out/${TAG}_full.log 2>&1
ls -la gpurun_out/
