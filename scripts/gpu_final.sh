#!/bin/bash
# Round verification on one B200: GPU suite + smoke, the default bench line (full contract) and
# secondary lines, the reference arm, a launch list of one timed C3 step and ncu traffic.
# usage: scripts/gpu_final.sh TAG
TAG=${1:-f}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { tail gpurun_out/${TAG}_build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${TAG}_smoke.log 2>&1; tail -1 gpurun_out/${TAG}_smoke.log
timeout 1500 python bench.py > gpurun_out/${TAG}_c3.json 2> gpurun_out/${TAG}_c3.err; echo "bench c3 rc=$?"
for cfg in c2 c5 c4 e6 td_l10 c1; do
  timeout 1200 python bench.py --config $cfg --no-cpu-solve > gpurun_out/${TAG}_$cfg.json 2> gpurun_out/${TAG}_$cfg.err; echo "bench $cfg rc=$?"
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err; echo "ref rc=$?"
MGB200_GMRES_LOOP=host timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/${TAG}_c3_step_launches.csv python scripts/profile_ops.py step --config c3 > gpurun_out/${TAG}_step.log 2>&1; echo "ncu step rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 3200 -c 1200 --csv --log-file gpurun_out/${TAG}_bench_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-mixed --no-orth-side > gpurun_out/${TAG}_bench_under_ncu.log 2>&1; echo "ncu bench rc=$?"
timeout 900 python bench.py --config ns > gpurun_out/${TAG}_ns.json 2> gpurun_out/${TAG}_ns.err; echo "bench ns rc=$?"
timeout 900 python bench.py --config pres --no-cpu-solve > gpurun_out/${TAG}_pres.json 2> gpurun_out/${TAG}_pres.err; echo "bench pres rc=$?"
# the N > 1 path (two processes time-slicing the one GPU through the IPC transport: functional)
MGB200_TRANSPORT=ipc timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config c5 --steps 3 --warmup 3 > gpurun_out/${TAG}_c5_n2_ipc.json 2> gpurun_out/${TAG}_c5_n2_ipc.err; echo "bench c5 n2 ipc rc=$?"
