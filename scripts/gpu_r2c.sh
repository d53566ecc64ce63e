#!/bin/bash
# round 2: device-side GMRES loop (parity + before/after timings), IPC tests,
# C5 weak-scaling bench at N=1 and N=2 (two processes sharing the GPU).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2c_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_ipc.py tests/test_gpu_parity.py -x -q > gpurun_out/r2c_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2c_pytest.log
for cfg in c1 c2 e6_vertex ns; do
  for mode in host device; do
    MGB200_GMRES_LOOP=$mode timeout 600 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --no-mixed > gpurun_out/r2c_${cfg}_${mode}.json 2> gpurun_out/r2c_${cfg}_${mode}.err
  done
done
timeout 900 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline --no-mixed > gpurun_out/r2c_c5_n1.json 2> gpurun_out/r2c_c5_n1.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29535 bench.py --gpus 2 --config c5 --steps 2 --warmup 3 > gpurun_out/r2c_c5_n2.json 2> gpurun_out/r2c_c5_n2.err
echo "rc=$?" >> gpurun_out/r2c_c5_n2.err
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-solve > gpurun_out/r2c_c3.json 2> gpurun_out/r2c_c3.err
