#!/bin/bash
# round 2: new parity tests (restart/truncation, >30 its, full-size C3/C5 element-wise +
# iteration parity), the multi-process IPC transport tests, a 2-rank bench on one GPU.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2b_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_ipc.py tests/test_gpu_parity.py -x -q > gpurun_out/r2b_pytest_a.log 2>&1
echo "rc=$?" >> gpurun_out/r2b_pytest_a.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/r2b_bench2.json 2> gpurun_out/r2b_bench2.err
echo "rc=$?" >> gpurun_out/r2b_bench2.err
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q -k "vcycle_elementwise or iterations_match_oracle" > gpurun_out/r2b_pytest_full.log 2>&1
echo "rc=$?" >> gpurun_out/r2b_pytest_full.log
