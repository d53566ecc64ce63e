#!/bin/bash
# round-2 probe: NCCL with 2 ranks on one GPU, CUDA IPC across processes on one
# device, ncu --set full (with source) of the C3 finest-level transfer kernels.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt 2>&1
timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 scripts/probe_nccl.py > gpurun_out/r2a_nccl.log 2>&1
echo "nccl rc=$?" >> gpurun_out/r2a_nccl.log
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_transfer -o gpurun_out/r2a_transfer python scripts/profile_ops.py kernels --config c3 > gpurun_out/r2a_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r2a_ncu.log
