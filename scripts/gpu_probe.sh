timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 scripts/probe_nccl.py 2>&1 | grep -E "rank|recv|Duplicate|WARN|Error" | head -20
nvidia-smi -q | grep -i -E "MIG Mode|Current  |Compute Mode" | head
nproc; free -g | head -2
