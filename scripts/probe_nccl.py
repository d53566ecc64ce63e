import os, torch, torch.distributed as dist
rank = int(os.environ["RANK"]); ws = int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(0)
os.environ.setdefault("NCCL_DEBUG", "WARN")
try:
    dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
    t = torch.ones(4, device="cuda") * (rank + 1)
    dist.all_reduce(t)
    torch.cuda.synchronize()
    print(f"rank {rank}: nccl allreduce ok {t.tolist()}", flush=True)
    if rank == 0:
        dist.send(torch.arange(3., device="cuda"), 1)
    else:
        r = torch.empty(3, device="cuda"); dist.recv(r, 0); torch.cuda.synchronize(); print("recv", r.tolist(), flush=True)
except Exception as e:
    print(f"rank {rank}: nccl failed: {type(e).__name__}: {str(e)[:300]}", flush=True)
