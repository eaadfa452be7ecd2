"""Probe: can two NCCL ranks share one GPU? (decides the 1-GPU multi-rank test transport)."""
import os, torch, torch.distributed as dist
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
t = torch.ones(4, device="cuda:0") * (dist.get_rank() + 1)
try:
    dist.all_reduce(t)
    torch.cuda.synchronize()
    print("rank", dist.get_rank(), "allreduce ok", t.tolist(), flush=True)
except Exception as e:
    print("rank", dist.get_rank(), "FAILED", type(e).__name__, str(e)[:300], flush=True)
dist.destroy_process_group()
