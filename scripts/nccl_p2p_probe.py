"""Latency of a 512 KB NCCL send/recv pair between 2 GPUs (torch.distributed),
eager and inside a CUDA graph.  Development aid for the halo exchange."""
import os
import time

import torch
import torch.distributed as dist

dist.init_process_group("nccl")
r = dist.get_rank()
torch.cuda.set_device(r)
n = 65536
sb = torch.ones(n, dtype=torch.float64, device="cuda")
rb = torch.empty(n, dtype=torch.float64, device="cuda")
peer = 1 - r


def xchg():
    ops = [dist.P2POp(dist.isend, sb, peer), dist.P2POp(dist.irecv, rb, peer)]
    for w in dist.batch_isend_irecv(ops):
        w.wait()


for _ in range(20):
    xchg()
torch.cuda.synchronize()
dist.barrier()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(200):
    xchg()
e1.record()
torch.cuda.synchronize()
print(f"rank {r}: eager send/recv 512 KB: {e0.elapsed_time(e1) / 200 * 1e3:.1f} us")
# with a concurrent bandwidth-bound kernel on another stream
big = torch.empty(2 ** 28, dtype=torch.float64, device="cuda")
s2 = torch.cuda.Stream()
dist.barrier()
torch.cuda.synchronize()
with torch.cuda.stream(s2):
    for _ in range(20):
        big.mul_(1.0000001)
e0.record()
for _ in range(50):
    xchg()
e1.record()
torch.cuda.synchronize()
print(f"rank {r}: send/recv 512 KB under a concurrent HBM-bound kernel: {e0.elapsed_time(e1) / 50 * 1e3:.1f} us")
dist.destroy_process_group()
