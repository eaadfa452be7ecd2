"""Setup timing probe (development aid, under torchrun): the 7-point nd^3 cube
split over the ranks, setup run three times, SetupStats per run on rank 0.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 scripts/setup_probe.py 585
"""
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_02352_b200 as pb  # noqa: E402

nd = int(sys.argv[1]) if len(sys.argv) > 1 else 585
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
obj = [pb.unique_id() if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
rt = pb.Runtime(rank, rank, world, obj[0])
n = nd ** 3
starts = pb.uniform_partition(n, world)
b0, b1 = int(starts[rank]), int(starts[rank + 1])
L = pb.lib()
nnz = L.pairamg_poisson_nnz(7, nd, nd, nd, b0, b1)
rp = torch.empty(b1 - b0 + 1, dtype=torch.int64, device="cuda")
ci = torch.empty(nnz, dtype=torch.int64, device="cuda")
va = torch.empty(nnz, dtype=torch.float64, device="cuda")
pb._check(L.pairamg_poisson_device(rt.h, 7, nd, nd, nd, b0, b1, pb._ptr(rp), pb._ptr(ci), pb._ptr(va)))
s = pb.Solver(rt)
for it in range(3):
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s.setup(n, starts, rp, ci, va, cfg=pb.SetupConfig(3, 40 * nd, 40))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    st = s.setup_stats()
    if rank == 0:
        print(f"setup {it}: {dt:.3f} s  matching {st['t_matching']:.3f} spmm {st['t_spmm']:.3f} "
              f"spmm_comm {st['t_spmm_comm']:.3f} total {st['t_total']:.3f}", flush=True)
s.close()
rt.close()
dist.destroy_process_group()
