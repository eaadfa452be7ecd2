"""Multi-rank timing probe (development aid): Poisson cube or z-box over the
ranks of a torchrun job, setup twice (cold / warm stats), solve twice, then
one solve with kernel timing: per-level V-cycle time and level-0 classes.

    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 \
        scripts/mp_probe.py --nd 585 [--zbox] [--stencil 7]
"""
import argparse
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, ".")
import paper_2303_02352_b200 as pb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--nd", type=int, default=256)
ap.add_argument("--stencil", type=int, default=7)
ap.add_argument("--zbox", action="store_true")
ap.add_argument("--setups", type=int, default=2)
a = ap.parse_args()
rank, world, local = (int(os.environ.get(k, d)) for k, d in (("RANK", 0), ("WORLD_SIZE", 1), ("LOCAL_RANK", 0)))
torch.cuda.set_device(local)
uid = None
if world > 1:
    dist.init_process_group("gloo")
    obj = [pb.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    uid = obj[0]
t0 = time.perf_counter()
rt = pb.Runtime(local, rank, world, uid)
if rank == 0:
    print(f"runtime create {time.perf_counter() - t0:.3f}s", flush=True)
nx = ny = a.nd
nz = a.nd * world if a.zbox else a.nd
n = nx * ny * nz
starts = pb.uniform_partition(n, world)
b0, b1 = int(starts[rank]), int(starts[rank + 1])
L = pb.lib()
nnz = L.pairamg_poisson_nnz(a.stencil, nx, ny, nz, b0, b1)
rp = torch.empty(b1 - b0 + 1, dtype=torch.int64, device="cuda")
ci = torch.empty(nnz, dtype=torch.int64, device="cuda")
va = torch.empty(nnz, dtype=torch.float64, device="cuda")
pb._check(L.pairamg_poisson_device(rt.h, a.stencil, nx, ny, nz, b0, b1, pb._ptr(rp), pb._ptr(ci), pb._ptr(va)))
s = pb.Solver(rt)


def bar():
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()


for i in range(a.setups):
    bar()
    t0 = time.perf_counter()
    s.setup(n, starts, rp, ci, va, cfg=pb.SetupConfig(3, 40 * a.nd, 40))
    bar()
    ts = time.perf_counter() - t0
    st = s.setup_stats()
    if rank == 0:
        print(f"setup {i}: {ts:.3f}s matching {st['t_matching']:.3f} spmm {st['t_spmm']:.3f} "
              f"spmm_comm {st['t_spmm_comm']:.3f} total {st['t_total']:.3f}", flush=True)
b = torch.ones(b1 - b0, dtype=torch.float64, device="cuda")
for i in range(2):
    u = torch.zeros(b1 - b0, dtype=torch.float64, device="cuda")
    bar()
    r = s.solve(b, u)
    if rank == 0:
        print(f"solve {i}: {r.iterations} it, {r.t_solve_s * 1e3:.2f} ms, {r.t_solve_s * 1e3 / r.iterations:.3f} ms/iter",
              flush=True)
s.set_kernel_timing(True)
u = torch.zeros(b1 - b0, dtype=torch.float64, device="cuda")
bar()
r = s.solve(b, u)
s.set_kernel_timing(False)
sizes = s.level_sizes()
lines = [f"rank {rank}: timed solve {r.t_solve_s * 1e3 / r.iterations:.3f} ms/iter"]
for k in range(min(len(sizes), 16)):
    t = s.kernel_timing(4 + k)
    if t["launches"]:
        lines.append(f"  level {k} rows {sizes[k][0]:>10d}: {t['ms'] / r.iterations * 1e3:8.1f} us/iter own work")
for k, name in enumerate(["L0 sweep", "L0 resid", "L0 spmv+dots", "update", "L0 zs-sweep", "L0 prolong-sweep"]):
    t = s.kernel_timing(k)
    if t["launches"]:
        lines.append(f"  {name}: {t['launches']} x {t['ms'] / t['launches'] * 1e3:.1f} us")
for q in range(world):
    if q == rank:
        print("\n".join(lines), flush=True)
    if world > 1:
        dist.barrier()
s.close()
rt.close()
if world > 1:
    dist.destroy_process_group()
