"""Kernel timeline of one FCG solve via CUPTI (torch.profiler), one process
per GPU (run plainly for N = 1 or under torchrun for N > 1).  Unlike ncu
this does not replay kernels, so it works on the multi-rank split launches
whose boundary blocks wait on a peer GPU.  Writes per rank:
  gpurun_out/trace/<tag>_r<rank>.json  -- per-kernel count / mean / total us,
      device busy time, first-to-last span and the idle gaps.
Weak problem as bench.py: nd x nd x (nd * world), z-slab row blocks."""
import argparse
import collections
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_02352_b200 as pb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--stencil", type=int, default=7)
ap.add_argument("--nd", type=int, default=256)
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--replicate-rows", type=int, default=2500000)
ap.add_argument("--tag", default="t")
a = ap.parse_args()

world = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
if world > 1:
    dist.init_process_group("gloo")
    obj = [pb.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    rt = pb.Runtime(local, rank, world, obj[0])
else:
    rt = pb.Runtime(local, 0, 1)
nx = ny = a.nd
nz = a.nd * world
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
s.setup(n, starts, rp, ci, va, cfg=pb.SetupConfig(3, 40 * a.nd, 40, replicate_rows=a.replicate_rows))
del rp, ci, va
b = torch.ones(b1 - b0, dtype=torch.float64, device="cuda")
u = torch.zeros(b1 - b0, dtype=torch.float64, device="cuda")
sc = pb.SolveConfig(1e-30, a.iters, 1)  # exactly `iters` iterations
for _ in range(2):
    u.zero_()
    s.solve(b, u, solve_cfg=sc)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]):  # CUPTI start-up, untraced
    torch.ones(1, device="cuda").add_(1)
    torch.cuda.synchronize()
u.zero_()
torch.cuda.synchronize()
if world > 1:
    dist.barrier()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    if world > 1:
        dist.barrier()  # both ranks tracing before the first halo wait
    st = s.solve(b, u, solve_cfg=sc)
    torch.cuda.synchronize()
os.makedirs("gpurun_out/trace", exist_ok=True)
path = f"gpurun_out/trace/{a.tag}_r{rank}.trace.json"
prof.export_chrome_trace(path)
with open(path) as f:
    ev = [e for e in json.load(f)["traceEvents"] if e.get("cat") == "kernel"]
os.remove(path)
ev.sort(key=lambda e: e["ts"])
per = collections.defaultdict(list)
for e in ev:
    nm = e["name"].replace("void ", "").replace("(anonymous namespace)::", "").replace("pb::", "")
    depth, cut = 0, len(nm)
    for i, ch in enumerate(nm):  # drop the argument list, keep the template arguments
        depth += ch == "<"
        depth -= ch == ">"
        if ch == "(" and depth == 0:
            cut = i
            break
    nm = nm[:cut]
    g = e.get("args", {}).get("grid")
    e["short"] = nm + (f" grid={g[0]}" if g else "")
    per[e["short"]].append(float(e["dur"]))
busy, end, gaps = 0.0, None, []
for e in ev:  # union of kernel intervals (streams may overlap)
    t0, t1 = float(e["ts"]), float(e["ts"]) + float(e["dur"])
    if end is None or t0 > end:
        if end is not None:
            gaps.append(t0 - end)
        busy += t1 - t0
        end = t1
    elif t1 > end:
        busy += t1 - end
        end = t1
span = (end - float(ev[0]["ts"])) if ev else 0.0
out = {"rank": rank, "world": world, "stencil": a.stencil, "nd": a.nd, "iterations": st.iterations,
       "levels": s.level_sizes(), "span_us": span, "busy_us": busy, "idle_us": span - busy,
       "gaps_over_2us": sum(1 for g in gaps if g > 2.0), "gap_hist_us": {k: sum(1 for g in gaps if lo <= g < hi)
                                                                   for k, (lo, hi) in {"<1": (0, 1), "1-2": (1, 2), "2-5": (2, 5), "5-10": (5, 10), ">=10": (10, 1e18)}.items()},
       "kernels": {k: {"count": len(v), "mean_us": sum(v) / len(v), "total_us": sum(v)}
                   for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1]))},
       # the raw timeline (CUPTI host-clock timestamps: comparable across the ranks of one box)
       "timeline": [[e["short"], float(e["ts"]), float(e["dur"])] for e in ev]}
with open(f"gpurun_out/trace/{a.tag}_r{rank}.json", "w") as f:
    json.dump(out, f, indent=1)
if rank == 0:
    print(f"{a.tag}: iters {st.iterations} span {span:.0f} us busy {busy:.0f} idle {span - busy:.0f}")
s.close()
rt.close()
if world > 1:
    dist.destroy_process_group()
