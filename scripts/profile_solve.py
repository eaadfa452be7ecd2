"""Profiling driver: build the hierarchy, warm up, then run ONE solve of
`--iters` FCG iterations between cudaProfilerStart/Stop (use ncu
--profile-from-start off).  Same kernels as bench.py's timed step."""
import argparse
import sys

import torch

sys.path.insert(0, ".")
import paper_2303_02352_b200 as pb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--stencil", type=int, default=7)
ap.add_argument("--nd", type=int, default=256)
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--problem", default="poisson", choices=["poisson", "varcoef"])
ap.add_argument("--levels", type=int, default=2)
ap.add_argument("--format", default="auto")
a = ap.parse_args()
nd = a.nd
n = nd ** 3
rt = pb.Runtime(0, 0, 1)
L = pb.lib()
nnz = L.pairamg_poisson_nnz(a.stencil, nd, nd, nd, 0, n)
rp = torch.empty(n + 1, dtype=torch.int64, device="cuda")
ci = torch.empty(nnz, dtype=torch.int64, device="cuda")
va = torch.empty(nnz, dtype=torch.float64, device="cuda")
if a.problem == "poisson":
    pb._check(L.pairamg_poisson_device(rt.h, a.stencil, nd, nd, nd, 0, n, pb._ptr(rp), pb._ptr(ci), pb._ptr(va)))
else:
    pb._check(L.pairamg_varcoef_device(rt.h, a.stencil, nd, nd, nd, a.levels, 1, 0, n, pb._ptr(rp), pb._ptr(ci),
                                       pb._ptr(va)))
s = pb.Solver(rt)
target = 40 * nd if a.problem == "poisson" else 200 * nd  # as bench.py
s.setup(n, [0, n], rp, ci, va, cfg=pb.SetupConfig(3, target, 40, storage=a.format))
b = torch.ones(n, dtype=torch.float64, device="cuda")
u = torch.zeros(n, dtype=torch.float64, device="cuda")
sc = pb.SolveConfig(1e-6, a.iters, 1)
s.solve(b, u, solve_cfg=sc)
u.zero_()
torch.cuda.synchronize()
torch.cuda.profiler.start()
st = s.solve(b, u, solve_cfg=sc)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(f"profiled solve: {st.iterations} iterations, levels {s.level_sizes()}")
