"""Profiling driver: set up one Poisson level-0 operator, then one SpMV at
level 0 and one V-cycle (so `ncu -k regex:<kernel> --launch-count k` sees the
level-0 launches first).  Development aid.

    python scripts/prof_one.py [stencil] [nd]
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2303_02352_b200 as pb  # noqa: E402

stencil = int(sys.argv[1]) if len(sys.argv) > 1 else 7
nd = int(sys.argv[2]) if len(sys.argv) > 2 else 256
n = nd ** 3
rt = pb.Runtime(0, 0, 1)
nnz = pb.lib().pairamg_poisson_nnz(stencil, nd, nd, nd, 0, n)
rp = torch.empty(n + 1, dtype=torch.int64, device="cuda")
ci = torch.empty(nnz, dtype=torch.int64, device="cuda")
va = torch.empty(nnz, dtype=torch.float64, device="cuda")
pb._check(pb.lib().pairamg_poisson_device(rt.h, stencil, nd, nd, nd, 0, n, pb._ptr(rp), pb._ptr(ci), pb._ptr(va)))
s = pb.Solver(rt)
s.setup(n, [0, n], rp, ci, va, cfg=pb.SetupConfig(3, 40 * nd, 40))
x = np.random.default_rng(0).standard_normal(n)
y = s.spmv(0, x)
z = s.vcycle(x)
torch.cuda.synchronize()
print("ok", float(np.abs(y).sum()), float(np.abs(z).sum()))
s.close()
rt.close()
