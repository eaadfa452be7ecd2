"""Strong-scaling config (configs[3], 7-point 585^3 = 200 M unknowns) at
p = 4 and 8 ranks as threads sharing ONE B200 (LOCAL runtime): the FCG
iteration count must match the reference's own count at the same partition
(tests/golden/ref_counts.json, oracle/_ref on the GPU box's host) within +-1.
Run as its own process by tests/test_local_ranks.py (a fresh memory pool:
the hierarchy of 200 M unknowns takes ~100 GB).  Prints one JSON line."""
import json
import os
import sys

os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2303_02352_b200 as pb  # noqa: E402


def main():
    nd = int(sys.argv[1]) if len(sys.argv) > 1 else 585
    ps = [int(x) for x in sys.argv[2:]] or [4, 8]
    n = nd ** 3
    L = pb.lib()
    out = {}
    for p in ps:
        starts = pb.uniform_partition(n, p)

        def prog(rt):
            b0, b1 = int(starts[rt.rank]), int(starts[rt.rank + 1])
            nnz = L.pairamg_poisson_nnz(7, nd, nd, nd, b0, b1)
            rp = torch.empty(b1 - b0 + 1, dtype=torch.int64, device="cuda")
            ci = torch.empty(nnz, dtype=torch.int64, device="cuda")
            va = torch.empty(nnz, dtype=torch.float64, device="cuda")
            pb._check(L.pairamg_poisson_device(rt.h, 7, nd, nd, nd, b0, b1, pb._ptr(rp), pb._ptr(ci), pb._ptr(va)))
            # every torch allocation BEFORE the setup: once a peer rank spins on
            # this rank's first halo push, a device-synchronising call here (torch's
            # allocator releasing cached blocks under memory pressure -> cudaFree)
            # would wait for that spin
            b = torch.ones(b1 - b0, dtype=torch.float64, device="cuda")
            u = torch.zeros(b1 - b0, dtype=torch.float64, device="cuda")
            s = pb.Solver(rt)
            s.setup(n, starts, rp, ci, va, cfg=pb.SetupConfig(3, 40 * nd, 40))
            st = s.solve(b, u)
            res = {"iterations": st.iterations, "relres": st.final_relres, "levels": s.level_sizes(),
                   "reductions_per_iter": st.reductions_per_iter, "t_solve_s": st.t_solve_s}
            s.close()
            return res

        torch.cuda.set_device(0)
        r = pb.spawn_ranks(p, prog)
        out[str(p)] = r[0]
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
