"""Small workload for compute-sanitizer (scripts/sanitize.sh): setup + V-cycle
+ solve of 7- and 27-point problems on one rank, the matching KAT kernels on a
tie-heavy graph, a replayed setup, and a two-rank LOCAL run (P2P halo flags,
dot allgather, replicated-rhs gather) -- every kernel family of the library."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_02352_b200 as pb  # noqa: E402


def one_rank(rt):
    for st, nd in ((7, 12), (27, 9)):
        rp, ci, va = pb.poisson(st, nd, nd, nd)
        n = len(rp) - 1
        s = pb.Solver(rt)
        s.setup(n, [0, n], rp, ci, va, cfg=pb.SetupConfig(3, 40, 40))
        s.vcycle(np.ones(n))
        s.spmv(0, np.ones(n))
        st_ = s.solve(np.ones(n))
        assert st_.converged
        trace = [s.matching(t) for t in range(s.num_matchings)]
        s.setup(n, [0, n], rp, ci, va, cfg=pb.SetupConfig(3, 40, 40, replay=trace))
        s.close()
    # Suitor on a graph where every weight ties (the 128-bit CAS path)
    rp, ci, _ = pb.poisson(7, 10, 10, 10)
    keep = ci != np.repeat(np.arange(len(rp) - 1), np.diff(rp))
    rows = np.repeat(np.arange(len(rp) - 1), np.diff(rp))[keep]
    grp = np.concatenate([[0], np.cumsum(np.bincount(rows, minlength=len(rp) - 1))])
    pb.match_graph(rt, grp, ci[keep], np.ones(int(keep.sum())))


def two_ranks():
    def prog(rt):
        nx, ny, nz = 10, 9, 12
        n = nx * ny * nz
        starts = pb.uniform_partition(n, 2)
        b0, b1 = int(starts[rt.rank]), int(starts[rt.rank + 1])
        rp, ci, va = pb.poisson(7, nx, ny, nz, b0, b1)
        s = pb.Solver(rt)
        s.setup(n, starts, rp, ci, va, cfg=pb.SetupConfig(3, 40, 40, replicate_rows=100))
        out = s.solve(np.ones(b1 - b0))
        s.close()
        return out.converged

    assert all(pb.spawn_ranks(2, prog))


if __name__ == "__main__":
    os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
    rt = pb.Runtime(0, 0, 1)
    one_rank(rt)
    rt.close()
    if "--no-ranks" not in sys.argv:
        two_ranks()
    print("sanitize_run ok")
