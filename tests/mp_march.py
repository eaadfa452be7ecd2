"""Multi-GPU program (torchrun, one process per GPU): the 27-point split launch
whose interior blocks are marching tiles (k_sten_march_split[_dots]).

192 x 192 x 384 is slab-aligned at 2 and 4 ranks, so the distributed
hierarchy is the one-rank hierarchy: rank 0 first runs the case alone on its
GPU, then every rank runs its row block and the level SpMVs, the V-cycle
(every level's pre/post sweeps and residual go through the split launch
where the level has halos) and the solve are compared with the one-rank run
bit for bit (the solve's history to the dot-product rounding, whose block
order differs).  Prints "MP_MARCH_OK" on rank 0.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2303_02352_b200 as pb  # noqa: E402

NX, NY, NZ = 192, 192, 384


def bits(a):
    a = np.asarray(a)
    return a.view(np.int64) if a.dtype == np.float64 else a


def run(rt, world):
    import torch

    n = NX * NY * NZ
    L = pb.lib()
    starts = pb.uniform_partition(n, world)
    b0, b1 = int(starts[rt.rank]), int(starts[rt.rank + 1])
    nnz = L.pairamg_poisson_nnz(27, NX, NY, NZ, b0, b1)
    rp = torch.empty(b1 - b0 + 1, dtype=torch.int64, device="cuda")
    ci = torch.empty(nnz, dtype=torch.int64, device="cuda")
    va = torch.empty(nnz, dtype=torch.float64, device="cuda")
    pb._check(L.pairamg_poisson_device(rt.h, 27, NX, NY, NZ, b0, b1, pb._ptr(rp), pb._ptr(ci), pb._ptr(va)))
    s = pb.Solver(rt)
    s.setup(n, starts, rp, ci, va, cfg=pb.SetupConfig(3, 40 * NX, 40))
    del rp, ci, va
    out = {"spmv": []}
    for k in range(s.num_levels):
        li = s.level_info(k)
        xg = np.sin(0.37 * np.arange(li["global_rows"]))
        out["spmv"].append(s.spmv(k, xg[li["row_begin"]:li["row_begin"] + li["local_rows"]]))
    out["vcycle"] = s.vcycle(np.cos(0.11 * np.arange(b0, b1)))
    st = s.solve(np.ones(b1 - b0))
    out["iters"], out["hist"], out["conv"] = st.iterations, list(st.history), st.converged
    s.close()
    return out


def main():
    import torch
    import torch.distributed as dist

    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    one = None
    if rank == 0:
        rt1 = pb.Runtime(local, 0, 1)
        one = run(rt1, 1)
        rt1.close()
    dist.barrier()
    obj = [pb.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    rt = pb.Runtime(local, rank, world, obj[0])
    mine = run(rt, world)
    allp = [None] * world
    dist.all_gather_object(allp, mine)
    if rank == 0:
        for k in range(len(one["spmv"])):
            got = np.concatenate([allp[r]["spmv"][k] for r in range(world)])
            assert np.array_equal(bits(got), bits(one["spmv"][k])), f"spmv level {k}"
        got = np.concatenate([allp[r]["vcycle"] for r in range(world)])
        assert np.array_equal(bits(got), bits(one["vcycle"])), "vcycle"
        assert allp[0]["conv"] and abs(allp[0]["iters"] - one["iters"]) <= 1, (allp[0]["iters"], one["iters"])
        m = min(len(allp[0]["hist"]), len(one["hist"]))
        np.testing.assert_allclose(allp[0]["hist"][:m], one["hist"][:m], rtol=1e-8)
        print(f"MP_MARCH_OK world={world} levels={len(one['spmv'])} iters={allp[0]['iters']} (one rank {one['iters']})",
              flush=True)
    dist.barrier()
    rt.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
