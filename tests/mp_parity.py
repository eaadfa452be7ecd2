"""Multi-rank parity program (launched by tests/test_multigpu.py under torchrun).

Each rank owns a row block of the fine system on its own GPU (NCCL halo
exchange / collectives inside libpairamg_b200.so); the owned pieces of every
hierarchy array are gathered to rank 0 and compared bit for bit with the
oracle restatement run at the SAME partition count (total-order matching
rule).  The solve must agree within +-1 iteration and meet rtol.
Prints "MP_PARITY_OK <case>" per case on rank 0.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_2303_02352_b200 as pb  # noqa: E402

CASES = [(7, 16, 16, 16), (7, 20, 17, 23), (27, 12, 12, 12), (7, 32, 32, 64), (7, 33, 33, 33)]


def bits(a):
    a = np.asarray(a)
    return a.view(np.int64) if a.dtype == np.float64 else a


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    obj = [pb.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    rt = pb.Runtime(local, rank, world, obj[0])
    for case in (CASES if len(sys.argv) < 2 else [tuple(int(x) for x in sys.argv[1:5])]):
        st, nx, ny, nz = case
        n = nx * ny * nz
        target = 40 * nx
        starts = pb.uniform_partition(n, world)
        b0, b1 = int(starts[rank]), int(starts[rank + 1])
        rp, ci, va = pb.poisson(st, nx, ny, nz, b0, b1)
        s = pb.Solver(rt)
        s.setup(n, starts, rp, ci, va, cfg=pb.SetupConfig(3, target, 40, setup_overlap=os.environ.get(
            "PAIRAMG_MP_SETUP_OVERLAP") == "1"))
        mine = {"levels": [s.level(k) for k in range(s.num_levels)],
                "P": [s.prolongator(k) for k in range(1, s.num_levels)],
                "M": [s.matching(t) for t in range(s.num_matchings)],
                "sizes": s.level_sizes(), "opc": s.opc}
        # distributed SpMV / V-cycle on a global probe vector
        vecs = {}
        for k in range(s.num_levels):
            li = s.level_info(k)
            xg = np.sin(0.37 * np.arange(li["global_rows"]))
            vecs[f"spmv{k}"] = s.spmv(k, xg[li["row_begin"]:li["row_begin"] + li["local_rows"]])
        rg = np.cos(0.11 * np.arange(n))
        vecs["vcycle"] = s.vcycle(rg[b0:b1])
        stt = s.solve(np.ones(b1 - b0))
        mine["vecs"] = vecs
        mine["solve"] = (stt.iterations, stt.final_relres, stt.converged, stt.history[:6])
        allp = [None] * world
        dist.all_gather_object(allp, mine)
        s.close()
        if rank == 0:
            o = oracle.Oracle("restatement", stencil=st, nx=nx, ny=ny, nz=nz, nranks=world,
                              coarse_size_target=target, matching_mode=1).setup()
            assert [tuple(x) for x in allp[0]["sizes"]] == [tuple(x) for x in o.level_sizes()], (allp[0]["sizes"], o.level_sizes())
            assert allp[0]["opc"] == o.opc
            for k in range(o.num_levels):
                ref = o.level(k)
                # concatenate owned row blocks
                rp_all = [allp[0]["levels"][k][0]]
                off = allp[0]["levels"][k][0][-1]
                for r in range(1, world):
                    rp_all.append(allp[r]["levels"][k][0][1:] + off)
                    off += allp[r]["levels"][k][0][-1]
                got = [np.concatenate(rp_all)] + [np.concatenate([allp[r]["levels"][k][i] for r in range(world)])
                                                  for i in range(1, 5)]
                for name, x, y in zip(["row_ptr", "col", "val", "w", "l1"], got, ref):
                    assert np.array_equal(bits(x), bits(y)), f"{case} level {k} {name}"
                y = o.spmv(k, np.sin(0.37 * np.arange(o.level_size(k)[0])))
                g = np.concatenate([allp[r]["vecs"][f"spmv{k}"] for r in range(world)])
                assert np.array_equal(bits(g), bits(y)), f"{case} spmv level {k}"
            for k in range(1, o.num_levels):
                oc, ov = o.prolongator(k)
                gc = np.concatenate([allp[r]["P"][k - 1][0] for r in range(world)])
                gv = np.concatenate([allp[r]["P"][k - 1][1] for r in range(world)])
                assert np.array_equal(gc, oc) and np.array_equal(bits(gv), bits(ov)), f"{case} P{k}"
            for t in range(o.num_matchings):
                gm = np.concatenate([allp[r]["M"][t] for r in range(world)])
                assert np.array_equal(gm, o.matching(t)), f"{case} matching {t}"
            g = np.concatenate([allp[r]["vecs"]["vcycle"] for r in range(world)])
            assert np.array_equal(bits(g), bits(o.vcycle(np.cos(0.11 * np.arange(n))))), f"{case} vcycle"
            ref = o.solve()
            it, rel, conv, hist = allp[0]["solve"]
            assert conv and rel < 1e-6 and abs(it - ref["iterations"]) <= 1, (case, it, ref["iterations"])
            m = min(len(hist), len(ref["history"]))
            np.testing.assert_allclose(hist[:m], ref["history"][:m], rtol=1e-8)
            print(f"MP_PARITY_OK {case} world={world} levels={o.num_levels} iters={it} (oracle {ref['iterations']})",
                  flush=True)
        dist.barrier()
    rt.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
