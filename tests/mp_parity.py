"""Multi-rank parity program: every hierarchy array, SpMV, V-cycle and the
FCG solve of a row-block partitioned run, gathered from all ranks and compared
bit for bit with the oracle restatement at the SAME partition count
(total-order matching rule).  The solve must agree within +-1 iteration, meet
rtol, and do exactly one cross-rank reduction per FCG iteration.

Two launchers share ``rank_program`` / ``check_case``:
  * tests/test_local_ranks.py -- ranks are threads of one process on ONE GPU
    (pb.spawn_ranks, the LOCAL runtime; the reference's own spawn_ranks model);
  * tests/test_multigpu.py    -- ``python tests/mp_parity.py`` under torchrun,
    one process per GPU over NCCL + CUDA IPC.
Prints "MP_PARITY_OK <case>" per case on rank 0 (torchrun mode).
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_2303_02352_b200 as pb  # noqa: E402

CASES = [(7, 16, 16, 16), (7, 20, 17, 23), (27, 12, 12, 12), (7, 32, 32, 64), (7, 33, 33, 33)]


def bits(a):
    a = np.asarray(a)
    return a.view(np.int64) if a.dtype == np.float64 else a


def rank_program(rt, case, setup_overlap=False, replicate_rows=2500000):
    """One rank's share of a case: setup, exports, distributed SpMV / V-cycle
    on global probe vectors, one solve.  Returns a picklable dict."""
    st, nx, ny, nz = case
    world, rank = rt.nranks, rt.rank
    n = nx * ny * nz
    target = 40 * nx
    starts = pb.uniform_partition(n, world)
    b0, b1 = int(starts[rank]), int(starts[rank + 1])
    rp, ci, va = pb.poisson(st, nx, ny, nz, b0, b1)
    s = pb.Solver(rt)
    s.setup(n, starts, rp, ci, va, cfg=pb.SetupConfig(3, target, 40, setup_overlap=setup_overlap,
                                                     replicate_rows=replicate_rows))
    mine = {"levels": [s.level(k) for k in range(s.num_levels)],
            "P": [s.prolongator(k) for k in range(1, s.num_levels)],
            "M": [s.matching(t) for t in range(s.num_matchings)],
            "sizes": s.level_sizes(), "opc": s.opc, "stats": s.setup_stats()}
    vecs = {}
    for k in range(s.num_levels):
        li = s.level_info(k)
        xg = np.sin(0.37 * np.arange(li["global_rows"]))
        vecs[f"spmv{k}"] = s.spmv(k, xg[li["row_begin"]:li["row_begin"] + li["local_rows"]])
    rg = np.cos(0.11 * np.arange(n))
    vecs["vcycle"] = s.vcycle(rg[b0:b1])
    stt = s.solve(np.ones(b1 - b0))
    mine["vecs"] = vecs
    mine["solve"] = (stt.iterations, stt.final_relres, stt.converged, stt.history[:6], stt.reductions_per_iter,
                     stt.halo_exchanges_per_iter)
    s.close()
    return mine


def check_case(case, world, allp):
    """Compare the gathered per-rank results with the oracle at p = world."""
    st, nx, ny, nz = case
    n = nx * ny * nz
    target = 40 * nx
    o = oracle.Oracle("restatement", stencil=st, nx=nx, ny=ny, nz=nz, nranks=world,
                      coarse_size_target=target, matching_mode=1).setup()
    assert [tuple(x) for x in allp[0]["sizes"]] == [tuple(x) for x in o.level_sizes()], (allp[0]["sizes"],
                                                                                       o.level_sizes())
    assert allp[0]["opc"] == o.opc
    for r in range(world):  # decoupled aggregation: matching and R*C are communication-free (amg.cpp:203, 138)
        assert allp[r]["stats"]["matching_messages"] == 0 and allp[r]["stats"]["rc_messages"] == 0
    for k in range(o.num_levels):
        ref = o.level(k)
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
    it, rel, conv, hist, reductions, halos = allp[0]["solve"]
    assert conv and rel < 1e-6 and abs(it - ref["iterations"]) <= 1, (case, it, ref["iterations"])
    m = min(len(hist), len(ref["history"]))
    np.testing.assert_allclose(hist[:m], ref["history"][:m], rtol=1e-8)
    # one cross-rank reduction per FCG iteration
    assert all(allp[r]["solve"][4] == 1 for r in range(world)), [allp[r]["solve"][4] for r in range(world)]
    return it, ref["iterations"], o.num_levels


def main():  # torchrun launcher (one process per GPU, NCCL)
    import torch
    import torch.distributed as dist

    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    obj = [pb.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    rt = pb.Runtime(local, rank, world, obj[0])
    ov = os.environ.get("PAIRAMG_MP_SETUP_OVERLAP") == "1"
    for case in (CASES if len(sys.argv) < 2 else [tuple(int(x) for x in sys.argv[1:5])]):
        mine = rank_program(rt, case, setup_overlap=ov)
        allp = [None] * world
        dist.all_gather_object(allp, mine)
        if rank == 0:
            it, ref_it, nl = check_case(case, world, allp)
            print(f"MP_PARITY_OK {case} world={world} levels={nl} iters={it} (oracle {ref_it})", flush=True)
        dist.barrier()
    rt.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
