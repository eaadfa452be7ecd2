"""Command-line harness (SPEC bench_cli): configure, set up,
solve and report OPC, iterations, tsetup, tsolve, titer and the setup-time
breakdown, as the paper's protocol does.

    python -m paper_2303_02352_b200.cli -n 64 [-s 7|27] [-P p] [-p 0|1] [-c cfg] [--json]
    python -m paper_2303_02352_b200.cli -m matrix.mtx [-P p] ...

One process per GPU: with -P p > 1 the command re-launches itself under
torch.distributed.run (p ranks on 127.0.0.1) unless it already runs as one of
p ranks.  With --threads the p ranks are threads of this one process instead
(the reference's spawn_ranks; LOCAL runtime, all on cuda:0 -- a multi-rank
run on a single GPU).  -n generates the 7/27-point Poisson operator on the device (z-box
nd x nd x (nd*p) with --zbox, else the nd^3 cube split by Partition::uniform);
-m reads a MatrixMarket file and hands every rank its row block
(read_matrix_market + distribute_matrix).  b = 1, u0 = 0, w0 = 1.

Config file: one `key = value` per line, '#' comments; keys
aggregation_exponent, coarse_size, max_levels, pre_sweeps, post_sweeps,
coarsest_sweeps, relax_weight, max_iters, rtol, precflag.  Unknown keys and
out-of-range values are errors with the offending line.  Defaults are the
paper's section-5 values (s = 3, sweeps 4/4/20, rtol 1e-6, 1000 iterations,
coarse size 40*nd for generated problems, 40 for files).

Exit status 0 iff the solve converged (the report is printed either way).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import sys
import time

KEYS = {
    "aggregation_exponent": int, "coarse_size": int, "max_levels": int, "pre_sweeps": int, "post_sweeps": int,
    "coarsest_sweeps": int, "relax_weight": float, "max_iters": int, "rtol": float, "precflag": int,
}


class ConfigError(ValueError):
    pass


def parse_config(text: str, name: str = "<config>") -> dict:
    """`key = value` lines -> dict of the given keys (validated)."""
    out = {}
    for ln, raw in enumerate(text.splitlines(), 1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        if "=" not in line:
            raise ConfigError(f"{name}:{ln}: expected 'key = value', got '{raw.strip()}'")
        k, v = (t.strip() for t in line.split("=", 1))
        if k not in KEYS:
            raise ConfigError(f"{name}:{ln}: unknown key '{k}'")
        try:
            val = KEYS[k](v)
        except ValueError:
            raise ConfigError(f"{name}:{ln}: bad value '{v}' for {k}") from None
        if k == "rtol" and not 0.0 < val < 1.0:
            raise ConfigError(f"{name}:{ln}: rtol must be in (0, 1)")
        if k == "precflag" and val not in (0, 1):
            raise ConfigError(f"{name}:{ln}: precflag must be 0 or 1")
        if k in ("aggregation_exponent", "coarse_size", "max_levels", "max_iters") and val < 1:
            raise ConfigError(f"{name}:{ln}: {k} must be positive")
        if k in ("pre_sweeps", "post_sweeps", "coarsest_sweeps") and val < 0:
            raise ConfigError(f"{name}:{ln}: {k} must be >= 0")
        out[k] = val
    return out


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="paper_2303_02352_b200.cli", description=__doc__.split("\n\n")[0])
    src = ap.add_mutually_exclusive_group(required=True)
    src.add_argument("-n", dest="nd", type=int, help="Poisson generator: cube side nd")
    src.add_argument("-m", dest="matrix", help="MatrixMarket file")
    ap.add_argument("-s", dest="stencil", type=int, default=7, choices=(7, 27))
    ap.add_argument("--zbox", action="store_true", help="generator: nd x nd x (nd*p) (weak scaling)")
    ap.add_argument("-P", dest="ranks", type=int, default=1)
    ap.add_argument("--threads", action="store_true", help="-P ranks as threads of this process on cuda:0")
    ap.add_argument("-p", dest="precflag", type=int, choices=(0, 1), default=None)
    ap.add_argument("-c", dest="config")
    ap.add_argument("--json", action="store_true")
    a = ap.parse_args(argv)
    if a.ranks < 1:
        ap.error("-P must be >= 1")
    cfg = {}
    if a.config:
        with open(a.config) as f:
            try:
                cfg = parse_config(f.read(), a.config)
            except ConfigError as e:
                print(f"config error: {e}", file=sys.stderr)
                return 2
    if a.precflag is not None:
        cfg["precflag"] = a.precflag

    if a.threads:
        # every kernel loaded up front: ranks sharing a GPU (runtime.cu)
        os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
        os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
        return run_threads(a, cfg)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if a.ranks > 1 and world != a.ranks:
        if world != 1:
            print(f"-P {a.ranks} but launched as {world} ranks", file=sys.stderr)
            return 2
        argv_ = sys.argv[1:] if argv is None else list(argv)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.ranks}",
               "--master-addr=127.0.0.1", f"--master-port={_free_port()}", "-m", "paper_2303_02352_b200.cli", *argv_]
        os.execv(sys.executable, cmd)
    return run(a, cfg, world)


def run_threads(a, cfg: dict) -> int:
    import torch

    import paper_2303_02352_b200 as pb

    torch.cuda.set_device(0)
    out = pb.spawn_ranks(a.ranks, lambda rt: run_rank(a, cfg, rt, a.ranks, rt.rank, 0, lambda: None))
    return out[0]


def run(a, cfg: dict, world: int) -> int:
    import torch

    import paper_2303_02352_b200 as pb

    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    uid = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("gloo")
        obj = [pb.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    rt = pb.Runtime(local, rank, world, uid)

    def barrier():
        if world > 1:
            import torch.distributed as dist

            dist.barrier()

    rc = run_rank(a, cfg, rt, world, rank, local, barrier)
    rt.close()
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return rc


def run_rank(a, cfg: dict, rt, world: int, rank: int, local: int, barrier) -> int:
    """One rank's generate / read, setup, solve and report (rank 0 prints)."""
    import torch

    import paper_2303_02352_b200 as pb

    dev = torch.device("cuda", local)
    if a.nd is not None:
        nx = ny = a.nd
        nz = a.nd * world if a.zbox else a.nd
        n = nx * ny * nz
        starts = pb.uniform_partition(n, world)
        b0, b1 = int(starts[rank]), int(starts[rank + 1])
        nnz = pb.lib().pairamg_poisson_nnz(a.stencil, nx, ny, nz, b0, b1)
        rp = torch.empty(b1 - b0 + 1, dtype=torch.int64, device=dev)
        ci = torch.empty(nnz, dtype=torch.int64, device=dev)
        va = torch.empty(nnz, dtype=torch.float64, device=dev)
        pb._check(pb.lib().pairamg_poisson_device(rt.h, a.stencil, nx, ny, nz, b0, b1, pb._ptr(rp), pb._ptr(ci),
                                                   pb._ptr(va)))
        problem = {"kind": "poisson", "stencil": a.stencil, "grid": [nx, ny, nz]}
        coarse_default = 40 * a.nd
    else:
        n, ncols, *_ = pb.read_matrix_market(a.matrix, 0, 0)
        if ncols != n:
            raise pb.PairamgError(2, f"{a.matrix}: matrix is {n} x {ncols}, not square")
        starts = pb.uniform_partition(n, world)
        b0, b1 = int(starts[rank]), int(starts[rank + 1])
        _, _, hrp, hci, hva = pb.read_matrix_market(a.matrix, b0, b1)
        rp, ci, va = (torch.from_numpy(x).to(dev) for x in (hrp, hci, hva))
        problem = {"kind": "matrixmarket", "path": os.path.abspath(a.matrix)}
        coarse_default = 40
    setup_cfg = pb.SetupConfig(cfg.get("aggregation_exponent", 3), cfg.get("coarse_size", coarse_default),
                               cfg.get("max_levels", 40))
    cycle = pb.CycleConfig(cfg.get("pre_sweeps", 4), cfg.get("post_sweeps", 4), cfg.get("coarsest_sweeps", 20),
                           cfg.get("relax_weight", 1.0))
    solve_cfg = pb.SolveConfig(cfg.get("rtol", 1e-6), cfg.get("max_iters", 1000), cfg.get("precflag", 1))

    s = pb.Solver(rt)
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if solve_cfg.precflag:
        s.setup(n, starts, rp, ci, va, cfg=setup_cfg)
    else:
        s.setup(n, starts, rp, ci, va, cfg=pb.SetupConfig(setup_cfg.aggregation_exponent, max(n, 1), 1))
    torch.cuda.synchronize()
    tsetup = time.perf_counter() - t0
    b = torch.ones(b1 - b0, dtype=torch.float64, device=dev)
    u = torch.zeros(b1 - b0, dtype=torch.float64, device=dev)
    barrier()
    st = s.solve(b, u, cycle=cycle, solve_cfg=solve_cfg)
    ss = s.setup_stats()
    levels = [{"rows": r, "nnz": z} for r, z in s.level_sizes()]
    other = max(ss["t_total"] - ss["t_matching"] - ss["t_spmm"] - ss["t_spmm_comm"], 0.0)
    report = {
        "problem": problem, "n": int(n), "nnz": int(levels[0]["nnz"]),
        "ranks": world, "precflag": int(solve_cfg.precflag),
        "setup_config": {"aggregation_exponent": setup_cfg.aggregation_exponent,
                         "coarse_size": setup_cfg.coarse_size_target, "max_levels": setup_cfg.max_levels},
        "cycle": {"pre_sweeps": cycle.pre_sweeps, "post_sweeps": cycle.post_sweeps,
                  "coarsest_sweeps": cycle.coarsest_sweeps, "relax_weight": cycle.relax_weight},
        "rtol": solve_cfg.rtol, "max_iters": solve_cfg.max_iters,
        "levels": levels, "nl": len(levels), "opc": ss["opc"],
        "iterations": st.iterations, "final_relres": st.final_relres, "converged": bool(st.converged),
        "tsetup_s": tsetup, "tsolve_s": st.t_solve_s,
        "titer_s": st.t_solve_s / st.iterations if st.iterations else None,
        "setup_breakdown_s": {"matching": ss["t_matching"], "spmm": ss["t_spmm"], "spmm_comm": ss["t_spmm_comm"],
                              "other": other},
        "messages": {"matching": ss["matching_messages"], "rc": ss["rc_messages"]},
    }
    if rank == 0:
        if a.json:
            print(json.dumps(report))
        else:
            print(f"problem      {problem}")
            print(f"ranks        {world}   precflag {report['precflag']}")
            for k, lv in enumerate(levels):
                print(f"level {k:2d}     rows {lv['rows']:>12d}   nnz {lv['nnz']:>14d}")
            print(f"opc          {ss['opc']:.4f}   levels {len(levels)}")
            print(f"iterations   {st.iterations}   relres {st.final_relres:.3e}   converged {bool(st.converged)}")
            print(f"tsetup       {tsetup:.4f} s  (matching {ss['t_matching']:.4f}, spmm {ss['t_spmm']:.4f}, "
                  f"spmm_comm {ss['t_spmm_comm']:.4f}, other {other:.4f})")
            ti = report["titer_s"]
            print(f"tsolve       {st.t_solve_s:.4f} s   titer {ti * 1e3 if ti else float('nan'):.3f} ms")
    s.close()
    return 0 if st.converged else 1


if __name__ == "__main__":
    sys.exit(main())
