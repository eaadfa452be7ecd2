#!/usr/bin/env python3
"""AMG-FCG solve benchmark (BASELINE.json metric) -- one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--stencil 7|27] [--nd 256] [--scaling weak|strong]
                    [--problem poisson|varcoef] [--levels L] [--format auto|sten|pat|dict|coded|plain]

A step is one complete flexible-CG solve to rtol 1e-6 (u0 = 0, b = 1) with the
AMG V-cycle preconditioner, hierarchy already built (setup is timed
separately and reported as setup_s).
  N = 1   : configs[1], 7-point 256^3 (16.8M unknowns) on one B200.
  N > 1   : weak scaling (configs[2]): z-box 256 x 256 x 256N, each rank owns
            one 256^3 slab (row-block partition); --scaling strong runs
            --nd^3 split across the N ranks instead (configs[3] is 585^3).
  --gpus N without a launcher re-executes itself under torch.distributed.run
  (N ranks, 127.0.0.1), as the reference's harness spawns its ranks
  (spawn_ranks, runtime.hpp:113-136); under a launcher WORLD_SIZE must be N.
  --problem varcoef: the variable-coefficient operator of the same sparsity
  (pairamg_varcoef_device; --levels 2 gives a few distinct values, 0 all
  distinct) -- the workload of the general storage formats, --format forces one.
value = solve seconds (device CUDA events on the solver stream, max over
ranks); e2e = the same solve through the C ABI with pinned host buffers
(pairamg_solve: H2D of b and u0, solve, D2H of u inside the timed region;
the copies are also timed apart by events inside the call).
--impl reference times the reference's own compiled CPU code
(oracle/_ref/libpairamg_ref.so: the reference's seven C++ units + the
restated FCG driver) on the host cores, same config and metric; the GPU
arm's cpu_baseline is that arm run in a subprocess.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "AMG-FCG solve s & ms/iter to rtol 1e-6 at 1/2/4/8 B200; SpMV GB/s vs HBM"
UNIT = "s"


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(kernel_key: str, workload: str, n_gpus: int):
    """DRAM bytes per launch of the dominant kernel from the committed ncu --set
    full summary, only when it was captured on this workload (1 GPU)."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            d = json.load(f).get(kernel_key, {})
        if n_gpus != 1 or d.get("workload") != workload:
            return None
        return d.get("dram_bytes_per_launch")
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm.sort()
        busy = [x for x in sm if x > 0.5 * mx] or sm
        return {"sm_mhz": busy[len(busy) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def problem_dims(args, world: int):
    """Grid and coarse-size target: 40*nd as the paper for
    Poisson; 200*nd for varcoef, whose pairwise coarsening stalls near 3*10^4
    rows at 256^3 (the reference's own setup stagnates below that, with an
    empty matching, scripts notes in DESIGN.md 6)."""
    nd = getattr(args, "nd", 0)
    target = 40 * nd if getattr(args, "problem", "poisson") == "poisson" else 200 * nd
    if world > 1 and args.scaling == "weak":
        return nd, nd, nd * world, target
    return nd, nd, nd, target


def slab(n: int, world: int, rank: int):
    """Row-block partition (Partition::uniform) and this rank's block."""
    import paper_2303_02352_b200 as pb

    starts = pb.uniform_partition(n, world)
    return starts, int(starts[rank]), int(starts[rank + 1])


def workload_name(args, world):
    nx, ny, nz, _ = problem_dims(args, world)
    base = f"poisson{args.stencil}" if args.problem == "poisson" else f"varcoef{args.stencil}L{args.levels}"
    fmt = "" if args.format == "auto" else f"_{args.format}"
    return f"{base}_{nx}x{ny}x{nz}" + (f"_{args.scaling}" if world > 1 else "") + fmt


def config_dict(args, world):
    nx, ny, nz, target = problem_dims(args, world)
    part = "dp1" if world == 1 else f"rowblock{world}"
    return {
        "workload": workload_name(args, world),
        "unknowns": nx * ny * nz, "stencil": args.stencil, "problem": args.problem,
        "storage": args.format, "coarse_size_target": target, "aggregation_exponent": 3,
        "replicate_rows": args.replicate_rows if world > 1 else None,
        "sweeps": "4/4/20 l1-Jacobi", "rtol": 1e-6, "parallelism": part,
        "step": "one full FCG solve to rtol (hierarchy prebuilt)",
        "l2": "working set larger than L2 (no flush): every level-0 vector is 8*unknowns bytes (134 MB at 256^3 "
              "vs 126 MB L2) and one FCG iteration streams several GB",
    }


# ----------------------------------------------------------------------------- CPU reference


def ref_counts():
    """Reference iteration counts of configs too large to solve inside the
    bench budget (tests/golden/ref_counts.json, made by scripts/ref_counts.py
    on the GPU box's host from oracle/_ref), keyed (stencil, nx, ny, nz, p)."""
    out = {(7, 64, 64, 64, 1): 19, (7, 128, 128, 128, 1): 25, (7, 256, 256, 256, 1): 42,
           (27, 192, 192, 192, 1): 32}
    p = os.path.join(ROOT, "tests", "golden", "ref_counts.json")
    if os.path.exists(p):
        with open(p) as f:
            for r in json.load(f).get("runs", []):
                if "iterations" in r:
                    out[(r["stencil"], *r["grid"], r["p"])] = r["iterations"]
    return out


def host_threads(n_slabs: int) -> int:
    """Largest power of two <= host cores that divides the slab count (slab-aligned partition)."""
    cores = os.cpu_count() or 1
    p = 1
    while p * 2 <= min(cores, 64) and n_slabs % (p * 2) == 0:
        p *= 2
    return p


def bench_reference(args, world):
    """The reference's own compiled CPU implementation on all usable host threads,
    same config and metric.  A step = a bounded sample of the solve (the first
    --ref-sample-iters FCG iterations); value = measured ms/iteration x the
    reference's own iteration count for the full solve (one full solve when it
    fits --ref-full-budget-s, else the committed count of tests/golden)."""
    import numpy as np

    import oracle

    nx, ny, nz, target = problem_dims(args, world)
    # partition = the GPU run's row blocks when N > 1 (decoupled aggregation
    # depends on it), else host threads (slab-aligned: same hierarchy as p=1)
    p = world if world > 1 else host_threads(nz)
    t0 = time.time()
    if args.problem == "poisson":
        o = oracle.Oracle("reference", stencil=args.stencil, nx=nx, ny=ny, nz=nz, nranks=p, coarse_size_target=target)
    else:
        import paper_2303_02352_b200 as pb

        rp, ci, va = pb.varcoef(args.stencil, nx, ny, nz, args.levels, args.seed)
        o = oracle.Oracle("reference", csr=(rp, ci, va), nranks=p, coarse_size_target=target)
    t_gen = time.time() - t0
    t0 = time.time()
    o.setup()
    setup_s = time.time() - t0
    o.set_solve(1e-6, 1)
    r = o.solve()
    ms_iter0 = 1e3 * r["t_solve"] / max(r["iterations"], 1)
    # iterations per step: up to --ref-sample-iters, a step of at most ~3 s
    k = max(1, min(args.ref_sample_iters, int(3000.0 / max(ms_iter0, 1e-3))))
    o.set_solve(1e-6, k)
    iters_full, full_s, full_rel = None, None, None
    if ms_iter0 * 1e-3 * 60 < args.ref_full_budget_s:
        o.set_solve(1e-6, 1000)
        rf = o.solve()
        iters_full, full_s, full_rel = rf["iterations"], rf["t_solve"], rf["relres"]
        o.set_solve(1e-6, k)
    elif args.problem == "poisson":
        iters_full = ref_counts().get((args.stencil, nx, ny, nz, p if world > 1 else 1))
    for _ in range(max(0, args.warmup - 1)):
        o.solve()
    step_ms, per_iter = [], []
    for _ in range(args.steps):
        r = o.solve()
        step_ms.append(1e3 * r["t_solve"])
        per_iter.append(1e3 * r["t_solve"] / max(r["iterations"], 1))
    ms_iter = float(np.mean(per_iter))
    value = ms_iter * 1e-3 * iters_full if iters_full else None
    how = (f"measured by one full reference solve ({full_s:.1f}s, relres {full_rel:.3e})" if full_s is not None
           else "the reference's count committed in tests/golden/ref_counts.json (scripts/ref_counts.py)")
    sample = (f"{config_dict(args, world)['workload']}; reference C++ (oracle/_ref, unmodified units + restated "
              f"FCG), {p} ranks = {p} host threads; setup {setup_s:.1f}s once; each step = the first {k} FCG "
              f"iterations; value = measured ms/iter x {iters_full} iterations ({how})")
    return {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": float(np.mean(step_ms)), "higher_is_better": False,
        "scaling": args.scaling if world > 1 else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args, world),
        "step": f"{k} FCG iterations of the reference solve (bounded sample; value extrapolates to the full solve)",
        "ms_per_iter": ms_iter, "iterations": iters_full, "full_solve_s": full_s, "setup_s": setup_s,
        "gen_s": t_gen,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": p, "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def cpu_baseline_subprocess(args):
    """The reference arm in its own process (the GPU process never loads oracle/)."""
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "1", "--steps", "2",
           "--warmup", "3", "--stencil", str(args.stencil), "--nd", str(args.nd), "--problem", args.problem,
           "--levels", str(args.levels), "--seed", str(args.seed), "--ref-sample-iters", str(args.ref_sample_iters),
           "--ref-full-budget-s", str(args.ref_full_budget_s)]
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
        line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
        d = json.loads(line)
        cb = d["cpu_baseline"]
        cb.update({"setup_s": d["setup_s"], "ms_per_iter": d["ms_per_iter"], "iterations": d["iterations"]})
        return cb
    except Exception as ex:  # reported, not fatal
        return {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"failed: {ex}"}


# ----------------------------------------------------------------------------- ours


def bench_ours(args, rank, world, local_rank):
    import numpy as np
    import torch

    import paper_2303_02352_b200 as pb

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    uid = None
    if world > 1:
        import torch.distributed as dist

        obj = [pb.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    rt = pb.Runtime(local_rank, rank, world, uid)
    nx, ny, nz, target = problem_dims(args, world)
    n = nx * ny * nz
    starts, b0, b1 = slab(n, world, rank)
    m = b1 - b0
    L = pb.lib()
    nnz = L.pairamg_poisson_nnz(args.stencil, nx, ny, nz, b0, b1)
    rp = torch.empty(m + 1, dtype=torch.int64, device=dev)
    ci = torch.empty(nnz, dtype=torch.int64, device=dev)
    va = torch.empty(nnz, dtype=torch.float64, device=dev)
    if args.problem == "poisson":
        pb._check(L.pairamg_poisson_device(rt.h, args.stencil, nx, ny, nz, b0, b1, pb._ptr(rp), pb._ptr(ci),
                                           pb._ptr(va)))
    else:
        pb._check(L.pairamg_varcoef_device(rt.h, args.stencil, nx, ny, nz, args.levels, args.seed, b0, b1,
                                           pb._ptr(rp), pb._ptr(ci), pb._ptr(va)))
    s = pb.Solver(rt)
    cfg = pb.SetupConfig(3, target, 40, storage=args.format, replicate_rows=args.replicate_rows)

    def barrier():
        if world > 1:
            import torch.distributed as dist

            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        import torch.distributed as dist

        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x: float) -> float:
        if world == 1:
            return x
        import torch.distributed as dist

        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    # setup (timed: device-resident inputs, includes validation + the whole hierarchy)
    setup_times = []
    for _ in range(2):
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s.setup(n, starts, rp, ci, va, cfg=cfg)
        torch.cuda.synchronize()
        setup_times.append(max_over_ranks(time.perf_counter() - t0))
    sstats = s.setup_stats()
    b = torch.ones(m, dtype=torch.float64, device=dev)
    u = torch.zeros(m, dtype=torch.float64, device=dev)
    stream = torch.cuda.ExternalStream(s.stream(), device=dev)
    for _ in range(args.warmup):
        u.zero_()
        st = s.solve(b, u)
    # timed region: K full solves, CUDA events on the solver stream
    times, iters, launches = [], [], 0
    with ClockSampler(local_rank) as clk:
        for _ in range(args.steps):
            u.zero_()
            barrier()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            st = s.solve(b, u)
            e1.record(stream)
            e1.synchronize()
            torch.cuda.synchronize()
            times.append(max_over_ranks(e0.elapsed_time(e1) * 1e-3))
            iters.append(st.iterations)
            launches += s.launch_count()
    clocks = clk.summary()
    t_solve = sum(times) / len(times)
    it = iters[-1]
    # instrumented step: per-launch CUDA events around every level-0 kernel
    s.set_kernel_timing(True)
    u.zero_()
    s.solve(b, u)
    s.set_kernel_timing(False)
    kt = [s.kernel_timing(k) for k in range(4)]
    # per-level V-cycle time per iteration (class 4 + k: entry to restriction + return to exit)
    level_us = [1e3 * s.kernel_timing(4 + k)["ms"] / max(1, it) for k in range(min(s.num_levels, 16))]
    peak, peak_src = measured_peaks()
    li0 = s.level_info(0)
    fmt0 = s.level_storage(0)
    sweep_kernel = {"sten": ("k_sten_march<kJacobi> (27-point STEN, 2.5-D tiles: each x-plane once into shared "
                             "memory by cp.async, streaming row sums)" if args.stencil == 27 else
                             "k_sten2<kJacobi> (STEN: one pattern byte per row, uniform offsets/values, two rows "
                             "per thread)"),
                    "pat": "k_pat<kJacobi> (PAT: one pattern byte per row)",
                    "dict": "k_sell<kJacobi> (DICT: one code byte per entry)",
                    "coded": "k_sell<kJacobi> (CODED SELL-32: one 32-bit column-delta/value-code word per entry)",
                    "plain": "k_sell<kJacobi> (PLAIN SELL-32: int32 column + f64 value per entry)"}[fmt0]
    csr_bytes = 12.0 * li0["local_nnz"] + 36.0 * li0["local_rows"]  # SURVEY 8d model: f64 values + int32 columns
    sweep = kt[0]
    sweep_ms = sweep["ms"] / max(sweep["launches"], 1)
    sweep_gbs = sweep["bytes_per_launch"] / (sweep_ms * 1e-3) / 1e9 if sweep["launches"] else None
    spmv = kt[2]
    spmv_ms = spmv["ms"] / max(spmv["launches"], 1)
    spmv_gbs = spmv["bytes_per_launch"] / (spmv_ms * 1e-3) / 1e9 if spmv["launches"] else None
    # e2e: the same solve through the C ABI with pinned host buffers; the
    # library times the copies apart (events inside pairamg_solve)
    hb = torch.ones(m, dtype=torch.float64).pin_memory()
    hu = torch.zeros(m, dtype=torch.float64).pin_memory()
    hb_np, hu_np = hb.numpy(), hu.numpy()
    e2e_times, h2d, d2h, dev_s = [], [], [], []
    for k in range(max(2, min(args.steps, 3)) + 1):
        hu_np[:] = 0.0
        barrier()
        t0 = time.perf_counter()
        st_e = s.solve(hb_np, hu_np)
        dt = max_over_ranks(time.perf_counter() - t0)
        if k > 0:
            e2e_times.append(dt)
            h2d.append(st_e.t_h2d_s)
            d2h.append(st_e.t_d2h_s)
            dev_s.append(st_e.t_solve_s)
    e2e = sum(e2e_times) / len(e2e_times)
    h2d_s, d2h_s, e2e_dev = (sum(x) / len(x) for x in (h2d, d2h, dev_s))
    # full pipeline once: host CSR -> setup -> solve -> host u
    pipe = None
    if args.pipeline and args.problem == "poisson":
        hrp, hci, hva = pb.poisson(args.stencil, nx, ny, nz, b0, b1)
        barrier()
        t0 = time.perf_counter()
        s2 = pb.Solver(rt)
        s2.setup(n, starts, hrp, hci, hva, cfg=cfg)
        hu_np[:] = 0.0
        s2.solve(hb_np, hu_np)
        pipe = max_over_ranks(time.perf_counter() - t0)
        s2.close()
    comm = None
    if world > 1:
        ms_iter = t_solve * 1e3 / it
        halo_all = sum_over_ranks(st.halo_bytes_per_iter)
        comm = {"reductions_per_iter": st.reductions_per_iter, "halo_exchanges_per_iter": st.halo_exchanges_per_iter,
                "halo_bytes_per_iter_rank0": st.halo_bytes_per_iter, "halo_bytes_per_iter_all_ranks": halo_all,
                "nvlink_gbs_avg_over_iteration": halo_all / (ms_iter * 1e-3) / 1e9,
                "note": "halo and replicated-rhs values received per FCG iteration over NVLink (P2P stores fused "
                        "into the row kernels); GB/s averaged over the whole iteration, not the exposed halo phase"}
    s.close()

    cpu = None
    if rank == 0 and world == 1 and args.cpu_baseline:
        cpu = cpu_baseline_subprocess(args)

    if rank != 0:
        return None
    key = "l1_jacobi_sweep_L0" + ("_27pt" if args.stencil == 27 else "") + \
        ("_" + fmt0 if args.problem != "poisson" else "")
    traffic = ncu_traffic(key, workload_name(args, world), world)
    return {
        "metric": METRIC, "value": t_solve, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_solve * 1e3, "higher_is_better": False,
        "scaling": args.scaling if world > 1 else "weak", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic ({args.problem} operator generated on device, b = 1, u0 = 0)",
        "config": config_dict(args, world),
        "iterations": it, "final_relres": st.final_relres, "ms_per_iter": t_solve * 1e3 / it,
        "setup_s": min(setup_times), "setup_breakdown": {k: sstats[k] for k in ("t_matching", "t_spmm", "t_spmm_comm")},
        "levels": sstats["levels"], "opc": sstats["opc"],
        "vcycle_level_us_per_iter": level_us,
        "spmv_gbs": spmv_gbs, "spmv_frac_hbm": spmv_gbs / peak if spmv_gbs else None,
        "roofline": {"bound": "hbm", "kernel": f"level-0 l1-Jacobi sweep, {sweep_kernel}", "storage": fmt0,
                     "bytes_model": "algorithmic bytes of the stored format: pattern/code/column+value bytes + x, r, "
                                    "(l1 d unless per pattern), y once per launch; gathered neighbours counted once",
                     "csr_model": {"bytes_per_launch": csr_bytes,
                                   "effective_gbs": csr_bytes / (sweep_ms * 1e-3) / 1e9 if sweep["launches"] else None,
                                   "frac": csr_bytes / (sweep_ms * 1e-3) / 1e9 / peak if sweep["launches"] else None,
                                   "note": "same launches against the SURVEY 8d 12*nnz+36*n model of an uncompressed "
                                           "CSR sweep (f64 value + int32 column per entry; x, r, d, y per row)"},
                     "achieved": sweep_gbs, "peak": peak, "unit": "GB/s",
                     "frac": sweep_gbs / peak if sweep_gbs else None, "traffic": traffic,
                     "bytes_per_launch": sweep["bytes_per_launch"], "avg_launch_us": sweep_ms * 1e3,
                     "launches": sweep["launches"], "peak_source": peak_src,
                     "measured": "per-launch CUDA events on the solver stream (event nodes inside the captured "
                                 "iteration graph) during an instrumented solve step following the timed steps",
                     "classes": {name: {"avg_us": 1e3 * k["ms"] / max(k["launches"], 1), "launches": k["launches"],
                                        "gbs": (k["bytes_per_launch"] / (k["ms"] / max(k["launches"], 1) * 1e-3) / 1e9)
                                        if k["launches"] else None}
                                 for name, k in zip(["sweep", "residual", "spmv_dots", "fcg_update"], kt)}},
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": 16 * m, "d2h_bytes_per_step": 8 * m,
                "api": "pairamg_solve (C ABI, pinned host b/u0 in, u out)",
                "h2d_s": h2d_s, "d2h_s": d2h_s, "device_solve_s": e2e_dev,
                "h2d_gbs": 16 * m / h2d_s / 1e9 if h2d_s else None,
                "d2h_gbs": 8 * m / d2h_s / 1e9 if d2h_s else None,
                "host_overhead_s": e2e - h2d_s - d2h_s - e2e_dev},
        "e2e_pipeline_s": pipe,
        "comm": comm,
        "gpu_launches": launches,
        "clocks": clocks,
        "cpu_baseline": cpu,
    }


def _free_port() -> int:
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--stencil", type=int, default=7, choices=[7, 27])
    ap.add_argument("--nd", type=int, default=None)
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--problem", default="poisson", choices=["poisson", "varcoef"])
    ap.add_argument("--levels", type=int, default=2, help="varcoef: distinct cell coefficients (0 = continuous)")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--format", default="auto", choices=["auto", "sten", "pat", "dict", "coded", "plain"])
    ap.add_argument("--replicate-rows", type=int, default=2500000,
                    help="N > 1: coarse levels with at most this many global rows are replicated on every rank")
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--no-pipeline", dest="pipeline", action="store_false")
    ap.add_argument("--ref-sample-iters", type=int, default=3)
    ap.add_argument("--ref-full-budget-s", type=float, default=60.0)
    args = ap.parse_args()
    if args.nd is None:
        args.nd = 256 if args.stencil == 7 else 192
    args.warmup = max(args.warmup, 3)
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is not None and int(env_world) != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but launched as {env_world} ranks (WORLD_SIZE)")
    if args.impl == "reference":
        # rank 0 alone runs the CPU reference; other launcher ranks exit without work
        if int(os.environ.get("RANK", "0")) == 0:
            print(json.dumps(bench_reference(args, args.gpus)), flush=True)
        return
    if args.gpus > 1 and env_world is None:
        # spawn the ranks (one process per GPU), as the reference's harness does
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
        os.execv(sys.executable, cmd)
    world = args.gpus
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    line = bench_ours(args, rank, world, local_rank)
    if line is not None:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
