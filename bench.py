#!/usr/bin/env python3
"""AMG-FCG solve benchmark (BASELINE.json metric) -- one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--stencil 7|27] [--nd 256] [--scaling weak|strong]

A step is one complete flexible-CG solve to rtol 1e-6 (u0 = 0, b = 1) of the
3-D Poisson system with the AMG V-cycle preconditioner, hierarchy already
built (setup is timed separately and reported as setup_s).
  N = 1   : configs[1], 7-point 256^3 (16.8M unknowns) on one B200.
  N > 1   : weak scaling (configs[2]): z-box 256 x 256 x 256N, each rank owns
            one 256^3 slab (row-block partition); --scaling strong runs
            --nd^3 split across the N ranks instead (configs[3] is 585^3).
value = solve seconds (device CUDA events on the solver stream, max over
ranks); e2e = the same solve through the C ABI with host buffers
(pairamg_solve: H2D of b and u0, solve, D2H of u inside the timed region).
--impl reference times the reference's own compiled CPU code
(oracle/_ref/libpairamg_ref.so: the reference's seven C++ units + the
restated FCG driver) on the host cores, same config and metric.
"""
from __future__ import annotations

import argparse
import json
import os
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
    nd = args.nd
    if world > 1 and args.scaling == "weak":
        return nd, nd, nd * world, 40 * nd
    return nd, nd, nd, 40 * nd


def slab(n: int, world: int, rank: int):
    import paper_2303_02352_b200 as pb

    starts = pb.uniform_partition(n, world)
    return starts, int(starts[rank]), int(starts[rank + 1])


# ----------------------------------------------------------------------------- CPU reference


def run_reference_cpu(stencil, nx, ny, nz, target, threads, max_iters, oracle_kind="reference"):
    """Reference CPU implementation on `threads` host cores (ranks = threads).
    Returns dict with setup_s, iterations, ms_per_iter, t_solve (for max_iters iterations)."""
    import oracle

    t0 = time.time()
    o = oracle.Oracle(oracle_kind, stencil=stencil, nx=nx, ny=ny, nz=nz, nranks=threads,
                      coarse_size_target=target, max_iters=max_iters)
    t_gen = time.time() - t0
    t0 = time.time()
    o.setup()
    t_setup = time.time() - t0
    r = o.solve()
    it = r["iterations"]
    return {"gen_s": t_gen, "setup_s": t_setup, "iterations": it, "t_solve": r["t_solve"],
            "ms_per_iter": 1e3 * r["t_solve"] / max(it, 1), "relres": r["relres"], "oracle": o}


def host_threads(n_slabs: int) -> int:
    """Largest power of two <= host cores that divides the slab count (slab-aligned partition)."""
    cores = os.cpu_count() or 1
    p = 1
    while p * 2 <= min(cores, 64) and n_slabs % (p * 2) == 0:
        p *= 2
    return p


def bench_reference(args, rank, world):
    """The reference's own compiled CPU implementation, all usable host threads, same config/metric."""
    if rank != 0:
        return None
    import oracle

    nx, ny, nz, target = problem_dims(args, world)
    p = host_threads(nz)
    o = oracle.Oracle("reference", stencil=args.stencil, nx=nx, ny=ny, nz=nz, nranks=p, coarse_size_target=target)
    t0 = time.time()
    o.setup()
    setup_s = time.time() - t0
    k = args.ref_sample_iters
    o.set_solve(1e-6, k)
    r = o.solve()  # first sample = warm-up 1
    ms_iter0 = 1e3 * r["t_solve"] / max(r["iterations"], 1)
    iters_full, full_s = None, None
    if ms_iter0 * 1e-3 * 60 < args.ref_full_budget_s:
        o.set_solve(1e-6, 1000)
        rf = o.solve()
        iters_full, full_s = rf["iterations"], rf["t_solve"]
        o.set_solve(1e-6, k)
    else:
        iters_full = GOLDEN_ITERS.get((args.stencil, nx, ny, nz))
    for _ in range(max(0, args.warmup - 1)):
        o.solve()
    per_iter = []
    for _ in range(args.steps):
        r = o.solve()
        per_iter.append(1e3 * r["t_solve"] / max(r["iterations"], 1))
    ms_iter = sum(per_iter) / len(per_iter)
    value = ms_iter * 1e-3 * iters_full if iters_full else None
    how = (f"measured by one full reference solve ({full_s:.1f}s)" if full_s is not None
           else "golden reference count (tests/golden)")
    sample = (f"{args.stencil}-point {nx}x{ny}x{nz}; reference C++ (oracle/_ref, unmodified units + restated FCG), "
              f"{p} ranks = {p} host threads (slab-aligned, same hierarchy as p=1); setup {setup_s:.1f}s once; "
              f"each step = {k} FCG iterations; solve s = ms/iter x {iters_full} iterations ({how})")
    return {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": value * 1e3 if value else None, "higher_is_better": False,
        "scaling": args.scaling if world > 1 else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args, world),
        "ms_per_iter": ms_iter, "iterations": iters_full, "setup_s": setup_s,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": p, "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


# Golden iteration counts of the reference for slab-aligned runs (tests/golden).
GOLDEN_ITERS = {(7, 64, 64, 64): 19, (7, 128, 128, 128): 25, (7, 256, 256, 256): 42, (27, 192, 192, 192): 32}


def config_dict(args, world):
    nx, ny, nz, target = problem_dims(args, world)
    part = "dp1" if world == 1 else f"rowblock{world}"
    return {
        "workload": f"poisson{args.stencil}_{nx}x{ny}x{nz}" + (f"_{args.scaling}" if world > 1 else ""),
        "unknowns": nx * ny * nz, "stencil": args.stencil, "coarse_size_target": target,
        "aggregation_exponent": 3, "sweeps": "4/4/20 l1-Jacobi", "rtol": 1e-6, "parallelism": part,
        "step": "one full FCG solve to rtol (hierarchy prebuilt)",
        "l2": "working set larger than L2 (no flush): every level-0 vector is 8*unknowns bytes (134 MB at 256^3 "
              "vs 126 MB L2) and one FCG iteration streams several GB",
    }


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
    pb._check(L.pairamg_poisson_device(rt.h, args.stencil, nx, ny, nz, b0, b1, pb._ptr(rp), pb._ptr(ci), pb._ptr(va)))
    s = pb.Solver(rt)
    cfg = pb.SetupConfig(3, target, 40)

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
    peak, peak_src = measured_peaks()
    li0 = s.level_info(0)
    fmt0 = s.level_storage(0)
    sweep_kernel = {"sten": "k_sten<kJacobi> (STEN: one pattern byte per row, uniform offsets/values)",
                    "pat": "k_pat<kJacobi> (PAT: one pattern byte per row)",
                    "dict": "k_sell<kJacobi> (DICT: one code byte per entry)",
                    "plain": "k_sell<kJacobi> (PLAIN SELL-32)"}[fmt0]
    survey_bytes = 12.0 * li0["local_nnz"] + 36.0 * li0["local_rows"]  # SURVEY 8d model: f64 values + int32 columns
    sweep = kt[0]
    sweep_ms = sweep["ms"] / max(sweep["launches"], 1)
    sweep_gbs = sweep["bytes_per_launch"] / (sweep_ms * 1e-3) / 1e9 if sweep["launches"] else None
    spmv = kt[2]
    spmv_ms = spmv["ms"] / max(spmv["launches"], 1)
    spmv_gbs = spmv["bytes_per_launch"] / (spmv_ms * 1e-3) / 1e9 if spmv["launches"] else None
    # e2e: the same solve through the C ABI with pinned host buffers
    hb = torch.ones(m, dtype=torch.float64).pin_memory()
    hu = torch.zeros(m, dtype=torch.float64).pin_memory()
    hb_np, hu_np = hb.numpy(), hu.numpy()
    e2e_times = []
    for k in range(max(2, min(args.steps, 3)) + 1):
        hu_np[:] = 0.0
        barrier()
        t0 = time.perf_counter()
        st_e = s.solve(hb_np, hu_np)
        dt = max_over_ranks(time.perf_counter() - t0)
        if k > 0:
            e2e_times.append(dt)
    e2e = sum(e2e_times) / len(e2e_times)
    # full pipeline once: host CSR -> setup -> solve -> host u
    pipe = None
    if args.pipeline:
        hrp, hci, hva = pb.poisson(args.stencil, nx, ny, nz, b0, b1)
        barrier()
        t0 = time.perf_counter()
        s2 = pb.Solver(rt)
        s2.setup(n, starts, hrp, hci, hva, cfg=cfg)
        hu_np[:] = 0.0
        s2.solve(hb_np, hu_np)
        pipe = max_over_ranks(time.perf_counter() - t0)
        s2.close()

    cpu = None
    if rank == 0 and world == 1 and args.cpu_baseline:
        try:
            p = host_threads(nz)
            r = run_reference_cpu(args.stencil, nx, ny, nz, target, p, args.ref_sample_iters)
            cpu_val = r["ms_per_iter"] * 1e-3 * it
            cpu = {"value": cpu_val, "unit": UNIT, "cores": p, "kind": "reference",
                   "sample": f"reference C++ (oracle/_ref) {p} ranks = {p} host threads: full setup "
                             f"{r['setup_s']:.1f}s + {r['iterations']} FCG iterations "
                             f"({r['ms_per_iter']:.0f} ms/iter) x {it} iterations of this config",
                   "setup_s": r["setup_s"], "ms_per_iter": r["ms_per_iter"]}
        except Exception as ex:  # reported, not fatal
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"failed: {ex}"}

    if rank != 0:
        return None
    traffic = ncu_traffic("l1_jacobi_sweep_L0", config_dict(args, world)["workload"], world)
    line = {
        "metric": METRIC, "value": t_solve, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_solve * 1e3, "higher_is_better": False,
        "scaling": args.scaling if world > 1 else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (3-D Poisson generated on device, b = 1, u0 = 0)",
        "config": config_dict(args, world),
        "iterations": it, "final_relres": st.final_relres, "ms_per_iter": t_solve * 1e3 / it,
        "setup_s": min(setup_times), "setup_breakdown": {k: sstats[k] for k in ("t_matching", "t_spmm", "t_spmm_comm")},
        "levels": sstats["levels"], "opc": sstats["opc"],
        "spmv_gbs": spmv_gbs, "spmv_frac_hbm": spmv_gbs / peak if spmv_gbs else None,
        "roofline": {"bound": "hbm", "kernel": f"level-0 l1-Jacobi sweep, {sweep_kernel}", "storage": fmt0,
                     "bytes_model": "algorithmic bytes of the stored format: pattern/code bytes + x, r, (l1 d unless "
                                    "per pattern), y once per launch; gathered neighbours counted once",
                     "survey_model": {"bytes_per_launch": survey_bytes,
                                      "effective_gbs": survey_bytes / (sweep_ms * 1e-3) / 1e9 if sweep["launches"] else None,
                                      "note": "same launches against the SURVEY 8d 12*nnz+36*n model of an uncompressed "
                                              "CSR sweep; > peak because the stored format moves fewer bytes"},
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
                "api": "pairamg_solve (C ABI, pinned host b/u0 in, u out)"},
        "e2e_pipeline_s": pipe,
        "gpu_launches": launches,
        "clocks": clocks,
        "cpu_baseline": cpu,
    }
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--stencil", type=int, default=7)
    ap.add_argument("--nd", type=int, default=None)
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--no-pipeline", dest="pipeline", action="store_false")
    ap.add_argument("--ref-sample-iters", type=int, default=3)
    ap.add_argument("--ref-full-budget-s", type=float, default=60.0)
    args = ap.parse_args()
    if args.nd is None:
        args.nd = 256 if args.stencil == 7 else 192
    args.warmup = max(args.warmup, 3)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        line = bench_reference(args, rank, world)
        if line is not None:
            print(json.dumps(line), flush=True)
        return
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
