"""Summarise ncu outputs into profiles/ (committed evidence).

    python scripts/ncu_summary.py --launches gpurun_out/launches.csv \
        --rep gpurun_out/prof_sweep.ncu-rep [--rep ...] --tag r01 [--key l1_jacobi_sweep_L0=k_sell<1]

Writes profiles/<tag>_launches.md (per-kernel share of one profiled solve, from
the gpu__time_duration launch list: cold-cache, serialised -> compare shares),
profiles/<tag>_ncu_full.md (per-launch DRAM bytes, throughput, occupancy,
registers, cache hit rates of the captured kernels) and merges
dram_bytes_per_launch for the keyed kernels into profiles/ncu_summary.json
(read by bench.py for roofline.traffic).
"""
import argparse
import collections
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

WANT = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_pct"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_pct"),
    ("l1tex__t_sector_hit_rate.pct", "l1_hit_pct"),
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "ms": 1e3, "s": 1e6}


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    mi = h.index("Metric Name") if "Metric Name" in h else None
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        if mi is not None and r[mi] != "gpu__time_duration.sum":
            continue
        try:
            v = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1)  # -> us
        except ValueError:
            continue
        name = r[ki].replace("(anonymous namespace)::", "").split("(")[0].replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += v
        tot += v
    return agg, tot


def raw(rep):
    """Rows of an .ncu-rep, or of its `--page raw --csv` export (.csv, made on
    the GPU box when the reports would not fit gpurun's copy-back limit)."""
    if rep.endswith(".csv"):
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")].replace("(anonymous namespace)::", "").split("(")[0].replace("void ", "")}
        for m, k in WANT:
            if m in h:
                i = h.index(m)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    v = None
                if v is not None and u[i] in SCALE and k in ("dram_read", "dram_write"):
                    v *= SCALE[u[i]]
                if v is not None and k == "time":
                    v *= SCALE.get(u[i], 1)
                d[k] = v
        d["dram_bytes"] = (d.get("dram_read") or 0) + (d.get("dram_write") or 0)
        res.append(d)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--rep", action="append", default=[])
    ap.add_argument("--tag", default="r01")
    ap.add_argument("--key", action="append", default=[], help="json_key=kernel-substring")
    ap.add_argument("--note", default="")
    ap.add_argument("--workload", default="poisson7_256x256x256", help="bench config.workload of the capture")
    a = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)
    if a.launches:
        agg, tot = launches(a.launches)
        lines = [f"# {a.tag}: launch list of one profiled solve ({a.note})", "",
                 "ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised: compare shares)",
                 "", "| share | launches | avg us | kernel |", "|---:|---:|---:|---|"]
        for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
            lines.append(f"| {100 * v / tot:.2f}% | {c} | {v / c:.1f} | `{k}` |")
        lines.append(f"\nTotal kernel time {tot / 1e3:.3f} ms over {sum(c for c, _ in agg.values())} launches.")
        open(os.path.join(PROF, f"{a.tag}_launches.md"), "w").write("\n".join(lines) + "\n")
    allrows = []
    for rep in a.rep:
        allrows += [dict(r, rep=os.path.basename(rep)) for r in raw(rep)]
    if allrows:
        lines = [f"# {a.tag}: ncu --set full captures ({a.note})", "",
                 "| kernel | time us | DRAM read MB | DRAM write MB | DRAM GB/s | DRAM % peak | SM % | occupancy % | "
                 "regs | grid x block | L2 hit % | L1 hit % |", "|---|---:|---:|---:|---:|---:|---:|---:|---:|---|---:|---:|"]
        for r in allrows:
            gbs = r["dram_bytes"] / (r["time"] * 1e-6) / 1e9 if r.get("time") else 0
            lines.append(f"| `{r['kernel'][:60]}` | {r.get('time', 0):.1f} | {(r.get('dram_read') or 0) / 1e6:.1f} | "
                         f"{(r.get('dram_write') or 0) / 1e6:.1f} | {gbs:.0f} | {r.get('dram_pct') or 0:.1f} | "
                         f"{r.get('sm_pct') or 0:.1f} | {r.get('occupancy_pct') or 0:.1f} | {r.get('regs') or 0:.0f} | "
                         f"{r.get('grid') or 0:.0f} x {r.get('block') or 0:.0f} | {r.get('l2_hit_pct') or 0:.1f} | "
                         f"{r.get('l1_hit_pct') or 0:.1f} |")
        open(os.path.join(PROF, f"{a.tag}_ncu_full.md"), "w").write("\n".join(lines) + "\n")
        jp = os.path.join(PROF, "ncu_summary.json")
        js = json.load(open(jp)) if os.path.exists(jp) else {}
        for kv in a.key:
            key, sub = kv.split("=", 1)
            sel = [r for r in allrows if sub in r["kernel"]]
            if sel:
                r = sel[0]
                js[key] = {"kernel": r["kernel"], "dram_bytes_per_launch": r["dram_bytes"], "time_us_ncu": r.get("time"),
                           "source": f"{a.tag} {r['rep']}", "workload": a.workload}
        json.dump(js, open(jp, "w"), indent=1)
    print(open(os.path.join(PROF, f"{a.tag}_launches.md")).read() if a.launches else "")


if __name__ == "__main__":
    main()
