"""Reference FCG iteration counts for the multi-GPU configs, from the REFERENCE
ITSELF (oracle/_ref: the reference's C++ compiled unmodified + restated FCG),
run on the GPU box's host cores (196 GB, 16 cores; this container has 62 GB).

    python scripts/ref_counts.py [--only NAME ...] > gpurun_out/ref_counts.jsonl

One JSON line per config as it finishes: stencil, grid, p (ranks = threads,
the partition the GPU run uses), levels, level sizes, OPC, iterations,
relres, setup / solve seconds, peak RSS.  Committed as
tests/golden/ref_counts.json; bench.py's reference arm and the iteration
parity test read it.
"""
import argparse
import json
import os
import resource
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

# name: (stencil, nx, ny, nz, p, coarse_size_target)
CONFIGS = {
    "zbox7_p2": (7, 256, 256, 512, 2, 40 * 256),
    "zbox7_p4": (7, 256, 256, 1024, 4, 40 * 256),
    "zbox7_p8": (7, 256, 256, 2048, 8, 40 * 256),
    "zbox27_p2": (27, 192, 192, 384, 2, 40 * 192),
    "zbox27_p4": (27, 192, 192, 768, 4, 40 * 192),
    "zbox27_p8": (27, 192, 192, 1536, 8, 40 * 192),
    "cube585_p8": (7, 585, 585, 585, 8, 40 * 585),
    "cube585_p4": (7, 585, 585, 585, 4, 40 * 585),
    "cube585_p2": (7, 585, 585, 585, 2, 40 * 585),
}


def run(name):
    st, nx, ny, nz, p, target = CONFIGS[name]
    t0 = time.time()
    o = oracle.Oracle("reference", stencil=st, nx=nx, ny=ny, nz=nz, nranks=p, coarse_size_target=target)
    t_gen = time.time() - t0
    t0 = time.time()
    o.setup()
    t_setup = time.time() - t0
    sizes = [list(x) for x in o.level_sizes()]
    r = o.solve()
    rec = {"name": name, "stencil": st, "grid": [nx, ny, nz], "p": p, "coarse_size_target": target,
           "levels": o.num_levels, "sizes": sizes, "opc": repr(o.opc), "iterations": r["iterations"],
           "relres": repr(r["relres"]), "gen_s": t_gen, "setup_s": t_setup, "solve_s": r["t_solve"],
           "peak_rss_gb": resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6,
           "source": "oracle/_ref (reference C++ unmodified), ranks = threads, Partition::uniform"}
    o.close()
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", nargs="*")
    a = ap.parse_args()
    for name in a.only or list(CONFIGS):
        try:
            rec = run(name)
        except Exception as e:  # report and continue with the next config
            rec = {"name": name, "error": str(e)}
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
