"""Generate tests/golden/*.json from the REFERENCE ITSELF (oracle/_ref: the
reference's seven C++ units compiled unmodified + the restated FCG driver).

Run here (needs /root/reference to build oracle/_ref):  python scripts/make_golden.py
The fixtures pin: per-level sizes/nnz, OPC, FCG iteration count, relative
residual and history, and SHA-256 digests of every hierarchy array (A^k
row_ptr/col/value bit patterns, w^k, l1 diagonals, composed prolongators,
pairwise matchings), plus digests of A^k x and B x for a fixed input vector.
`total_order_equal` records whether the total-order tie rule (matching_mode
1, the GPU's rule) reproduces the reference hierarchy for that case.
"""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

CASES = [
    dict(stencil=7, nx=16, ny=16, nz=16, nranks=1),
    dict(stencil=7, nx=16, ny=16, nz=16, nranks=2),
    dict(stencil=7, nx=24, ny=24, nz=24, nranks=3),
    dict(stencil=7, nx=20, ny=17, nz=23, nranks=2),
    dict(stencil=7, nx=33, ny=33, nz=33, nranks=1),
    dict(stencil=7, nx=33, ny=33, nz=33, nranks=3),
    dict(stencil=27, nx=12, ny=12, nz=12, nranks=1),
    dict(stencil=27, nx=12, ny=12, nz=12, nranks=2),
    dict(stencil=7, nx=32, ny=32, nz=64, nranks=2),   # z-box weak-scaling proxy (32^3 per rank)
    dict(stencil=7, nx=64, ny=64, nz=64, nranks=1),   # configs[0] (SURVEY-pinned numbers)
]

# BASELINE.json's single-GPU configs (python scripts/make_golden.py --big ->
# tests/golden/hierarchies_big.json).  Slab-aligned, so the hierarchy is the
# same at every power-of-two p; the reference runs at p = 8 host threads.
BIG_CASES = [
    dict(stencil=7, nx=256, ny=256, nz=256, nranks=8),   # configs[1]
    dict(stencil=27, nx=192, ny=192, nz=192, nranks=8),  # configs[4], one GPU's 192^3
]


def digest(a) -> str:
    a = np.ascontiguousarray(a)
    if a.dtype == np.float64:
        a = a.view(np.int64)
    return hashlib.sha256(a.astype("<i8").tobytes()).hexdigest()[:32]


def probe_vector(n):
    i = np.arange(n, dtype=np.float64)
    return np.sin(0.37 * i) + 0.25 * np.cos(1.3 * i)


def hierarchy_record(o):
    rec = {"levels": o.num_levels, "sizes": [list(x) for x in o.level_sizes()], "opc": repr(o.opc), "level_digest": [],
           "prolongator_digest": [], "matching_digest": [], "spmv_digest": [], "partition": []}
    for k in range(o.num_levels):
        rp, ci, va, w, l1 = o.level(k)
        rec["level_digest"].append({"row_ptr": digest(rp), "col": digest(ci), "val": digest(va), "w": digest(w),
                                    "l1": digest(l1)})
        rec["spmv_digest"].append(digest(o.spmv(k, probe_vector(len(w)))))
        rec["partition"].append([int(x) for x in o.level_partition(k)])
    for k in range(1, o.num_levels):
        c, v = o.prolongator(k)
        rec["prolongator_digest"].append({"col": digest(c), "val": digest(v)})
    for s in range(o.num_matchings):
        rec["matching_digest"].append(digest(o.matching(s)))
    rec["vcycle_digest"] = digest(o.vcycle(probe_vector(o.n)))
    return rec


def main():
    big = "--big" in sys.argv
    out = []
    for c in (BIG_CASES if big else CASES):
        nd = max(c["nx"], c["ny"], c["nz"]) if c["nz"] == c["nx"] else c["nx"]
        target = 40 * nd
        ref = oracle.Oracle("reference", coarse_size_target=target, **c).setup()
        rec = {"case": c, "coarse_size_target": target}
        rec.update(hierarchy_record(ref))
        sol = ref.solve()
        rec["iterations"] = sol["iterations"]
        rec["relres"] = repr(sol["relres"])
        rec["history"] = [repr(x) for x in sol["history"]]
        tot = oracle.Oracle("restatement", coarse_size_target=target, matching_mode=1, **c).setup()
        rec2 = hierarchy_record(tot)
        rec["total_order_equal"] = all(rec[k] == rec2[k] for k in ("sizes", "level_digest", "prolongator_digest",
                                                                  "matching_digest"))
        if not rec["total_order_equal"]:
            rec["total_order"] = {"sizes": rec2["sizes"], "opc": rec2["opc"], "level_digest": rec2["level_digest"],
                                  "prolongator_digest": rec2["prolongator_digest"],
                                  "matching_digest": rec2["matching_digest"], "spmv_digest": rec2["spmv_digest"],
                                  "vcycle_digest": rec2["vcycle_digest"], "iterations": tot.solve()["iterations"]}
        if big:  # the p = 8 hierarchy must be the p = 1 hierarchy (slab-aligned): check it
            one = oracle.Oracle("reference", coarse_size_target=target, **{**c, "nranks": 1}).setup()
            r1 = hierarchy_record(one)
            rec["same_hierarchy_p1"] = all(rec[k] == r1[k] for k in ("sizes", "level_digest", "prolongator_digest",
                                                                    "matching_digest", "spmv_digest",
                                                                    "vcycle_digest"))
            del one
        print(c, rec["levels"], rec["opc"], rec["iterations"], rec["relres"], "total_order_equal",
              rec["total_order_equal"], rec.get("same_hierarchy_p1"), flush=True)
        out.append(rec)
    os.makedirs(os.path.join(ROOT, "tests", "golden"), exist_ok=True)
    name = "hierarchies_big.json" if big else "hierarchies.json"
    with open(os.path.join(ROOT, "tests", "golden", name), "w") as f:
        json.dump({"generator": "scripts/make_golden.py (oracle/_ref = reference C++ compiled unmodified)",
                   "probe_vector": "sin(0.37 i) + 0.25 cos(1.3 i)", "cases": out}, f, indent=1)


if __name__ == "__main__":
    main()
