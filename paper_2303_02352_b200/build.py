"""Build libpairamg_b200.so in-tree: nvcc for sm_100a, one object per .cu.

    python -m paper_2303_02352_b200.build [--force] [--verbose-ptxas]

Flags: -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false
(--fmad=false: the reference objects contain no FMA, so bitwise parity of
every per-row kernel needs separately rounded multiply and add), static
cudart, NCCL from the system (libnccl.so.2; torch's bundled NCCL satisfies
the same soname when torch is already loaded).
"""
from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libpairamg_b200.so")
SOURCES = ["runtime.cu", "sparse.cu", "sell.cu", "setup.cu", "solve.cu", "mmio.cu", "spgemm.cu", "p2p.cu", "capi.cu"]


def nvcc() -> str:
    for c in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def flags(ptxas_verbose: bool = False) -> list[str]:
    f = [
        "-gencode", "arch=compute_100a,code=sm_100a",
        "-O3", "-lineinfo", "-std=c++17", "--fmad=false",
        "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
        "-I", os.path.join(ROOT, "include"), "-I", CSRC,
        "-Wno-deprecated-gpu-targets",
    ]
    if ptxas_verbose:
        f += ["-Xptxas", "-v"]
    return f


def _headers_mtime() -> float:
    hs = [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".cuh", ".h"))]
    hs.append(os.path.join(ROOT, "include", "pairamg_b200.h"))
    return max(os.path.getmtime(h) for h in hs)


def build(force: bool = False, ptxas_verbose: bool = False, quiet: bool = True) -> str:
    os.makedirs(OBJ, exist_ok=True)
    hm = _headers_mtime()
    jobs = []
    objs = []
    for src in SOURCES:
        sp = os.path.join(CSRC, src)
        op = os.path.join(OBJ, src.replace(".cu", ".o"))
        objs.append(op)
        if force or not os.path.exists(op) or os.path.getmtime(op) < max(os.path.getmtime(sp), hm):
            jobs.append([nvcc(), *flags(ptxas_verbose), "-c", sp, "-o", op])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        return cmd, r

    failed = []
    with ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        for cmd, r in ex.map(run, jobs):
            if r.returncode != 0:
                failed.append((cmd[-3], r.stderr))
            elif not quiet or ptxas_verbose:
                sys.stderr.write(r.stderr)
    if failed:
        msg = "\n".join(f"--- {s}\n{e}" for s, e in failed)
        raise RuntimeError(f"nvcc failed:\n{msg}")
    if jobs or not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs):
        cmd = [nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", LIB, *objs,
               "-L/usr/lib/x86_64-linux-gnu", "-lnccl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    return LIB


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose-ptxas", action="store_true")
    a = ap.parse_args()
    print(build(force=a.force, ptxas_verbose=a.verbose_ptxas, quiet=False))


if __name__ == "__main__":
    main()
