"""CPU checkers for the AMG-FCG hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product (``paper_2303_02352_b200``) never imports it and has no CPU fallback.

Two implementations expose the same C API (``oracle_api.h``):

* ``Oracle("restatement")`` -> ``_build/libpairamg_oracle.so``: plain-C
  restatement of the reference algorithm (``pairamg_oracle.c``), each function
  citing the reference file:line it follows.
* ``Oracle("reference")`` -> ``_ref/libpairamg_ref.so``: the reference's own
  seven C++ translation units compiled unmodified (``Makefile``), plus
  ``ref_driver.cpp`` which restates only the absent generator and FCG.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {
    "restatement": os.path.join(HERE, "_build", "libpairamg_oracle.so"),
    "reference": os.path.join(HERE, "_ref", "libpairamg_ref.so"),
}

ERROR_NAMES = [
    "ok", "invalid_argument", "contract_violation", "missing_row", "singular_smoother",
    "stagnation", "breakdown", "deadlock", "parse_error", "io_error", "internal",
]


class OracleError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{ERROR_NAMES[status] if 0 <= status < len(ERROR_NAMES) else status}: {msg}")
        self.status = status
        self.code = ERROR_NAMES[status] if 0 <= status < len(ERROR_NAMES) else str(status)


class Config(C.Structure):
    _fields_ = [
        ("stencil", C.c_int), ("nx", C.c_int64), ("ny", C.c_int64), ("nz", C.c_int64),
        ("nranks", C.c_int), ("aggregation_exponent", C.c_int), ("coarse_size_target", C.c_int64),
        ("max_levels", C.c_int), ("matching_mode", C.c_int), ("pre_sweeps", C.c_int),
        ("post_sweeps", C.c_int), ("coarsest_sweeps", C.c_int), ("relax_weight", C.c_double),
        ("rtol", C.c_double), ("max_iters", C.c_int), ("precflag", C.c_int), ("threads", C.c_int),
    ]


class SetupStats(C.Structure):
    _fields_ = [
        ("t_total", C.c_double), ("t_matching", C.c_double), ("t_spmm", C.c_double),
        ("t_spmm_comm", C.c_double), ("matching_messages", C.c_int64), ("rc_messages", C.c_int64),
    ]


def build(which: str = "all") -> None:
    """Compile the checkers (make in oracle/). 'ref' is skipped without /root/reference."""
    subprocess.run(["make", "-s", "-C", HERE, which], check=True)


_loaded: dict[str, C.CDLL] = {}


def _lib(kind: str) -> C.CDLL:
    if kind in _loaded:
        return _loaded[kind]
    path = LIBS[kind]
    if not os.path.exists(path):
        build("restatement" if kind == "restatement" else "ref")
    L = C.CDLL(path)
    vp, i64, dp, ip = C.c_void_p, C.c_int64, C.POINTER(C.c_double), C.POINTER(C.c_int64)
    L.orc_default_config.argtypes = [C.POINTER(Config)]
    L.orc_create.argtypes = [C.POINTER(Config)]
    L.orc_create.restype = vp
    L.orc_create_csr.argtypes = [C.POINTER(Config), i64, vp, vp, vp]
    L.orc_create_csr.restype = vp
    L.orc_destroy.argtypes = [vp]
    L.orc_last_error.restype = C.c_char_p
    L.orc_last_status.restype = C.c_int
    L.orc_global_n.argtypes = [vp]
    L.orc_global_n.restype = i64
    L.orc_global_nnz.argtypes = [vp]
    L.orc_global_nnz.restype = i64
    L.orc_export_input.argtypes = [vp, vp, vp, vp]
    L.orc_setup.argtypes = [vp]
    L.orc_num_levels.argtypes = [vp]
    L.orc_opc.argtypes = [vp]
    L.orc_opc.restype = C.c_double
    L.orc_get_setup_stats.argtypes = [vp, C.POINTER(SetupStats)]
    L.orc_level_size.argtypes = [vp, C.c_int, ip, ip]
    L.orc_level_partition.argtypes = [vp, C.c_int, vp]
    L.orc_export_level.argtypes = [vp, C.c_int, vp, vp, vp, vp, vp]
    L.orc_export_prolongator.argtypes = [vp, C.c_int, vp, vp]
    L.orc_num_matchings.argtypes = [vp]
    L.orc_export_matching.argtypes = [vp, C.c_int, vp]
    L.orc_matching_size.argtypes = [vp, C.c_int]
    L.orc_matching_size.restype = i64
    L.orc_spmv.argtypes = [vp, C.c_int, vp, vp]
    L.orc_vcycle.argtypes = [vp, vp, vp]
    L.orc_solve.argtypes = [vp, vp, vp, vp, C.c_int, C.POINTER(C.c_int), dp, dp]
    L.orc_set_solve.argtypes = [vp, C.c_double, C.c_int]
    L.orc_build_weights.argtypes = [i64, vp, vp, vp, vp, vp, vp, vp]
    L.orc_build_weights.restype = i64
    L.orc_match_graph.argtypes = [i64, vp, vp, vp, C.c_int, vp]
    if hasattr(L, "orc_mm_load"):  # reference checker only
        L.orc_mm_load.argtypes = [C.c_char_p]
        L.orc_mm_load.restype = vp
        L.orc_mm_info.argtypes = [vp, ip, ip, ip]
        L.orc_mm_export.argtypes = [vp, vp, vp, vp]
        L.orc_mm_free.argtypes = [vp]
        L.orc_mm_write.argtypes = [C.c_char_p, i64, i64, vp, vp, vp]
        L.orc_spgemm.argtypes = [i64, i64, vp, vp, vp, i64, vp, vp, vp]
        L.orc_spgemm.restype = vp
    _loaded[kind] = L
    return L


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def build_weights(kind, rp, col, val, w):
    """build_weights (matching.cpp:28-60) of a square block -> (grp, gcol, gw)."""
    L = _lib(kind)
    rp, col = np.ascontiguousarray(rp, np.int64), np.ascontiguousarray(col, np.int64)
    val, w = np.ascontiguousarray(val, np.float64), np.ascontiguousarray(w, np.float64)
    n = len(rp) - 1
    grp = np.empty(n + 1, np.int64)
    gcol = np.empty(max(len(col), 1), np.int64)
    gw = np.empty(max(len(col), 1), np.float64)
    m = L.orc_build_weights(n, _p(rp), _p(col), _p(val), _p(w), _p(grp), _p(gcol), _p(gw))
    if m < 0:
        raise OracleError(L.orc_last_status(), L.orc_last_error().decode())
    return grp, gcol[:m], gw[:m]


def match_graph(kind, rp, col, w, mode=0):
    """suitor_match (matching.cpp:62-100) on a weighted graph CSR -> mate."""
    L = _lib(kind)
    rp, col = np.ascontiguousarray(rp, np.int64), np.ascontiguousarray(col, np.int64)
    w = np.ascontiguousarray(w, np.float64)
    mate = np.empty(len(rp) - 1, np.int64)
    if L.orc_match_graph(len(rp) - 1, _p(rp), _p(col), _p(w), mode, _p(mate)) != 0:
        raise OracleError(L.orc_last_status(), L.orc_last_error().decode())
    return mate


def mm_read(path: str):
    """Reference read_matrix_market (mm_io.cpp:26-88): (nrows, ncols, row_ptr, col, val)."""
    L = _lib("reference")
    h = L.orc_mm_load(os.fsencode(path))
    if not h:
        raise OracleError(L.orc_last_status(), L.orc_last_error().decode())
    try:
        n, nc, nz = C.c_int64(), C.c_int64(), C.c_int64()
        L.orc_mm_info(h, C.byref(n), C.byref(nc), C.byref(nz))
        rp = np.empty(n.value + 1, np.int64)
        ci = np.empty(nz.value, np.int64)
        va = np.empty(nz.value, np.float64)
        L.orc_mm_export(h, _p(rp), _p(ci), _p(va))
    finally:
        L.orc_mm_free(h)
    return n.value, nc.value, rp, ci, va


def spgemm(A, B):
    """Reference spgemm_local (csr.cpp:206-279). A, B = (row_ptr, col, val, ncols)."""
    L = _lib("reference")
    arp, acol, aval, am = A
    brp, bcol, bval, bm = B
    arp, acol, brp, bcol = (np.ascontiguousarray(x, np.int64) for x in (arp, acol, brp, bcol))
    aval, bval = (np.ascontiguousarray(x, np.float64) for x in (aval, bval))
    h = L.orc_spgemm(len(arp) - 1, am, _p(arp), _p(acol), _p(aval), bm, _p(brp), _p(bcol), _p(bval))
    if not h:
        raise OracleError(L.orc_last_status(), L.orc_last_error().decode())
    try:
        n, nc, nz = C.c_int64(), C.c_int64(), C.c_int64()
        L.orc_mm_info(h, C.byref(n), C.byref(nc), C.byref(nz))
        rp = np.empty(n.value + 1, np.int64)
        ci = np.empty(nz.value, np.int64)
        va = np.empty(nz.value, np.float64)
        L.orc_mm_export(h, _p(rp), _p(ci), _p(va))
    finally:
        L.orc_mm_free(h)
    return rp, ci, va


def mm_write(path: str, row_ptr, col, val, ncols=None):
    """Reference write_matrix_market (mm_io.cpp:90-110)."""
    L = _lib("reference")
    rp = np.ascontiguousarray(row_ptr, np.int64)
    ci = np.ascontiguousarray(col, np.int64)
    va = np.ascontiguousarray(val, np.float64)
    n = len(rp) - 1
    rc = L.orc_mm_write(os.fsencode(path), n, n if ncols is None else ncols, _p(rp), _p(ci), _p(va))
    if rc:
        raise OracleError(rc, L.orc_last_error().decode())


class Oracle:
    """One problem instance + hierarchy in a CPU checker."""

    def __init__(self, kind: str = "restatement", *, stencil=7, nd=None, nx=16, ny=None, nz=None,
                 nranks=1, csr=None, **cfg):
        self.kind = kind
        self.L = _lib(kind)
        c = Config()
        self.L.orc_default_config(C.byref(c))
        if nd is not None:
            nx = ny = nz = nd
        c.nx = nx
        c.ny = nx if ny is None else ny
        c.nz = nx if nz is None else nz
        c.stencil = stencil
        c.nranks = nranks
        for k, v in cfg.items():
            if not hasattr(c, k):
                raise TypeError(f"unknown oracle config key {k}")
            setattr(c, k, v)
        self.cfg = c
        if csr is not None:
            rp, ci, va = (np.ascontiguousarray(csr[0], np.int64), np.ascontiguousarray(csr[1], np.int64),
                          np.ascontiguousarray(csr[2], np.float64))
            self.h = self.L.orc_create_csr(C.byref(c), len(rp) - 1, _p(rp), _p(ci), _p(va))
        else:
            self.h = self.L.orc_create(C.byref(c))
        if not self.h:
            self._raise()

    def _raise(self):
        raise OracleError(self.L.orc_last_status(), self.L.orc_last_error().decode())

    def _check(self, rc):
        if rc != 0:
            self._raise()

    def close(self):
        if getattr(self, "h", None):
            self.L.orc_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def n(self) -> int:
        return self.L.orc_global_n(self.h)

    @property
    def nnz(self) -> int:
        return self.L.orc_global_nnz(self.h)

    def input_csr(self):
        rp = np.empty(self.n + 1, np.int64)
        ci = np.empty(self.nnz, np.int64)
        va = np.empty(self.nnz, np.float64)
        self._check(self.L.orc_export_input(self.h, _p(rp), _p(ci), _p(va)))
        return rp, ci, va

    def setup(self):
        self._check(self.L.orc_setup(self.h))
        return self

    @property
    def num_levels(self) -> int:
        return self.L.orc_num_levels(self.h)

    @property
    def opc(self) -> float:
        return self.L.orc_opc(self.h)

    def setup_stats(self) -> dict:
        s = SetupStats()
        self._check(self.L.orc_get_setup_stats(self.h, C.byref(s)))
        return {k: getattr(s, k) for k, _ in SetupStats._fields_}

    def level_size(self, k):
        n, nnz = C.c_int64(), C.c_int64()
        self._check(self.L.orc_level_size(self.h, k, C.byref(n), C.byref(nnz)))
        return n.value, nnz.value

    def level_sizes(self):
        return [self.level_size(k) for k in range(self.num_levels)]

    def level_partition(self, k):
        s = np.empty(self.cfg.nranks + 1, np.int64)
        self._check(self.L.orc_level_partition(self.h, k, _p(s)))
        return s

    def level(self, k):
        """(row_ptr, col, val, w, l1) of A^k assembled globally."""
        n, nnz = self.level_size(k)
        rp = np.empty(n + 1, np.int64)
        ci = np.empty(nnz, np.int64)
        va = np.empty(nnz, np.float64)
        w = np.empty(n, np.float64)
        l1 = np.empty(n, np.float64)
        self._check(self.L.orc_export_level(self.h, k, _p(rp), _p(ci), _p(va), _p(w), _p(l1)))
        return rp, ci, va, w, l1

    def prolongator(self, k):
        """(col, val) of the composed prolongator into level k, one entry per fine row."""
        nf, _ = self.level_size(k - 1)
        ci = np.empty(nf, np.int64)
        va = np.empty(nf, np.float64)
        self._check(self.L.orc_export_prolongator(self.h, k, _p(ci), _p(va)))
        return ci, va

    def matchings(self):
        return [self.matching(s) for s in range(self.num_matchings)]

    def matching(self, step):
        n = self.L.orc_matching_size(self.h, step)
        m = np.empty(n, np.int64)
        self._check(self.L.orc_export_matching(self.h, step, _p(m)))
        return m

    @property
    def num_matchings(self) -> int:
        return self.L.orc_num_matchings(self.h)

    def spmv(self, k, x):
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty(self.level_size(k)[0], np.float64)
        self._check(self.L.orc_spmv(self.h, k, _p(x), _p(y)))
        return y

    def vcycle(self, r):
        r = np.ascontiguousarray(r, np.float64)
        x = np.empty_like(r)
        self._check(self.L.orc_vcycle(self.h, _p(r), _p(x)))
        return x

    def set_solve(self, rtol=None, max_iters=None):
        rtol = self.cfg.rtol if rtol is None else rtol
        max_iters = self.cfg.max_iters if max_iters is None else max_iters
        self.cfg.rtol, self.cfg.max_iters = rtol, max_iters
        self._check(self.L.orc_set_solve(self.h, rtol, max_iters))

    def solve(self, b=None, want_u=False, hist_cap=1024):
        if b is not None:
            b = np.ascontiguousarray(b, np.float64)
        u = np.empty(self.n, np.float64) if want_u else None
        hist = np.zeros(hist_cap, np.float64)
        it = C.c_int()
        rel = C.c_double()
        t = C.c_double()
        self._check(self.L.orc_solve(self.h, _p(b), _p(u), _p(hist), hist_cap, C.byref(it), C.byref(rel),
                                     C.byref(t)))
        return {"iterations": it.value, "relres": rel.value, "t_solve": t.value,
                "history": hist[: it.value + 1].copy(), "u": u}
