"""pairamg-b200: B200-native AMG-preconditioned flexible CG (BootCMatchGX hot path).

The product is ``libpairamg_b200.so`` (hand-written sm_100a CUDA + NCCL behind
the C ABI in ``include/pairamg_b200.h``).  This module is a thin ctypes
binding that mirrors the reference's C++ solver/preconditioner API
(``setup_hierarchy`` / ``vcycle_apply`` / ``spmv_dist`` / ``pcg_solve``,
``SetupConfig`` / ``CycleConfig`` / ``SolveConfig``, ``ErrorCode``) so parity
tests read like the reference's own.  There is no CPU fallback: importing
fails loudly when the library has not been built.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libpairamg_b200.so")

ERROR_NAMES = [
    "ok", "invalid_argument", "contract_violation", "missing_row", "singular_smoother",
    "stagnation", "breakdown", "deadlock", "parse_error", "io_error", "internal",
]

# Every exported symbol of include/pairamg_b200.h (checked by tests/test_abi.py).
EXPORTS = [
    "pairamg_default_setup_config", "pairamg_default_cycle_config", "pairamg_default_solve_config",
    "pairamg_status_name", "pairamg_last_error", "pairamg_abi_version", "pairamg_comm_unique_id",
    "pairamg_comm_local_id",
    "pairamg_runtime_create", "pairamg_runtime_destroy", "pairamg_solver_create", "pairamg_solver_destroy",
    "pairamg_setup", "pairamg_setup_device", "pairamg_solve", "pairamg_solve_device", "pairamg_vcycle",
    "pairamg_spmv", "pairamg_hierarchy_info", "pairamg_level_info", "pairamg_level_storage", "pairamg_level_export",
    "pairamg_prolongator_export", "pairamg_num_matchings", "pairamg_matching_export",
    "pairamg_get_setup_stats", "pairamg_set_kernel_timing", "pairamg_kernel_timing", "pairamg_launch_count",
    "pairamg_solver_stream", "pairamg_poisson_nnz", "pairamg_poisson_host", "pairamg_poisson_device",
    "pairamg_match_graph", "pairamg_mm_open", "pairamg_mm_rows", "pairamg_mm_copy_rows", "pairamg_mm_close",
    "pairamg_mm_write", "pairamg_spgemm", "pairamg_setup_warnings", "pairamg_setup_warning",
    "pairamg_varcoef_host", "pairamg_varcoef_device",
]

STORAGE = {"auto": -1, "plain": 0, "dict": 1, "pat": 2, "sten": 3, "coded": 4}


class PairamgError(RuntimeError):
    """pairamg::Error (types.hpp:26-35): message plus ErrorCode name."""

    def __init__(self, status: int, msg: str):
        self.status = status
        self.code = ERROR_NAMES[status] if 0 <= status < len(ERROR_NAMES) else str(status)
        super().__init__(f"{self.code}: {msg}")


class SetupConfig(C.Structure):  # amg.hpp:17-23
    """SetupConfig (amg.hpp:17-23).  ``replay`` = MatchingTrace::steps: a list
    of global mate arrays, one per pairwise step (amg.cpp:182-197).  The B200
    extensions: ``storage`` ("auto", "sten", "pat", "dict", "coded", "plain"),
    ``replicate_rows`` and ``setup_overlap`` (include/pairamg_b200.h)."""

    _fields_ = [("aggregation_exponent", C.c_int), ("coarse_size_target", C.c_int64), ("max_levels", C.c_int),
                ("replay_steps", C.c_int), ("replay_mates", C.POINTER(C.POINTER(C.c_int64))),
                ("replay_sizes", C.POINTER(C.c_int64)), ("storage", C.c_int), ("replicate_rows", C.c_int64),
                ("setup_overlap", C.c_int)]

    def __init__(self, aggregation_exponent=3, coarse_size_target=40, max_levels=40, replay=None,
                 storage="auto", replicate_rows=2500000, setup_overlap=False):
        super().__init__(aggregation_exponent, coarse_size_target, max_levels)
        self.storage = STORAGE[storage] if isinstance(storage, str) else int(storage)
        self.replicate_rows = replicate_rows
        self.setup_overlap = 1 if setup_overlap else 0
        self._replay = None
        if replay is not None:
            arrs = [np.ascontiguousarray(m, np.int64) for m in replay]
            ptrs = (C.POINTER(C.c_int64) * len(arrs))(*[a.ctypes.data_as(C.POINTER(C.c_int64)) for a in arrs])
            sizes = (C.c_int64 * len(arrs))(*[len(a) for a in arrs])
            self._replay = (arrs, ptrs, sizes)  # keep the buffers alive
            self.replay_steps = len(arrs)
            self.replay_mates = ptrs
            self.replay_sizes = sizes


class CycleConfig(C.Structure):  # cycle.hpp:7-12
    _fields_ = [("pre_sweeps", C.c_int), ("post_sweeps", C.c_int), ("coarsest_sweeps", C.c_int),
                ("relax_weight", C.c_double)]

    def __init__(self, pre_sweeps=4, post_sweeps=4, coarsest_sweeps=20, relax_weight=1.0):
        super().__init__(pre_sweeps, post_sweeps, coarsest_sweeps, relax_weight)


class SolveConfig(C.Structure):
    _fields_ = [("rtol", C.c_double), ("max_iters", C.c_int), ("precflag", C.c_int)]

    def __init__(self, rtol=1e-6, max_iters=1000, precflag=1):
        super().__init__(rtol, max_iters, precflag)


class _SolveStats(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("final_relres", C.c_double),
                ("rnorm0", C.c_double), ("t_solve_s", C.c_double), ("history", C.POINTER(C.c_double)),
                ("history_cap", C.c_int), ("t_h2d_s", C.c_double), ("t_d2h_s", C.c_double),
                ("reductions_per_iter", C.c_int), ("halo_exchanges_per_iter", C.c_int),
                ("halo_bytes_per_iter", C.c_double)]


class _SetupStats(C.Structure):
    _fields_ = [("t_total", C.c_double), ("t_matching", C.c_double), ("t_spmm", C.c_double),
                ("t_spmm_comm", C.c_double), ("matching_messages", C.c_int64), ("rc_messages", C.c_int64),
                ("levels", C.c_int), ("opc", C.c_double)]


@dataclass
class SolveStats:
    iterations: int
    converged: bool
    final_relres: float
    rnorm0: float
    t_solve_s: float
    history: np.ndarray
    t_h2d_s: float = 0.0
    t_d2h_s: float = 0.0
    reductions_per_iter: int = 0
    halo_exchanges_per_iter: int = 0
    halo_bytes_per_iter: float = 0.0


_lib = None


def lib() -> C.CDLL:
    """Load the CUDA library (raises if it was not built -- no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2303_02352_b200.build` "
                          "(the B200 path has no CPU fallback)")
    # torch first: its bundled libnccl.so.2 (newer) must be the copy the
    # process binds; loading ours first would bind the system one and break
    # a later `import torch` (missing ncclDevCommCreate).
    import torch  # noqa: F401

    L = C.CDLL(LIB_PATH)
    vp, i64, st = C.c_void_p, C.c_int64, C.c_int
    sig = {
        "pairamg_status_name": ([st], C.c_char_p),
        "pairamg_last_error": ([], C.c_char_p),
        "pairamg_abi_version": ([], C.c_int),
        "pairamg_comm_unique_id": ([vp], st),
        "pairamg_comm_local_id": ([vp], st),
        "pairamg_runtime_create": ([C.c_int, C.c_int, C.c_int, vp, C.POINTER(vp)], st),
        "pairamg_runtime_destroy": ([vp], st),
        "pairamg_solver_create": ([vp, C.POINTER(vp)], st),
        "pairamg_solver_destroy": ([vp], st),
        "pairamg_setup": ([vp, i64, vp, i64, vp, vp, vp, vp, C.POINTER(SetupConfig)], st),
        "pairamg_setup_device": ([vp, i64, vp, i64, i64, vp, vp, vp, vp, C.POINTER(SetupConfig)], st),
        "pairamg_solve": ([vp, vp, vp, C.POINTER(CycleConfig), C.POINTER(SolveConfig), C.POINTER(_SolveStats)], st),
        "pairamg_solve_device": ([vp, vp, vp, C.POINTER(CycleConfig), C.POINTER(SolveConfig),
                                  C.POINTER(_SolveStats)], st),
        "pairamg_vcycle": ([vp, vp, vp, C.POINTER(CycleConfig), C.c_int], st),
        "pairamg_spmv": ([vp, C.c_int, vp, vp, C.c_int], st),
        "pairamg_hierarchy_info": ([vp, C.POINTER(C.c_int), C.POINTER(C.c_double)], st),
        "pairamg_level_info": ([vp, C.c_int] + [C.POINTER(i64)] * 5, st),
        "pairamg_level_storage": ([vp, C.c_int, C.POINTER(C.c_int)], st),
        "pairamg_level_export": ([vp, C.c_int, vp, vp, vp, vp, vp], st),
        "pairamg_prolongator_export": ([vp, C.c_int, vp, vp], st),
        "pairamg_num_matchings": ([vp, C.POINTER(C.c_int)], st),
        "pairamg_matching_export": ([vp, C.c_int, C.POINTER(i64), vp], st),
        "pairamg_get_setup_stats": ([vp, C.POINTER(_SetupStats)], st),
        "pairamg_set_kernel_timing": ([vp, C.c_int], st),
        "pairamg_kernel_timing": ([vp, C.c_int, C.POINTER(i64), C.POINTER(C.c_double), C.POINTER(C.c_double)], st),
        "pairamg_launch_count": ([vp, C.POINTER(i64)], st),
        "pairamg_solver_stream": ([vp], vp),
        "pairamg_poisson_nnz": ([C.c_int, i64, i64, i64, i64, i64], i64),
        "pairamg_poisson_host": ([C.c_int, i64, i64, i64, i64, i64, vp, vp, vp], st),
        "pairamg_poisson_device": ([vp, C.c_int, i64, i64, i64, i64, i64, vp, vp, vp], st),
        "pairamg_varcoef_host": ([C.c_int, i64, i64, i64, C.c_int, C.c_uint64, i64, i64, vp, vp, vp], st),
        "pairamg_varcoef_device": ([vp, C.c_int, i64, i64, i64, C.c_int, C.c_uint64, i64, i64, vp, vp, vp], st),
        "pairamg_match_graph": ([vp, i64, vp, vp, vp, vp], st),
        "pairamg_mm_open": ([C.c_char_p, C.POINTER(vp), C.POINTER(i64), C.POINTER(i64), C.POINTER(i64)], st),
        "pairamg_mm_rows": ([vp, i64, i64, C.POINTER(i64)], st),
        "pairamg_mm_copy_rows": ([vp, i64, i64, vp, vp, vp], st),
        "pairamg_mm_close": ([vp], st),
        "pairamg_mm_write": ([C.c_char_p, i64, i64, vp, vp, vp], st),
        "pairamg_spgemm": ([vp, i64, i64, vp, vp, vp, i64, vp, vp, vp, C.POINTER(vp), C.POINTER(i64)], st),
        "pairamg_setup_warnings": ([vp, C.POINTER(C.c_int)], st),
        "pairamg_setup_warning": ([vp, C.c_int, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)], st),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def _check(rc: int) -> None:
    if rc != 0:
        raise PairamgError(rc, lib().pairamg_last_error().decode())


def _ptr(a):
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data_as(C.c_void_p)
    if hasattr(a, "data_ptr"):  # torch tensor on the device
        return C.c_void_p(a.data_ptr())
    return C.c_void_p(int(a))


def unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(lib().pairamg_comm_unique_id(buf))
    return bytes(buf)


def local_id() -> bytes:
    """Join id for ranks that are threads of this process (pairamg_comm_local_id)."""
    buf = (C.c_uint8 * 128)()
    _check(lib().pairamg_comm_local_id(buf))
    return bytes(buf)


def spawn_ranks(nranks: int, program, devices=None, timeout: float = 900.0):
    """spawn_ranks (runtime.hpp:113-136): run ``program(rt)`` on ``nranks``
    threads of this process, one Runtime each (LOCAL transport; all on GPU 0
    unless ``devices`` lists one per rank).  Returns the per-rank results in
    rank order; the first rank failure is re-raised as "rank r: ..." like the
    reference (runtime.cpp:139-151).  Ranks sharing a GPU need
    CUDA_MODULE_LOADING=EAGER and CUDA_DEVICE_MAX_CONNECTIONS >= 2 * ranks
    (e.g. 32) in the environment before CUDA is initialised,
    and ``program`` must not make device-synchronising CUDA calls
    (cudaFree / torch.cuda.empty_cache, cudaDeviceSynchronize) between
    library calls: a peer rank's halo wait may be running on the same GPU."""
    import threading

    uid = local_id()
    devices = devices or [0] * nranks
    out, err = [None] * nranks, [None] * nranks

    def body(r):
        rt = None
        try:
            rt = Runtime(devices[r], r, nranks, uid)
            out[r] = program(rt)
        except BaseException as e:  # noqa: BLE001 -- re-raised below
            err[r] = e
        finally:
            if rt is not None:
                rt.close()

    ts = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(nranks)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout)
    if any(t.is_alive() for t in ts):
        raise PairamgError(7, "spawn_ranks: a rank thread did not finish (deadlock)")
    for r, e in enumerate(err):
        if e is not None:
            if isinstance(e, PairamgError):
                raise PairamgError(e.status, f"rank {r}: {e}") from e
            raise RuntimeError(f"rank {r}: {e}") from e
    return out


def read_matrix_market(path: str, row_begin: int = 0, row_end: int | None = None):
    """MatrixMarket file -> (nrows, ncols, row_ptr, col, val) of rows
    [row_begin, row_end) (read_matrix_market + distribute_matrix, mm_io.cpp:26-110,
    dist.cpp:349-363): local row_ptr from 0, global ascending columns."""
    L = lib()
    h = C.c_void_p()
    n, nc, nz = C.c_int64(), C.c_int64(), C.c_int64()
    _check(L.pairamg_mm_open(os.fsencode(path), C.byref(h), C.byref(n), C.byref(nc), C.byref(nz)))
    try:
        e = n.value if row_end is None else row_end
        k = C.c_int64()
        _check(L.pairamg_mm_rows(h, row_begin, e, C.byref(k)))
        rp = np.empty(max(e - row_begin, 0) + 1, np.int64)
        ci = np.empty(k.value, np.int64)
        va = np.empty(k.value, np.float64)
        _check(L.pairamg_mm_copy_rows(h, row_begin, e, _ptr(rp), _ptr(ci), _ptr(va)))
    finally:
        L.pairamg_mm_close(h)
    return n.value, nc.value, rp, ci, va


def spgemm(rt: "Runtime", A, B):
    """C = A*B on rt's GPU in the reference's summation order (spgemm_local,
    csr.cpp:206-272).  A, B = (row_ptr, col, val, ncols) host arrays;
    returns (row_ptr, col, val)."""
    L = lib()
    arp, acol, aval, am = A
    brp, bcol, bval, bm = B
    arp, acol, brp, bcol = (np.ascontiguousarray(x, np.int64) for x in (arp, acol, brp, bcol))
    aval, bval = (np.ascontiguousarray(x, np.float64) for x in (aval, bval))
    h = C.c_void_p()
    nz = C.c_int64()
    _check(L.pairamg_spgemm(rt.h, len(arp) - 1, am, _ptr(arp), _ptr(acol), _ptr(aval), bm, _ptr(brp), _ptr(bcol),
                            _ptr(bval), C.byref(h), C.byref(nz)))
    try:
        n = len(arp) - 1
        rp = np.empty(n + 1, np.int64)
        ci = np.empty(nz.value, np.int64)
        va = np.empty(nz.value, np.float64)
        _check(L.pairamg_mm_copy_rows(h, 0, n, _ptr(rp), _ptr(ci), _ptr(va)))
    finally:
        L.pairamg_mm_close(h)
    return rp, ci, va


def write_matrix_market(path: str, row_ptr, col, val, ncols: int | None = None) -> None:
    """coordinate real general, %.17g values (write_matrix_market, mm_io.cpp:90-110)."""
    rp = np.ascontiguousarray(row_ptr, np.int64)
    ci = np.ascontiguousarray(col, np.int64)
    va = np.ascontiguousarray(val, np.float64)
    n = len(rp) - 1
    _check(lib().pairamg_mm_write(os.fsencode(path), n, n if ncols is None else ncols, _ptr(rp), _ptr(ci), _ptr(va)))


def poisson(stencil: int, nx: int, ny: int, nz: int, row_begin: int = 0, row_end: int | None = None):
    """Owned rows of the 7/27-point Poisson operator (host CSR, int64/f64)."""
    L = lib()
    if row_end is None:
        row_end = nx * ny * nz
    nnz = L.pairamg_poisson_nnz(stencil, nx, ny, nz, row_begin, row_end)
    rp = np.empty(row_end - row_begin + 1, np.int64)
    ci = np.empty(nnz, np.int64)
    va = np.empty(nnz, np.float64)
    _check(L.pairamg_poisson_host(stencil, nx, ny, nz, row_begin, row_end, _ptr(rp), _ptr(ci), _ptr(va)))
    return rp, ci, va


def varcoef(stencil: int, nx: int, ny: int, nz: int, levels: int = 2, seed: int = 1, row_begin: int = 0,
            row_end: int | None = None):
    """Owned rows of the variable-coefficient operator (pairamg_varcoef_host):
    Poisson sparsity, couplings -(k_i + k_j)/2 from hashed cell coefficients."""
    L = lib()
    if row_end is None:
        row_end = nx * ny * nz
    nnz = L.pairamg_poisson_nnz(stencil, nx, ny, nz, row_begin, row_end)
    rp = np.empty(row_end - row_begin + 1, np.int64)
    ci = np.empty(nnz, np.int64)
    va = np.empty(nnz, np.float64)
    _check(L.pairamg_varcoef_host(stencil, nx, ny, nz, levels, seed, row_begin, row_end, _ptr(rp), _ptr(ci), _ptr(va)))
    return rp, ci, va


def uniform_partition(n: int, p: int) -> np.ndarray:
    """Partition::uniform (runtime.cpp:13-22)."""
    return np.array([(n // p) * r + min(n % p, r) for r in range(p + 1)], np.int64)


def match_graph(rt: "Runtime", row_ptr, col, weight) -> np.ndarray:
    """GPU parallel Suitor (total-order ties) on a weighted graph CSR -> mate."""
    rp = np.ascontiguousarray(row_ptr, np.int64)
    ci = np.ascontiguousarray(col, np.int64)
    w = np.ascontiguousarray(weight, np.float64)
    mate = np.empty(len(rp) - 1, np.int64)
    _check(lib().pairamg_match_graph(rt.h, len(rp) - 1, _ptr(rp), _ptr(ci), _ptr(w), _ptr(mate)))
    return mate


class Runtime:
    """One rank = one GPU (spawn_ranks / RankCtx, runtime.hpp:71-136)."""

    def __init__(self, device: int = 0, rank: int = 0, nranks: int = 1, uid: bytes | None = None):
        self.rank, self.nranks, self.device = rank, nranks, device
        h = C.c_void_p()
        idbuf = (C.c_uint8 * 128).from_buffer_copy(uid) if uid is not None else None
        _check(lib().pairamg_runtime_create(device, rank, nranks, idbuf, C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib().pairamg_runtime_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Solver:
    """The hierarchy + FCG solver of one rank (pairamg_solver)."""

    def __init__(self, rt: Runtime):
        self.rt = rt
        h = C.c_void_p()
        _check(lib().pairamg_solver_create(rt.h, C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib().pairamg_solver_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # setup_hierarchy (amg.hpp:84-85)
    def setup(self, global_n, part_starts, row_ptr, col, val, w0=None, cfg: SetupConfig | None = None):
        cfg = cfg or SetupConfig()
        starts = np.ascontiguousarray(part_starts, np.int64)
        if hasattr(row_ptr, "data_ptr"):  # device tensors
            n_local = int(row_ptr.numel()) - 1
            _check(lib().pairamg_setup_device(self.h, global_n, _ptr(starts), n_local, int(col.numel()),
                                              _ptr(row_ptr), _ptr(col), _ptr(val), _ptr(w0), C.byref(cfg)))
        else:
            rp = np.ascontiguousarray(row_ptr, np.int64)
            ci = np.ascontiguousarray(col, np.int64)
            va = np.ascontiguousarray(val, np.float64)
            w = None if w0 is None else np.ascontiguousarray(w0, np.float64)
            _check(lib().pairamg_setup(self.h, global_n, _ptr(starts), len(rp) - 1, _ptr(rp), _ptr(ci), _ptr(va),
                                       _ptr(w), C.byref(cfg)))
        return self

    # pcg_solve; host numpy arrays or device tensors
    def solve(self, b, u=None, cycle: CycleConfig | None = None, solve_cfg: SolveConfig | None = None,
              hist_cap: int = 1024) -> SolveStats:
        cycle = cycle or CycleConfig()
        solve_cfg = solve_cfg or SolveConfig()
        hist = np.zeros(hist_cap, np.float64)
        st = _SolveStats()
        st.history = hist.ctypes.data_as(C.POINTER(C.c_double))
        st.history_cap = hist_cap
        if hasattr(b, "data_ptr"):
            _check(lib().pairamg_solve_device(self.h, _ptr(b), _ptr(u), C.byref(cycle), C.byref(solve_cfg),
                                              C.byref(st)))
        else:
            b = np.ascontiguousarray(b, np.float64)
            if u is None:
                u = np.zeros_like(b)
            _check(lib().pairamg_solve(self.h, _ptr(b), _ptr(u), C.byref(cycle), C.byref(solve_cfg), C.byref(st)))
        return SolveStats(st.iterations, bool(st.converged), st.final_relres, st.rnorm0, st.t_solve_s,
                          hist[: st.iterations + 1].copy(), st.t_h2d_s, st.t_d2h_s, st.reductions_per_iter,
                          st.halo_exchanges_per_iter, st.halo_bytes_per_iter)

    def vcycle(self, r, cycle: CycleConfig | None = None):
        cycle = cycle or CycleConfig()
        r = np.ascontiguousarray(r, np.float64)
        x = np.empty_like(r)
        _check(lib().pairamg_vcycle(self.h, _ptr(r), _ptr(x), C.byref(cycle), 0))
        return x

    def spmv(self, level, x):
        x = np.ascontiguousarray(x, np.float64)
        n = self.level_info(level)["local_rows"]
        y = np.empty(n, np.float64)
        _check(lib().pairamg_spmv(self.h, level, _ptr(x), _ptr(y), 0))
        return y

    @property
    def num_levels(self) -> int:
        nl, opc = C.c_int(), C.c_double()
        _check(lib().pairamg_hierarchy_info(self.h, C.byref(nl), C.byref(opc)))
        return nl.value

    @property
    def opc(self) -> float:
        nl, opc = C.c_int(), C.c_double()
        _check(lib().pairamg_hierarchy_info(self.h, C.byref(nl), C.byref(opc)))
        return opc.value

    def level_info(self, k) -> dict:
        v = [C.c_int64() for _ in range(5)]
        _check(lib().pairamg_level_info(self.h, k, *[C.byref(x) for x in v]))
        return dict(zip(["global_rows", "global_nnz", "row_begin", "local_rows", "local_nnz"], [x.value for x in v]))

    STORAGE = ("plain", "dict", "pat", "sten", "coded")

    def level_storage(self, k) -> str:
        """Solve-time storage format of level k (which row kernels run)."""
        f = C.c_int()
        _check(lib().pairamg_level_storage(self.h, k, C.byref(f)))
        return self.STORAGE[f.value]

    def level_sizes(self):
        return [(self.level_info(k)["global_rows"], self.level_info(k)["global_nnz"]) for k in range(self.num_levels)]

    def level(self, k):
        """Owned rows of A^k: (row_ptr, global col, val, w, l1)."""
        li = self.level_info(k)
        n, nnz = li["local_rows"], li["local_nnz"]
        rp = np.empty(n + 1, np.int64)
        ci = np.empty(nnz, np.int64)
        va = np.empty(nnz, np.float64)
        w = np.empty(n, np.float64)
        l1 = np.empty(n, np.float64)
        _check(lib().pairamg_level_export(self.h, k, _ptr(rp), _ptr(ci), _ptr(va), _ptr(w), _ptr(l1)))
        return rp, ci, va, w, l1

    def prolongator(self, k):
        nf = self.level_info(k - 1)["local_rows"]
        ci = np.empty(nf, np.int64)
        va = np.empty(nf, np.float64)
        _check(lib().pairamg_prolongator_export(self.h, k, _ptr(ci), _ptr(va)))
        return ci, va

    @property
    def num_matchings(self) -> int:
        s = C.c_int()
        _check(lib().pairamg_num_matchings(self.h, C.byref(s)))
        return s.value

    def matching(self, step):
        n = C.c_int64()
        _check(lib().pairamg_matching_export(self.h, step, C.byref(n), None))
        m = np.empty(n.value, np.int64)
        _check(lib().pairamg_matching_export(self.h, step, C.byref(n), _ptr(m)))
        return m

    def warnings(self) -> list[str]:
        """Hierarchy::warnings (amg.cpp:230-234) + validate_cycle_config's (cycle.cpp:7-13)."""
        n = C.c_int()
        _check(lib().pairamg_setup_warnings(self.h, C.byref(n)))
        out = []
        for i in range(n.value):
            ln = C.c_size_t()
            _check(lib().pairamg_setup_warning(self.h, i, None, 0, C.byref(ln)))
            buf = C.create_string_buffer(ln.value + 1)
            _check(lib().pairamg_setup_warning(self.h, i, buf, ln.value + 1, None))
            out.append(buf.value.decode())
        return out

    def setup_stats(self) -> dict:
        s = _SetupStats()
        _check(lib().pairamg_get_setup_stats(self.h, C.byref(s)))
        return {k: getattr(s, k) for k, _ in _SetupStats._fields_}

    def set_kernel_timing(self, on: bool):
        _check(lib().pairamg_set_kernel_timing(self.h, 1 if on else 0))

    def kernel_timing(self, kclass: int) -> dict:
        n, ms, b = C.c_int64(), C.c_double(), C.c_double()
        _check(lib().pairamg_kernel_timing(self.h, kclass, C.byref(n), C.byref(ms), C.byref(b)))
        return {"launches": n.value, "ms": ms.value, "bytes_per_launch": b.value}

    def launch_count(self) -> int:
        n = C.c_int64()
        _check(lib().pairamg_launch_count(self.h, C.byref(n)))
        return n.value

    def stream(self) -> int:
        return lib().pairamg_solver_stream(self.h) or 0
