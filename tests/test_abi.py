"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/*.h declares, carries sm_100a SASS, and the product never
imports the oracle (no CPU fallback)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    names = set()
    for h in os.listdir(os.path.join(ROOT, "include")):
        if not h.endswith(".h"):
            continue
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names |= set(re.findall(r"\b(pairamg_[a-z0-9_]+)\s*\(", src))
    return sorted(names)


@pytest.fixture(scope="module")
def lib():
    import paper_2303_02352_b200 as pb
    from paper_2303_02352_b200 import build

    build.build()
    return pb.lib()


def test_header_declares_boundary():
    names = declared_functions()
    for must in ("pairamg_setup", "pairamg_solve", "pairamg_vcycle", "pairamg_spmv", "pairamg_runtime_create"):
        assert must in names


def test_every_declared_symbol_exported(lib):
    import paper_2303_02352_b200 as pb

    for name in declared_functions():
        assert hasattr(lib, name), f"{name} declared in include/ but not exported"
    assert set(pb.EXPORTS) == set(declared_functions())


def test_status_names(lib):
    import paper_2303_02352_b200 as pb

    assert pb.lib().pairamg_abi_version() == 2
    for i, name in enumerate(pb.ERROR_NAMES):
        assert lib.pairamg_status_name(i).decode() == name


def test_host_poisson_generator(lib):
    """pairamg_poisson_host equals the oracle's generator."""
    import numpy as np

    import oracle
    import paper_2303_02352_b200 as pb

    for st, dims in ((7, (5, 4, 3)), (27, (4, 4, 4)), (7, (1, 1, 1))):
        o = oracle.Oracle("restatement", stencil=st, nx=dims[0], ny=dims[1], nz=dims[2])
        ref = o.input_csr()
        got = pb.poisson(st, *dims)
        for a, b in zip(got, ref):
            np.testing.assert_array_equal(a, b)
        n = dims[0] * dims[1] * dims[2]
        # any row block
        b0, b1 = n // 3, n - n // 4
        rp, ci, va = pb.poisson(st, *dims, b0, b1)
        np.testing.assert_array_equal(ci, ref[1][ref[0][b0]:ref[0][b1]])
        np.testing.assert_array_equal(rp, ref[0][b0:b1 + 1] - ref[0][b0])


def test_sm100a_code_present(lib):
    import paper_2303_02352_b200 as pb

    out = subprocess.run(["cuobjdump", "--list-elf", pb.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_product_does_not_use_oracle():
    pkg = os.path.join(ROOT, "paper_2303_02352_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "oracle_api.h" not in src and "libpairamg_ref" not in src, f
    import paper_2303_02352_b200 as pb

    out = subprocess.run(["ldd", pb.LIB_PATH], capture_output=True, text=True).stdout
    assert "pairamg_oracle" not in out and "pairamg_ref" not in out


def test_no_load_ahead_of_grid_dependency_wait(lib):
    """Kernels launched with programmatic dependent launch may start while
    their predecessor still writes: no global load may precede the
    griddepcontrol.wait (SASS ACQBULK) -- ptxas hoists ld.global.nc loads."""
    import subprocess
    import sys

    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "check_pdl_sass.py")], capture_output=True,
                       text=True)
    assert r.returncode == 0, r.stdout + r.stderr


def _splitmix_coef(c, seed, levels):
    import numpy as np

    with np.errstate(over="ignore"):
        z = np.uint64(seed) + np.uint64(0x9E3779B97F4A7C15) * (c.astype(np.uint64) + np.uint64(1))
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    if levels > 0:
        return 1.0 + (z % np.uint64(levels)).astype(np.float64)
    return 0.5 + (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def test_host_varcoef_generator(lib):
    """pairamg_varcoef_host = its definition (include/pairamg_b200.h): Poisson
    sparsity, couplings -(k_i + k_j)/2, diagonal = sum over the stencil
    directions (k_i across the boundary), symmetric, diagonally dominant."""
    import numpy as np

    import paper_2303_02352_b200 as pb

    for st, dims, levels in ((7, (5, 4, 6), 2), (7, (6, 5, 4), 0), (27, (4, 5, 3), 3)):
        nx, ny, nz = dims
        n = nx * ny * nz
        rp, ci, va = pb.varcoef(st, nx, ny, nz, levels, 7)
        prp, pci, _ = pb.poisson(st, nx, ny, nz)
        np.testing.assert_array_equal(rp, prp)
        np.testing.assert_array_equal(ci, pci)
        k = _splitmix_coef(np.arange(n), 7, levels)
        rows = np.repeat(np.arange(n), np.diff(rp))
        off = ci != rows
        np.testing.assert_array_equal(va[off], -((k[rows[off]] + k[ci[off]]) * 0.5))
        A = np.zeros((n, n))
        A[rows, ci] = va
        np.testing.assert_array_equal(A, A.T)
        d = np.diag(A)
        assert np.all(d >= np.abs(A - np.diag(d)).sum(axis=1) - 1e-12)
        # diagonal: every direction's (k_i + k_j)/2, or k_i across the boundary, summed in direction order
        for r in (0, n // 2, n - 1):
            i, j, kk = r % nx, (r // nx) % ny, r // (nx * ny)
            s = 0.0
            for dk in (-1, 0, 1):
                for dj in (-1, 0, 1):
                    for di in (-1, 0, 1):
                        man = (di != 0) + (dj != 0) + (dk != 0)
                        if man == 0 or (st == 7 and man > 1):
                            continue
                        ii, jj, k2 = i + di, j + dj, kk + dk
                        inside = 0 <= ii < nx and 0 <= jj < ny and 0 <= k2 < nz
                        s = s + ((k[r] + k[ii + nx * (jj + ny * k2)]) * 0.5 if inside else k[r])
            assert A[r, r] == s
