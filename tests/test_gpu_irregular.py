"""The CUDA path on matrices that are NOT constant-coefficient stencils:
random diagonally dominant SPD matrices (irregular rows, many distinct
values -> PLAIN / DICT / PAT storage, generic STEN lengths) and a
variable-coefficient 7-point operator.  Hierarchy, per-level SpMV and the
V-cycle must be bitwise the oracle's (matching_mode=1), formats included."""
import numpy as np
import pytest

import oracle
from tests.test_oracle import random_spd

pytestmark = pytest.mark.gpu


def bits(a):
    a = np.asarray(a)
    return a.view(np.int64) if a.dtype == np.float64 else a


def varcoef7(nd, rng):
    """7-point operator with random positive edge conductances (SPD, M-matrix)."""
    n = nd ** 3
    idx = np.arange(n).reshape(nd, nd, nd)
    kx = 0.5 + rng.random((nd, nd, nd))
    rows = [dict() for _ in range(n)]
    for ax in range(3):
        a = np.moveaxis(idx, ax, 0)
        c = np.moveaxis(kx, ax, 0)
        for s in range(nd - 1):
            for i, j, w in zip(a[s].ravel(), a[s + 1].ravel(), (c[s] + c[s + 1]).ravel() / 2):
                rows[i][j] = -w
                rows[j][i] = -w
    rp, ci, va = [0], [], []
    for i in range(n):
        d = -sum(rows[i].values()) + 0.1
        ent = sorted(list(rows[i].items()) + [(i, d)])
        ci += [c for c, _ in ent]
        va += [v for _, v in ent]
        rp.append(len(ci))
    return np.array(rp), np.array(ci), np.array(va)


@pytest.fixture(scope="module")
def runtime():
    import paper_2303_02352_b200 as pb

    return pb.Runtime(0, 0, 1)


# pairamg_setup_config::storage; a forced format falls back to PLAIN where it cannot encode the rows
FORMATS = ["auto", "pat", "dict", "plain", "coded"]


def check_pair(runtime, rp, ci, va, target, s_exp=3, all_levels=False, storage="auto"):
    import paper_2303_02352_b200 as pb

    orc = oracle.Oracle("restatement", csr=(rp, ci, va), nranks=1, coarse_size_target=target,
                        aggregation_exponent=s_exp, matching_mode=1).setup()
    s = pb.Solver(runtime)
    s.setup(len(rp) - 1, [0, len(rp) - 1], rp, ci, va, cfg=pb.SetupConfig(s_exp, target, 40, storage=storage))
    assert s.level_sizes() == orc.level_sizes()
    for k in range(orc.num_levels):
        for name, x, y in zip(["row_ptr", "col", "val", "w", "l1"], s.level(k), orc.level(k)):
            np.testing.assert_array_equal(bits(x), bits(y), err_msg=f"level {k} {name}")
    rng = np.random.default_rng(3)
    for k in range(orc.num_levels):
        x = rng.standard_normal(orc.level_size(k)[0])
        np.testing.assert_array_equal(bits(s.spmv(k, x)), bits(orc.spmv(k, x)), err_msg=f"spmv level {k}")
    r = rng.standard_normal(orc.n)
    np.testing.assert_array_equal(bits(s.vcycle(r)), bits(orc.vcycle(r)), err_msg="vcycle")
    st = s.solve(np.ones(orc.n))
    assert st.converged and abs(st.iterations - orc.solve()["iterations"]) <= 1
    fmts = [s.level_storage(k) for k in range(orc.num_levels)]
    s.close()
    return fmts if all_levels else fmts[0]


@pytest.mark.parametrize("fmt", FORMATS)
@pytest.mark.parametrize("seed", [0, 1])
def test_random_spd(runtime, fmt, seed):
    rng = np.random.default_rng(100 + seed)
    rp, ci, va, _ = random_spd(300 + 50 * seed, 0.03, rng)
    # random values: DICT/PAT/STEN do not apply and the builder must fall back
    # to PLAIN whatever is requested
    assert check_pair(runtime, rp, ci, va, target=20, s_exp=2, storage=fmt) == "plain"


@pytest.mark.parametrize("fmt", FORMATS)
def test_variable_coefficient_poisson(runtime, fmt):
    rp, ci, va = varcoef7(12, np.random.default_rng(5))
    check_pair(runtime, rp, ci, va, target=200, storage=fmt)


def test_scaled_poisson_keeps_sten(runtime):
    """A constant-coefficient operator with a non-unit scale (h^-2 Poisson)
    still nests into one main pattern at every level."""
    import paper_2303_02352_b200 as pb

    rp, ci, va = pb.poisson(7, 14, 14, 14)
    assert check_pair(runtime, rp, ci, va * 225.0, target=560) == "sten"


def test_odd_grid_coarse_levels_coded(runtime):
    """Odd grids: the pairwise aggregates stop lining up, the coarse operators
    have thousands of distinct column offsets (no DICT / PAT / STEN) but a few
    dozen distinct values -> CODED storage (value code + 24-bit column delta),
    still bitwise."""
    import paper_2303_02352_b200 as pb

    rp, ci, va = pb.poisson(7, 33, 31, 29)
    fmts = check_pair(runtime, rp, ci, va, target=40 * 33, all_levels=True)
    assert fmts[0] == "sten"
    assert "coded" in fmts[1:], fmts


@pytest.mark.parametrize("fmt", ["auto", "coded"])
def test_random_pattern_few_values(runtime, fmt):
    """Random sparsity with quantised values: CODED at level 0."""
    rng = np.random.default_rng(7)
    n = 400
    A = np.zeros((n, n))
    mask = np.triu(rng.random((n, n)) < 0.02, 1)
    q = -rng.integers(1, 5, (n, n)) * 0.25
    A[mask] = q[mask]
    A = A + A.T
    np.fill_diagonal(A, -A.sum(axis=1) + 1.0)
    rp, ci, va = [0], [], []
    for i in range(n):
        nz = np.nonzero(A[i])[0]
        ci.extend(nz.tolist())
        va.extend(A[i, nz].tolist())
        rp.append(len(ci))
    fmts = check_pair(runtime, np.array(rp), np.array(ci), np.array(va), target=20, s_exp=2, all_levels=True,
                      storage=fmt)
    assert fmts[0] == "coded", fmts


def test_dense_coarse_rows(runtime):
    """A coupling row that touches every unknown (arrow matrix): the coarse row
    of its aggregate gathers more R*(A*P) contributions than the block
    kernel's shared memory holds (> 4096), which takes the global-memory
    stable-sort path of the Galerkin product -- still bitwise the oracle."""
    n = 6000
    rows = []
    for i in range(n):
        ent = {}
        if i > 0:
            ent[i - 1] = -1.0
        if i < n - 1:
            ent[i + 1] = -1.0
        ent[i] = 2.5
        rows.append(ent)
    for j in range(2, n):  # row/column 0 coupled to everything
        rows[0][j] = -1e-3
        rows[j][0] = -1e-3
        rows[j][j] += 1e-3
    rows[0][0] += 1e-3 * (n - 2)
    rp, ci, va = [0], [], []
    for ent in rows:
        for c in sorted(ent):
            ci.append(c)
            va.append(ent[c])
        rp.append(len(ci))
    check_pair(runtime, np.array(rp), np.array(ci), np.array(va), target=50, s_exp=3)


@pytest.mark.parametrize("levels", [2, 0])
def test_varcoef_generator_hierarchy(runtime, levels):
    """The device varcoef workload (bench --problem varcoef) at a size with
    several levels and multi-block kernels: bitwise the oracle."""
    import paper_2303_02352_b200 as pb

    rp, ci, va = pb.varcoef(7, 40, 40, 40, levels, 1)
    check_pair(runtime, rp, ci, va, target=1600)
