"""CUDA path vs the CPU oracle on identical inputs (SURVEY.md 8c bit-parity rules).

Hierarchy (matchings, aggregates, prolongators, every A^k pattern AND value,
w^k, l1 diagonals), per-level SpMV and the V-cycle are required bit-exact;
the FCG solve agrees within +-1 iteration and meets rtol, with residual
histories equal to 1e-8 relative over the first iterations (the dot products
are tree reductions on the GPU, sequential on the CPU).  The checker is the
restated oracle with the total-order matching tie rule (matching_mode=1),
itself pinned bit-exact to the compiled reference in tests/test_oracle.py.
"""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

CASES = [
    (7, 16, 16, 16),
    (7, 24, 24, 24),
    (7, 33, 33, 33),
    (7, 20, 17, 23),
    (27, 12, 12, 12),
    (27, 17, 17, 17),
]


def bits(a):
    a = np.asarray(a)
    return a.view(np.int64) if a.dtype == np.float64 else a


@pytest.fixture(scope="module")
def runtime():
    import paper_2303_02352_b200 as pb

    return pb.Runtime(0, 0, 1)


def build_pair(runtime, stencil, nx, ny, nz, target=None, storage="auto"):
    import paper_2303_02352_b200 as pb

    nd = max(nx, ny, nz)
    target = 40 * nd if target is None else target
    orc = oracle.Oracle("restatement", stencil=stencil, nx=nx, ny=ny, nz=nz, nranks=1,
                        coarse_size_target=target, matching_mode=1).setup()
    rp, ci, va = orc.input_csr()
    s = pb.Solver(runtime)
    s.setup(len(rp) - 1, [0, len(rp) - 1], rp, ci, va, cfg=pb.SetupConfig(3, target, 40, storage=storage))
    return orc, s


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}pt-{c[1]}x{c[2]}x{c[3]}")
def test_hierarchy_bitexact(runtime, case):
    orc, s = build_pair(runtime, *case)
    assert s.num_levels == orc.num_levels
    assert s.level_sizes() == orc.level_sizes()
    assert s.opc == orc.opc
    assert s.num_matchings == orc.num_matchings
    for st in range(orc.num_matchings):
        np.testing.assert_array_equal(s.matching(st), orc.matching(st), err_msg=f"matching step {st}")
    for k in range(orc.num_levels):
        g = s.level(k)
        o = orc.level(k)
        for name, x, y in zip(["row_ptr", "col", "val", "w", "l1"], g, o):
            np.testing.assert_array_equal(bits(x), bits(y), err_msg=f"level {k} {name}")
    for k in range(1, orc.num_levels):
        gc, gv = s.prolongator(k)
        oc, ov = orc.prolongator(k)
        np.testing.assert_array_equal(gc, oc, err_msg=f"P{k} cols")
        np.testing.assert_array_equal(bits(gv), bits(ov), err_msg=f"P{k} vals")


@pytest.mark.parametrize("case", CASES[:4], ids=lambda c: f"{c[0]}pt-{c[1]}x{c[2]}x{c[3]}")
def test_spmv_and_vcycle_bitexact(runtime, case):
    orc, s = build_pair(runtime, *case)
    rng = np.random.default_rng(7)
    for k in range(orc.num_levels):
        n = orc.level_size(k)[0]
        x = rng.standard_normal(n)
        np.testing.assert_array_equal(bits(s.spmv(k, x)), bits(orc.spmv(k, x)), err_msg=f"spmv level {k}")
    r = rng.standard_normal(orc.n)
    np.testing.assert_array_equal(bits(s.vcycle(r)), bits(orc.vcycle(r)))


# solve-time storage of every level (csrc/sell.cu, pairamg_setup_config::storage): all must be bit-identical
FORMATS = ["sten", "pat", "dict", "plain", "coded"]


@pytest.mark.parametrize("fmt", FORMATS)
@pytest.mark.parametrize("case", [CASES[1], CASES[3], CASES[4]], ids=lambda c: f"{c[0]}pt-{c[1]}x{c[2]}x{c[3]}")
def test_storage_formats_bitexact(runtime, case, fmt):
    orc, s = build_pair(runtime, *case, storage=fmt)
    assert s.level_storage(0) == fmt
    rng = np.random.default_rng(11)
    for k in range(orc.num_levels):
        x = rng.standard_normal(orc.level_size(k)[0])
        np.testing.assert_array_equal(bits(s.spmv(k, x)), bits(orc.spmv(k, x)), err_msg=f"{fmt} spmv level {k}")
    r = rng.standard_normal(orc.n)
    np.testing.assert_array_equal(bits(s.vcycle(r)), bits(orc.vcycle(r)), err_msg=f"{fmt} vcycle")
    st = s.solve(np.ones(orc.n))
    assert st.converged and abs(st.iterations - orc.solve()["iterations"]) <= 1


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}pt-{c[1]}x{c[2]}x{c[3]}")
def test_fcg_solve(runtime, case):
    import paper_2303_02352_b200 as pb

    orc, s = build_pair(runtime, *case)
    ref = orc.solve()
    b = np.ones(orc.n)
    st = s.solve(b)
    assert st.converged and st.final_relres < 1e-6
    assert abs(st.iterations - ref["iterations"]) <= 1
    m = min(6, len(ref["history"]), len(st.history))
    np.testing.assert_allclose(st.history[:m], ref["history"][:m], rtol=1e-8)
    # solution check: |b - A u| / |b| < rtol via the oracle's exact SpMV
    u = np.zeros(orc.n)
    st2 = s.solve(b, u)
    assert st2.iterations == st.iterations
    res = b - orc.spmv(0, u)
    assert np.linalg.norm(res) / np.linalg.norm(b) < 1e-6


def test_unpreconditioned_cg(runtime):
    import paper_2303_02352_b200 as pb

    orc, s = build_pair(runtime, 7, 16, 16, 16)
    o2 = oracle.Oracle("restatement", stencil=7, nd=16, precflag=0)
    ref = o2.solve()
    st = s.solve(np.ones(orc.n), solve_cfg=pb.SolveConfig(1e-6, 1000, 0))
    assert abs(st.iterations - ref["iterations"]) <= 1
    np.testing.assert_allclose(st.history[:20], ref["history"][:20], rtol=1e-8)


def test_errors(runtime):
    import paper_2303_02352_b200 as pb

    s = pb.Solver(runtime)
    with pytest.raises(pb.PairamgError) as e:
        s.solve(np.ones(8))
    assert e.value.code == "contract_violation"
    rp = np.array([0, 2, 3], np.int64)
    ci = np.array([1, 0, 1], np.int64)  # row 0 columns not strictly increasing
    ci[0], ci[1] = 1, 0
    with pytest.raises(pb.PairamgError) as e:
        s.setup(2, [0, 2], rp, ci, np.ones(3))
    assert e.value.code == "contract_violation"
    # singular smoother: a zero row
    rp = np.array([0, 1, 1], np.int64)
    with pytest.raises(pb.PairamgError) as e:
        s.setup(2, [0, 2], rp, np.array([0], np.int64), np.ones(1), cfg=pb.SetupConfig(3, 40, 40))
    assert e.value.code == "singular_smoother"
    # the failed setup leaves a usable solver: a valid setup + solve afterwards
    rp, ci, va = pb.poisson(7, 6, 6, 6)
    s.setup(len(rp) - 1, [0, len(rp) - 1], rp, ci, va, cfg=pb.SetupConfig(3, 40, 40))
    assert s.solve(np.ones(len(rp) - 1)).converged
    s.close()


@pytest.mark.gpu
def test_runtime_destroyed_before_solver():
    """Either destruction order is safe (GC finalises reference cycles in any order)."""
    import paper_2303_02352_b200 as pb

    rt = pb.Runtime(0, 0, 1)
    s = pb.Solver(rt)
    rp, ci, va = pb.poisson(7, 6, 6, 6)
    s.setup(len(rp) - 1, [0, len(rp) - 1], rp, ci, va, cfg=pb.SetupConfig(3, 40, 40))
    rt.close()
    with pytest.raises(pb.PairamgError) as e:
        s.solve(np.ones(len(rp) - 1))
    assert e.value.code == "contract_violation"
    s.close()
