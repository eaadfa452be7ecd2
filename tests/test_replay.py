"""SetupConfig::replay (amg.hpp:13-23, amg.cpp:182-197) on the GPU setup.

The GPU's parallel Suitor breaks weight ties by a total order; the reference's
sequential Suitor keeps the incumbent (matching.cpp:82).  On coarse steps of
odd grids the two matchings differ, so a bitwise comparison against the
UNMODIFIED reference needs the reference's own matchings replayed: the
recorded MatchingTrace of oracle/_ref (the reference's C++ compiled as is)
is fed to pairamg_setup, and every hierarchy array, every SpMV and the
V-cycle must then equal the reference's bit for bit.
"""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def bits(a):
    a = np.asarray(a)
    return a.view(np.int64) if a.dtype == np.float64 else a


@pytest.fixture(scope="module")
def runtime():
    import paper_2303_02352_b200 as pb

    return pb.Runtime(0, 0, 1)


def reference(stencil, nx, ny, nz, target):
    return oracle.Oracle("reference", stencil=stencil, nx=nx, ny=ny, nz=nz, nranks=1,
                         coarse_size_target=target).setup()


@pytest.mark.parametrize("case", [(7, 33, 33, 33), (7, 33, 31, 29), (27, 15, 15, 15)],
                         ids=lambda c: f"{c[0]}pt-{c[1]}x{c[2]}x{c[3]}")
def test_replayed_reference_hierarchy_bitexact(runtime, case):
    import paper_2303_02352_b200 as pb

    st, nx, ny, nz = case
    target = 40 * nx
    ref = reference(st, nx, ny, nz, target)
    trace = ref.matchings()
    rp, ci, va = ref.input_csr()
    n = len(rp) - 1
    s = pb.Solver(runtime)
    s.setup(n, [0, n], rp, ci, va, cfg=pb.SetupConfig(3, target, 40, replay=trace))
    assert s.level_sizes() == ref.level_sizes()
    assert s.opc == ref.opc
    assert s.num_matchings == len(trace)
    for t, m in enumerate(trace):
        np.testing.assert_array_equal(s.matching(t), m, err_msg=f"matching {t}")
    for k in range(ref.num_levels):
        for name, x, y in zip(["row_ptr", "col", "val", "w", "l1"], s.level(k), ref.level(k)):
            np.testing.assert_array_equal(bits(x), bits(y), err_msg=f"level {k} {name}")
    for k in range(1, ref.num_levels):
        gc, gv = s.prolongator(k)
        oc, ov = ref.prolongator(k)
        np.testing.assert_array_equal(gc, oc)
        np.testing.assert_array_equal(bits(gv), bits(ov))
    rng = np.random.default_rng(5)
    for k in range(ref.num_levels):
        x = rng.standard_normal(ref.level_size(k)[0])
        np.testing.assert_array_equal(bits(s.spmv(k, x)), bits(ref.spmv(k, x)), err_msg=f"spmv {k}")
    r = rng.standard_normal(n)
    np.testing.assert_array_equal(bits(s.vcycle(r)), bits(ref.vcycle(r)))
    out = ref.solve()
    got = s.solve(np.ones(n))
    assert got.converged and abs(got.iterations - out["iterations"]) <= 1
    s.close()


def test_replay_is_needed_on_odd_grids(runtime):
    """Without replay the total-order matching differs from the reference's on
    a coarse step of 33^3 (so the replay test above is not vacuous)."""
    import paper_2303_02352_b200 as pb

    ref = reference(7, 33, 33, 33, 40 * 33)
    rp, ci, va = ref.input_csr()
    n = len(rp) - 1
    s = pb.Solver(runtime)
    s.setup(n, [0, n], rp, ci, va, cfg=pb.SetupConfig(3, 40 * 33, 40))
    k = min(s.num_matchings, ref.num_matchings)
    differs = [t for t in range(k) if len(s.matching(t)) != len(ref.matching(t))
               or not np.array_equal(s.matching(t), ref.matching(t))]
    assert differs, "total-order and reference matchings coincide on 33^3"
    assert differs[0] > 0  # the fine level (all weights tied at 7/6) agrees
    s.close()


def test_replay_errors(runtime):
    import paper_2303_02352_b200 as pb

    rp, ci, va = pb.poisson(7, 10, 10, 10)
    n = len(rp) - 1
    s = pb.Solver(runtime)
    s.setup(n, [0, n], rp, ci, va, cfg=pb.SetupConfig(3, 40, 40))
    trace = [s.matching(t) for t in range(s.num_matchings)]
    # exhausted trace (amg.cpp:184-185)
    with pytest.raises(pb.PairamgError) as e:
        s.setup(n, [0, n], rp, ci, va, cfg=pb.SetupConfig(3, 40, 40, replay=trace[:2]))
    assert e.value.code == "contract_violation" and "trace exhausted" in str(e.value)
    # non-mutual mates (build_pairwise_prolongator, amg.cpp:54-57)
    bad = [m.copy() for m in trace]
    j = int(np.nonzero(bad[0] >= 0)[0][0])
    bad[0][j] = (bad[0][j] + 2) % n
    with pytest.raises(pb.PairamgError) as e:
        s.setup(n, [0, n], rp, ci, va, cfg=pb.SetupConfig(3, 40, 40, replay=bad))
    assert e.value.code == "contract_violation"
    # out-of-range mate = crosses the (single-rank) partition (amg.cpp:187-189)
    bad = [m.copy() for m in trace]
    bad[0][0] = n + 5
    with pytest.raises(pb.PairamgError) as e:
        s.setup(n, [0, n], rp, ci, va, cfg=pb.SetupConfig(3, 40, 40, replay=bad))
    assert e.value.code == "contract_violation" and "crosses the rank partition" in str(e.value)
    # the replay of the solver's own trace reproduces it
    s.setup(n, [0, n], rp, ci, va, cfg=pb.SetupConfig(3, 40, 40, replay=trace))
    assert [s.matching(t).tolist() for t in range(s.num_matchings)] == [m.tolist() for m in trace]
    s.close()


def test_warnings_exported(runtime):
    """Hierarchy::warnings and validate_cycle_config's asymmetry warning."""
    import paper_2303_02352_b200 as pb

    rp, ci, va = pb.poisson(7, 8, 8, 8)
    n = len(rp) - 1
    s = pb.Solver(runtime)
    s.setup(n, [0, n], rp, ci, va, cfg=pb.SetupConfig(3, 40, 40))
    base = s.warnings()
    s.solve(np.ones(n), cycle=pb.CycleConfig(2, 3, 20, 1.0))
    w = s.warnings()
    assert w[-1] == "pre_sweeps != post_sweeps: the V-cycle preconditioner is not symmetric"
    assert w[:-1] == base
    s.solve(np.ones(n))
    assert s.warnings() == base
    s.close()
