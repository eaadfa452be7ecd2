"""General SpGEMM against the reference's spgemm_local
(csr.cpp:206-272, compiled in oracle/_ref): bitwise, signed zeros included."""
import os

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
ref_available = os.path.exists(oracle.LIBS["reference"]) or os.path.isdir("/root/reference")


def rand_csr(n, m, per_row, rng, zeros=0.0, sort=True):
    rp = [0]
    cols, vals = [], []
    for _ in range(n):
        k = int(rng.integers(0, per_row + 1))
        c = rng.choice(m, size=min(k, m), replace=False) if m else np.zeros(0, int)
        if sort:
            c = np.sort(c)
        v = rng.standard_normal(len(c)) * 10.0 ** rng.integers(-5, 5, len(c))
        if zeros:
            z = rng.random(len(c)) < zeros
            v[z] = np.where(rng.random(z.sum()) < 0.5, 0.0, -0.0)
        cols += list(c)
        vals += list(v)
        rp.append(len(cols))
    return np.array(rp, np.int64), np.array(cols, np.int64), np.array(vals, np.float64), m


@pytest.fixture(scope="module")
def rt():
    import paper_2303_02352_b200 as pb

    r = pb.Runtime(0, 0, 1)
    yield r
    r.close()


@pytest.mark.skipif(not ref_available, reason="reference checker not built")
@pytest.mark.parametrize("shape", [(50, 40, 30, 5), (200, 200, 200, 12), (7, 300, 9, 60), (120, 60, 500, 20),
                                   (1, 1, 1, 1), (30, 30, 30, 0)])
@pytest.mark.parametrize("zeros", [0.0, 0.3])
def test_spgemm_bitwise(rt, shape, zeros):
    import paper_2303_02352_b200 as pb

    n, m, k, per = shape
    g = np.random.default_rng(n * 7 + m + k + int(zeros * 10))
    A = rand_csr(n, m, per, g, zeros)
    B = rand_csr(m, k, per, g, zeros)
    rp, ci, va = pb.spgemm(rt, A, B)
    rrp, rci, rva = oracle.spgemm(A, B)
    np.testing.assert_array_equal(rp, rrp)
    np.testing.assert_array_equal(ci, rci)
    np.testing.assert_array_equal(va.view(np.uint64), rva.view(np.uint64))


@pytest.mark.skipif(not ref_available, reason="reference checker not built")
def test_spgemm_galerkin_of_a_level(rt):
    """R (A P) for the first pairwise step of a Poisson operator equals the
    reference's Galerkin pieces."""
    import paper_2303_02352_b200 as pb

    rp, ci, va = pb.poisson(7, 8, 8, 8)
    n = len(rp) - 1
    A = (rp, ci, va, n)
    # piecewise-constant P: pairs (2i, 2i+1) -> i with 1/sqrt(2)
    nc = n // 2
    P = (np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int64) // 2, np.full(n, 2 ** -0.5), nc)
    AP = pb.spgemm(rt, A, P)
    rAP = oracle.spgemm(A, P)
    for a, b in zip(AP, rAP):
        np.testing.assert_array_equal(np.asarray(a).view(np.uint64), np.asarray(b).view(np.uint64))


def test_spgemm_errors(rt):
    import paper_2303_02352_b200 as pb

    A = (np.array([0, 1], np.int64), np.array([5], np.int64), np.array([1.0]), 3)  # column 5 >= 3
    B = (np.array([0, 0, 0, 0], np.int64), np.zeros(0, np.int64), np.zeros(0), 2)
    with pytest.raises(pb.PairamgError) as e:
        pb.spgemm(rt, A, B)
    assert e.value.code == "contract_violation"
