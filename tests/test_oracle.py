"""Pin the CPU oracle (plain-C restatement) to the reference itself.

* tests/golden/hierarchies.json was produced by the reference's own compiled
  C++ (scripts/make_golden.py, oracle/_ref); the restatement must reproduce
  every digest, size, OPC, iteration count and residual history bit for bit.
* When oracle/_ref is present (built here from /root/reference) the two are
  also compared live on cases outside the fixture set.
* SPEC.md KATs / acceptance criteria that pin this path.
"""
import json
import os

import numpy as np
import pytest

import oracle
from scripts.make_golden import digest, hierarchy_record

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "hierarchies.json")
REF_OK = os.path.exists(oracle.LIBS["reference"])


def golden_cases():
    with open(GOLDEN) as f:
        return json.load(f)["cases"]


@pytest.mark.parametrize("rec", golden_cases(), ids=lambda r: "{stencil}pt-{nx}x{ny}x{nz}-p{nranks}".format(**r["case"]))
def test_restatement_matches_reference_golden(rec):
    o = oracle.Oracle("restatement", coarse_size_target=rec["coarse_size_target"], **rec["case"]).setup()
    got = hierarchy_record(o)
    for key in ("levels", "sizes", "opc", "level_digest", "prolongator_digest", "matching_digest", "spmv_digest",
                "vcycle_digest", "partition"):
        assert got[key] == rec[key], key
    sol = o.solve()
    assert sol["iterations"] == rec["iterations"]
    assert repr(sol["relres"]) == rec["relres"]
    assert [repr(x) for x in sol["history"]] == rec["history"]


@pytest.mark.parametrize("rec", golden_cases(), ids=lambda r: "{stencil}pt-{nx}x{ny}x{nz}-p{nranks}".format(**r["case"]))
def test_total_order_rule(rec):
    """matching_mode 1 (the GPU's rule) vs the reference hierarchy: equal where recorded."""
    o = oracle.Oracle("restatement", coarse_size_target=rec["coarse_size_target"], matching_mode=1,
                      **rec["case"]).setup()
    got = hierarchy_record(o)
    want = rec if rec["total_order_equal"] else rec["total_order"]
    for key in ("sizes", "level_digest", "prolongator_digest", "matching_digest"):
        assert got[key] == want[key], key
    it = o.solve()["iterations"]
    assert abs(it - rec["iterations"]) <= 1  # north star: iteration count within +-1 of the reference


def test_survey_pinned_numbers():
    """64^3 -> rows 262144/32768/4096/2048, nnz 1810432/223232/27136/13312,
    OPC 1.1456, 19 iterations, relres 3.330e-07."""
    rec = [r for r in golden_cases() if r["case"]["nx"] == 64][0]
    assert rec["sizes"] == [[262144, 1810432], [32768, 223232], [4096, 27136], [2048, 13312]]
    assert round(float(rec["opc"]), 4) == 1.1456
    assert rec["iterations"] == 19
    assert f"{float(rec['relres']):.3e}" == "3.330e-07"


@pytest.mark.skipif(not REF_OK, reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("case", [(7, 18, 18, 18, 4), (7, 21, 19, 17, 3), (27, 14, 14, 14, 3), (7, 45, 45, 45, 2)])
def test_restatement_vs_reference_live(case):
    st, nx, ny, nz, p = case
    kw = dict(stencil=st, nx=nx, ny=ny, nz=nz, nranks=p, coarse_size_target=40 * nx)
    a = oracle.Oracle("reference", **kw).setup()
    b = oracle.Oracle("restatement", **kw).setup()
    ra, rb = hierarchy_record(a), hierarchy_record(b)
    assert ra == rb
    sa, sb = a.solve(), b.solve()
    assert sa["iterations"] == sb["iterations"]
    np.testing.assert_array_equal(sa["history"].view(np.int64), sb["history"].view(np.int64))


def random_spd(n, density, rng):
    """Symmetric diagonally dominant random matrix (ascending-column CSR)."""
    A = np.zeros((n, n))
    mask = np.triu(rng.random((n, n)) < density, 1)
    vals = -rng.random((n, n))
    A[mask] = vals[mask]
    A = A + A.T
    np.fill_diagonal(A, -A.sum(axis=1) + 0.5 + rng.random(n))
    rp = [0]
    ci, va = [], []
    for i in range(n):
        nz = np.nonzero(A[i])[0]
        ci.extend(nz.tolist())
        va.extend(A[i, nz].tolist())
        rp.append(len(ci))
    return np.array(rp), np.array(ci), np.array(va), A


@pytest.mark.skipif(not REF_OK, reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("seed", range(6))
def test_random_spd_vs_reference(seed):
    rng = np.random.default_rng(seed)
    rp, ci, va, _ = random_spd(60 + 10 * seed, 0.08, rng)
    for p in (1, 2, 3):
        kw = dict(csr=(rp, ci, va), nranks=p, coarse_size_target=8, aggregation_exponent=2)
        b = oracle.Oracle("restatement", **kw)
        try:
            b.setup()
        except oracle.OracleError as e:
            # Decoupled aggregation can leave no local edges; the reference
            # segfaults in its multi-rank error path here, so
            # only the restatement's error code is checked.
            assert e.code == "stagnation"
            continue
        a = oracle.Oracle("reference", **kw).setup()
        assert hierarchy_record(a) == hierarchy_record(b)
        sa, sb = a.solve(), b.solve()
        assert sa["iterations"] == sb["iterations"]
        np.testing.assert_array_equal(sa["history"].view(np.int64), sb["history"].view(np.int64))


# --------------------------------------------------------------------- SPEC KATs

def lap1d(n):
    rp, ci, va = [0], [], []
    for i in range(n):
        for j, v in ((i - 1, -1.0), (i, 2.0), (i + 1, -1.0)):
            if 0 <= j < n:
                ci.append(j)
                va.append(v)
        rp.append(len(ci))
    return np.array(rp), np.array(ci), np.array(va)


def test_kat_weights():
    """[[2,-1],[-1,2]], w = 1 -> edge weight 1.5."""
    grp, gcol, gw = oracle.build_weights("restatement", [0, 2, 4], [0, 1, 0, 1], [2, -1, -1, 2], [1, 1])
    assert gw.tolist() == [1.5, 1.5]


def test_kat_suitor_path():
    """path 0-1-2 with weights 1, 2 -> (1, 2) matched, 0 unmatched."""
    for mode in (0, 1):
        m = oracle.match_graph("restatement", [0, 1, 3, 4], [1, 0, 2, 1], [1.0, 1.0, 2.0, 2.0], mode)
        assert m.tolist() == [-1, 2, 1]


def test_kat_galerkin_1d():
    """1-D Laplacian n=4, one pairwise step -> [[1,-1/2],[-1/2,1]] (to 1e-12)."""
    o = oracle.Oracle("restatement", csr=lap1d(4), coarse_size_target=2, aggregation_exponent=1).setup()
    rp, ci, va, w, l1 = o.level(1)
    A = np.zeros((2, 2))
    for i in range(2):
        A[i, ci[rp[i]:rp[i + 1]]] = va[rp[i]:rp[i + 1]]
    np.testing.assert_allclose(A, [[1, -0.5], [-0.5, 1]], atol=1e-12)
    pc, pv = o.prolongator(1)
    assert pc.tolist() == [0, 0, 1, 1]
    np.testing.assert_array_equal(pv, np.full(4, 1 / np.sqrt(2)))


def test_kat_l1_diagonal():
    """row (-1, 2, -1) -> 4; interior 7-point row -> 12."""
    o = oracle.Oracle("restatement", csr=lap1d(5), coarse_size_target=100).setup()
    assert o.level(0)[4][2] == 4.0
    o = oracle.Oracle("restatement", nd=4, coarse_size_target=100).setup()
    l1 = o.level(0)[4]
    assert l1[1 + 4 * (1 + 4 * 1)] == 12.0


def test_acceptance_opc_and_convergence():
    """OPC(64^3) in [1.05, 1.30]; nd=30 converges < 60 its, fewer than CG."""
    rec = [r for r in golden_cases() if r["case"]["nx"] == 64][0]
    assert 1.05 <= float(rec["opc"]) <= 1.30
    o = oracle.Oracle("restatement", nd=30, coarse_size_target=40 * 30).setup()
    amg = o.solve()
    cg = oracle.Oracle("restatement", nd=30, precflag=0).solve()
    assert amg["relres"] < 1e-6 and amg["iterations"] < 60
    assert amg["iterations"] < cg["iterations"]


def test_acceptance_rank_robustness():
    """nd=24, p in {1,2,4}: converges, iterations(p=4) <= 1.5 iterations(p=1)."""
    its = [oracle.Oracle("restatement", nd=24, nranks=p, coarse_size_target=40 * 24).setup().solve()["iterations"]
           for p in (1, 2, 4)]
    assert its[2] <= 1.5 * its[0]


def test_fcg_equals_textbook_pcg_identity():
    """with B = I the flexible CG reproduces textbook CG (to 1e-10, 20 its)."""
    o = oracle.Oracle("restatement", nd=16, precflag=0)
    rp, ci, va = o.input_csr()
    n = len(rp) - 1
    A = np.zeros((n, n))
    for i in range(n):
        A[i, ci[rp[i]:rp[i + 1]]] = va[rp[i]:rp[i + 1]]
    b = np.ones(n)
    x = np.zeros(n)
    r = b.copy()
    p = r.copy()
    hist = [1.0]
    r0 = np.linalg.norm(r)
    for _ in range(20):
        Ap = A @ p
        a = (r @ r) / (p @ Ap)
        x += a * p
        rn = r - a * Ap
        hist.append(np.linalg.norm(rn) / r0)
        p = rn + ((rn @ rn) / (r @ r)) * p
        r = rn
    got = o.solve()["history"][:21]
    np.testing.assert_allclose(got, hist[: len(got)], rtol=1e-10)


def test_errors():
    with pytest.raises(oracle.OracleError) as e:
        oracle.Oracle("restatement", csr=(np.array([0, 1, 1]), np.array([0]), np.array([1.0])),
                      coarse_size_target=100).setup()
    assert e.value.code == "singular_smoother"
    with pytest.raises(oracle.OracleError) as e:
        oracle.Oracle("restatement", csr=(np.array([0, 2, 3]), np.array([1, 0, 1]), np.ones(3)))
    assert e.value.code == "contract_violation"


def test_digest_helper_stable():
    assert digest(np.arange(4, dtype=np.int64)) == digest(np.arange(4, dtype=np.int64))
