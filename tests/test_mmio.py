"""MatrixMarket ingest / distribute / write against the
reference's own read_matrix_market / write_matrix_market (mm_io.cpp:26-110)
compiled into oracle/_ref.  CPU only: the reader is host code behind the C ABI."""
import os

import numpy as np
import pytest

import oracle
import paper_2303_02352_b200 as pb

ref_available = os.path.exists(oracle.LIBS["reference"]) or os.path.isdir("/root/reference")
needs_ref = pytest.mark.skipif(not ref_available, reason="reference checker (oracle/_ref) not built")

rng = np.random.default_rng(5)


def rand_sparse(n, m, density, symmetric=False, skew=False, pattern=False):
    """Random coordinate entries (1-based) with distinct positions."""
    cells = set()
    k = max(1, int(density * n * m))
    while len(cells) < k:
        r, c = int(rng.integers(n)), int(rng.integers(m))
        if (symmetric or skew) and r < c:
            r, c = c, r
        if skew and r == c:
            continue
        cells.add((r, c))
    cells = sorted(cells, key=lambda t: rng.random())
    vals = rng.standard_normal(len(cells)) * 10.0 ** rng.integers(-300, 300, len(cells))
    return [(r + 1, c + 1, v) for (r, c), v in zip(cells, vals)]


def write_mm(path, n, m, entries, field="real", symmetry="general", crlf=False, comments=True, fmt="%.17g"):
    nl = "\r\n" if crlf else "\n"
    lines = [f"%%MatrixMarket matrix coordinate {field} {symmetry}"]
    if comments:
        lines += ["% a comment", "", "%another"]
    lines.append(f"{n} {m} {len(entries)}")
    for i, (r, c, v) in enumerate(entries):
        if comments and i % 7 == 3:
            lines.append("% interleaved comment")
        if field == "pattern":
            lines.append(f"{r} {c}")
        elif field == "integer":
            lines.append(f"{r} {c} {int(v) % 1000 - 500}")
        else:
            lines.append(f"{r} {c} " + (fmt % v))
    with open(path, "w", newline="") as f:
        f.write(nl.join(lines) + nl)


CASES = [
    dict(n=40, m=40, symmetry="general", field="real"),
    dict(n=37, m=53, symmetry="general", field="real"),
    dict(n=50, m=50, symmetry="symmetric", field="real"),
    dict(n=45, m=45, symmetry="skew-symmetric", field="real"),
    dict(n=30, m=30, symmetry="general", field="pattern"),
    dict(n=30, m=30, symmetry="symmetric", field="integer"),
    dict(n=25, m=25, symmetry="general", field="real", crlf=True),
    dict(n=25, m=25, symmetry="symmetric", field="real", crlf=True, comments=False),
    dict(n=1, m=1, symmetry="general", field="real"),
]


@needs_ref
@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c['n']}x{c['m']}-{c['symmetry']}-{c['field']}")
def test_read_matches_reference(tmp_path, case):
    path = str(tmp_path / "a.mtx")
    sym = case["symmetry"]
    ents = rand_sparse(case["n"], case["m"], 0.15, symmetric=sym == "symmetric", skew=sym == "skew-symmetric")
    write_mm(path, case["n"], case["m"], ents, field=case["field"], symmetry=sym, crlf=case.get("crlf", False),
             comments=case.get("comments", True))
    try:
        rn, rm, rrp, rci, rva = oracle.mm_read(path)
    except oracle.OracleError as er:  # e.g. a CRLF blank line: the reference rejects it, so must we
        with pytest.raises(pb.PairamgError) as eo:
            pb.read_matrix_market(path)
        assert str(eo.value) == str(er)
        return
    n, m, rp, ci, va = pb.read_matrix_market(path)
    assert (n, m) == (rn, rm)
    np.testing.assert_array_equal(rp, rrp)
    np.testing.assert_array_equal(ci, rci)
    np.testing.assert_array_equal(va.view(np.uint64), rva.view(np.uint64))  # bitwise values


@needs_ref
def test_distribute_blocks(tmp_path):
    path = str(tmp_path / "a.mtx")
    rp0, ci0, va0 = pb.poisson(7, 6, 5, 4)
    pb.write_matrix_market(path, rp0, ci0, va0)
    n = len(rp0) - 1
    starts = [0, 31, 64, 64, 97, n]
    cols, vals = [], []
    for b, e in zip(starts[:-1], starts[1:]):
        nn, m, rp, ci, va = pb.read_matrix_market(path, b, e)
        assert nn == n and m == n and len(rp) == e - b + 1 and rp[0] == 0
        np.testing.assert_array_equal(rp, rp0[b:e + 1] - rp0[b])
        cols.append(ci)
        vals.append(va)
    np.testing.assert_array_equal(np.concatenate(cols), ci0)
    np.testing.assert_array_equal(np.concatenate(vals), va0)
    with pytest.raises(pb.PairamgError) as ei:
        pb.read_matrix_market(path, 10, n + 1)
    assert ei.value.code == "contract_violation"


@needs_ref
def test_write_matches_reference(tmp_path):
    ents = rand_sparse(30, 30, 0.2)
    src = str(tmp_path / "src.mtx")
    write_mm(src, 30, 30, ents)
    _, _, rp, ci, va = pb.read_matrix_market(src)
    ours, ref = str(tmp_path / "ours.mtx"), str(tmp_path / "ref.mtx")
    pb.write_matrix_market(ours, rp, ci, va)
    oracle.mm_write(ref, rp, ci, va)
    assert open(ours, "rb").read() == open(ref, "rb").read()
    _, _, rp2, ci2, va2 = pb.read_matrix_market(ours)  # %.17g round-trips every double
    np.testing.assert_array_equal(va2.view(np.uint64), va.view(np.uint64))


BAD = {
    "empty": "",
    "banner": "%%MatrixMarkt matrix coordinate real general\n1 1 1\n1 1 1\n",
    "object": "%%MatrixMarket vector coordinate real general\n1 1 1\n1 1 1\n",
    "format": "%%MatrixMarket matrix array real general\n1 1\n1\n",
    "field": "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n",
    "symmetry": "%%MatrixMarket matrix coordinate real hermitian\n1 1 1\n1 1 1\n",
    "no_size": "%%MatrixMarket matrix coordinate real general\n% only comments\n",
    "bad_size": "%%MatrixMarket matrix coordinate real general\n3 x 1\n",
    "neg_size": "%%MatrixMarket matrix coordinate real general\n-3 3 1\n1 1 1\n",
    "eof": "%%MatrixMarket matrix coordinate real general\n3 3 3\n1 1 1\n2 2 2\n",
    "bad_entry": "%%MatrixMarket matrix coordinate real general\n3 3 1\n1 q 1\n",
    "no_value": "%%MatrixMarket matrix coordinate real general\n3 3 1\n1 1\n",
    "oob": "%%MatrixMarket matrix coordinate real general\n3 3 1\n4 1 1.0\n",
    "skew_diag": "%%MatrixMarket matrix coordinate real skew-symmetric\n3 3 1\n2 2 1.0\n",
    "duplicate": "%%MatrixMarket matrix coordinate real general\n3 3 2\n2 1 1.0\n2 1 3.0\n",
    "sym_duplicate": "%%MatrixMarket matrix coordinate real symmetric\n3 3 2\n2 1 1.0\n1 2 3.0\n",
}


@needs_ref
@pytest.mark.parametrize("name", sorted(BAD))
def test_errors_match_reference(tmp_path, name):
    path = str(tmp_path / f"{name}.mtx")
    with open(path, "w") as f:
        f.write(BAD[name])
    with pytest.raises(oracle.OracleError) as er:
        oracle.mm_read(path)
    with pytest.raises(pb.PairamgError) as eo:
        pb.read_matrix_market(path)
    assert eo.value.code == er.value.code == "parse_error"
    assert str(eo.value) == str(er.value)  # same "path:line: message"


@needs_ref
def test_missing_file(tmp_path):
    path = str(tmp_path / "nope.mtx")
    with pytest.raises(oracle.OracleError) as er:
        oracle.mm_read(path)
    with pytest.raises(pb.PairamgError) as eo:
        pb.read_matrix_market(path)
    assert eo.value.code == er.value.code == "io_error"
    assert str(eo.value) == str(er.value)
