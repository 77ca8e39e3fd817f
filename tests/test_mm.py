"""Matrix Market ingest against the reference's own reader.

CPU: the host parser (plnmf_mm_read) accepts and rejects exactly what
read_matrix_market does (proj/src/matrix_market.cpp), with the same message
and line number, for a battery of well-formed and malformed files.
GPU: the device assembly (rows bucketed, columns sorted keeping file order,
duplicates summed in file order, :147-172) gives the reference's CSR bit for
bit, and an engine built from the file iterates like one built from that CSR.
"""
import numpy as np
import pytest

from _helpers import bits_equal
from oracle import oracle as O
from paper_1904_07935_b200 import plnmf as P

needs_ref = pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built (needs /root/reference)")

HDR = "%%MatrixMarket matrix coordinate real general\n"
GOOD = {
    "coordinate": HDR + "% comment\n\n3 4 4\n1 1 2.5\n3 4 1\n1 1 0.5\n2 2 3e-1\n",
    "crlf_comments": HDR.replace("\n", "\r\n") + "  % indented comment\r\n2 2 1\r\n2 1 7\r\n",
    "pattern": "%%MatrixMarket matrix coordinate pattern general\n3 3 3\n1 2\n3 3\n1 2\n",
    "case_banner": "%%matrixmarket MATRIX Coordinate REAL General\n2 2 1\n1 2 4\n",
    "empty_coord": HDR + "5 6 0\n",
    "array": "%%MatrixMarket matrix array real general\n2 3\n1\n2\n3 4\n5\n6\n",
    "zeros": HDR + "2 2 2\n1 1 0\n2 2 0.0\n",
}
BAD = {
    "empty": "",
    "no_banner": "%MatrixMarket matrix coordinate real general\n1 1 0\n",
    "object": "%%MatrixMarket vector coordinate real general\n1 1 0\n",
    "format": "%%MatrixMarket matrix sparse real general\n1 1 0\n",
    "field": "%%MatrixMarket matrix coordinate complex general\n1 1 0\n",
    "symmetry": "%%MatrixMarket matrix coordinate real symmetric\n1 1 0\n",
    "pattern_array": "%%MatrixMarket matrix array pattern general\n1 1\n",
    "no_size": HDR + "% only comments\n",
    "size_trailing": HDR + "2 2 1 7\n1 1 1\n",
    "size_short": HDR + "2 2\n",
    "negative_size": HDR + "-2 2 0\n",
    "no_value": HDR + "2 2 1\n1 1\n",
    "trailing": HDR + "2 2 1\n1 1 1 x\n",
    "inf": HDR + "2 2 1\n1 1 inf\n",
    "nan": HDR + "2 2 1\n1 1 nan\n",
    "negative": HDR + "2 2 2\n1 1 1\n2 2 -0.5\n",
    "row_oob": HDR + "2 2 1\n3 1 1\n",
    "col_oob": HDR + "2 2 1\n1 0 1\n",
    "eof": HDR + "2 2 3\n1 1 1\n2 2 1\n",
    "extra": HDR + "2 2 1\n1 1 1\n2 2 1\n",
    "bad_index": HDR + "2 2 1\nx 1 1\n",
    "array_missing": "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n",
    "array_extra": "%%MatrixMarket matrix array real general\n1 2\n1 2 3\n",
    "array_extra_line": "%%MatrixMarket matrix array real general\n1 1\n1\n2\n",
    "array_negative": "%%MatrixMarket matrix array real general\n1 2\n1\n-2\n",
}


def _write(tmp_path, name, text):
    p = tmp_path / f"{name}.mtx"
    p.write_bytes(text.encode())
    return p


@needs_ref
@pytest.mark.parametrize("name", sorted(BAD))
def test_rejects_like_the_reference(tmp_path, name):
    p = _write(tmp_path, name, BAD[name])
    with pytest.raises(O.RefError) as ref_err:
        O.ref_read_mm(p)
    with pytest.raises(P.ParseError) as ours:
        P.read_matrix_market(str(p))
    assert str(ours.value) == ref_err.value.args[1]


@needs_ref
@pytest.mark.parametrize("name", sorted(GOOD))
def test_accepts_like_the_reference(tmp_path, name):
    p = _write(tmp_path, name, GOOD[name])
    ref = O.ref_read_mm(p)
    mm = P.read_matrix_market(str(p))
    assert (mm.rows, mm.cols) == (ref["rows"], ref["cols"])
    assert mm.sparse == ("rp" in ref)


def test_missing_file_and_string_source():
    with pytest.raises(P.ParseError, match="cannot open file"):
        P.read_matrix_market("/nonexistent/none.mtx")
    with pytest.raises(P.ParseError) as e:
        P.MatrixMarket(text=BAD["negative"], source="mem.mtx")
    assert str(e.value) == "mem.mtx:4: value must be non-negative" and e.value.line == 4


def _random_mm(rng, rows, cols, n, dup_frac=0.3, pattern=False):
    r = rng.integers(1, rows + 1, n)
    c = rng.integers(1, cols + 1, n)
    k = int(n * dup_frac)
    if n and k:  # plant duplicates at random later positions
        src = rng.integers(0, n, k)
        dst = rng.integers(0, n, k)
        r[dst], c[dst] = r[src], c[src]
    v = rng.uniform(0.0, 3.0, n)
    kind = "pattern" if pattern else "real"
    lines = [f"%%MatrixMarket matrix coordinate {kind} general", f"{rows} {cols} {n}"]
    for i in range(n):
        lines.append(f"{r[i]} {c[i]}" if pattern else f"{r[i]} {c[i]} {float(v[i])!r}")
    return "\n".join(lines) + "\n"


@needs_ref
@pytest.mark.gpu
@pytest.mark.parametrize("rows,cols,n,pattern", [(1, 1, 3, False), (40, 30, 500, False), (300, 200, 20000, False),
                                                 (50, 60, 800, True), (1000, 5, 4000, False)])
def test_device_assembly_matches_reference_csr(gpu, tmp_path, rows, cols, n, pattern):
    rng = np.random.default_rng(rows * 7 + n)
    p = _write(tmp_path, "rand", _random_mm(rng, rows, cols, n, pattern=pattern))
    ref = O.ref_read_mm(p)
    eng = P.read_matrix_market(str(p)).engine(rank=3)
    got = eng.get_csr()
    assert (got.row_ptr == ref["rp"]).all()
    assert (got.col_idx == ref["ci"]).all()
    assert bits_equal(got.values, ref["val"])
    assert eng.norm_sq == O.RefInput(rows, cols, ref["rp"], ref["ci"], ref["val"]).norm_sq


@needs_ref
@pytest.mark.gpu
def test_engine_from_file_iterates_like_engine_from_csr(gpu, tmp_path):
    rng = np.random.default_rng(5)
    p = _write(tmp_path, "it", _random_mm(rng, 120, 90, 3000))
    ref = O.ref_read_mm(p)
    cfg = P.SolverConfig(rank=6, max_iters=4, rel_tol=0.0, tile_size=4)
    f = P.init_factors(120, 90, cfg)
    e1 = P.read_matrix_market(str(p)).engine(6)
    e1.set_factors(f)
    t1 = e1.iterate(cfg, P.Algorithm.tiled)
    e2 = P.Engine(P.InputMatrix(P.CsrMatrix(120, 90, ref["rp"], ref["ci"], ref["val"])), 6)
    e2.set_factors(f)
    t2 = e2.iterate(cfg, P.Algorithm.tiled)
    assert [r.rel_error for r in t1.records] == [r.rel_error for r in t2.records]
    assert bits_equal(e1.get_factors().w, e2.get_factors().w)


@needs_ref
@pytest.mark.gpu
def test_dense_array_file(gpu, tmp_path):
    p = _write(tmp_path, "arr", GOOD["array"])
    ref = O.ref_read_mm(p)
    eng = P.read_matrix_market(str(p)).engine(2)
    assert (eng.v, eng.d, eng.nnz) == (2, 3, 6)
    assert eng.norm_sq == float(np.sum(ref["dense"].ravel(order="F") ** 2))
