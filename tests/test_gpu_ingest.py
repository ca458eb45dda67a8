"""GPU: Matrix Market ingest and device build_coo against the reference library.

Mirrors proj/tests/test_io.cpp; the reference's own read_matrix_market / build_coo /
write_matrix_market (oracle/_ref) are the checker: same canonical COO bit for bit, same
exception class, message and line number for every malformed input, byte-identical files.
"""
import numpy as np
import pytest

import paper_2108_13162_b200 as kg

pytestmark = pytest.mark.gpu

WORKED = ("%%MatrixMarket matrix coordinate real general\n"
          "% the 5x5 worked example\n"
          "5 5 11\n"
          "1 1 -5\n1 2 14\n2 2 8\n2 3 1\n3 1 2\n3 3 10\n4 2 4\n4 4 2\n4 5 9\n5 3 15\n5 5 7\n")

H = "%%MatrixMarket matrix coordinate real general\n"
CASES = {
    "worked": WORKED,
    "symmetric": "%%MatrixMarket matrix coordinate real symmetric\n2 2 3\n1 1 2\n2 1 -1\n2 2 3\n",
    "integer": "%%MatrixMarket matrix coordinate integer general\n1 1 1\n1 1 7\n",
    "upper_banner_words": "%%MatrixMarket MATRIX Coordinate REAL General\n2 2 1\n2 2 1.5\n",
    "comments_blank": H + "% c\n\n  \n2 3 2\n% mid\n\n1 3 1e-3\n  2 1   -2.5e+2  trailing words\n",
    "crlf": H.replace("\n", "\r\n") + "2 2 2\r\n1 1 1.0\r\n2 2 2.0\r\n",
    "extra_lines_ignored": H + "2 2 1\n1 1 1.0\nthis is not an entry\n9 9 9\n",
    "duplicates": H + "3 3 5\n1 1 1.0\n1 1 2.0\n3 2 0.5\n2 2 1.0\n3 2 0.25\n",
    "signs_exponents": H + "2 2 3\n+1 +2 -.5\n2 1 5.\n2 2 1E3\n",
    "value_prefix": H + "2 2 1\n1 1 2.5abc\n",
    "zero_entries": H + "4 3 0\n",
    "empty": "",
    "no_banner": "5 5 0\n",
    "array": "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n",
    "pattern": "%%MatrixMarket matrix coordinate pattern general\n2 2 1\n1 1\n",
    "complex": "%%MatrixMarket matrix coordinate complex general\n2 2 1\n1 1 1.0 0.0\n",
    "unknown_field": "%%MatrixMarket matrix coordinate quaternion general\n2 2 1\n1 1 1\n",
    "skew": "%%MatrixMarket matrix coordinate real skew-symmetric\n2 2 1\n2 1 1\n",
    "no_size": H + "% only a comment\n",
    "bad_size": H + "2 x 2\n",
    "negative_size": H + "2 -2 2\n",
    "truncated": H + "2 2 2\n1 1 1.0\n",
    "malformed": H + "2 2 1\n1 x 1.0\n",
    "missing_value": H + "2 2 2\n1 1 1.0\n2 2\n",
    "out_of_range": H + "2 2 2\n1 1 1.0\n3 1 1.0\n",
    "zero_index": H + "2 2 1\n0 1 1.0\n",
    "inf_value": H + "2 2 1\n1 1 inf\n",
}


def coo_arrays(A):
    m = A.to_host()
    return m.row_idx, m.col_idx, m.values


@pytest.mark.parametrize("name", sorted(CASES))
def test_parse_matches_reference(ctx, ref, name):
    text = CASES[name]
    want, rc, msg, line = ref.parse_matrix_market(text)
    if rc:
        with pytest.raises(kg.Error) as ei:
            ctx.parse_matrix_market(text)
        assert ei.value.code == rc and str(ei.value) == msg
        if rc == kg.ParseError.code:
            assert ei.value.line_number == line
        return
    A = ctx.parse_matrix_market(text, fmt="coo")
    r, c, v = ref.get_coo(want)
    gr, gc, gv = coo_arrays(A)
    np.testing.assert_array_equal(gr, r)
    np.testing.assert_array_equal(gc, c)
    np.testing.assert_array_equal(gv, v)


def test_worked_example_csr(ctx, port):
    A = ctx.parse_matrix_market(WORKED, fmt="csr")
    m = A.to_host()
    np.testing.assert_array_equal(m.row_ptr, [0, 2, 4, 6, 9, 11])
    np.testing.assert_array_equal(m.values, [-5, 14, 8, 1, 2, 10, 4, 2, 9, 15, 7])


def big_text(rng, n, nnz, symmetric=False, dup=True):
    r = rng.integers(1, n + 1, nnz)
    c = rng.integers(1, n + 1, nnz)
    if symmetric:
        r, c = np.maximum(r, c), np.minimum(r, c)
    if dup:  # every key at most twice: a + b == b + a, so any sort order sums identically
        k = r * (n + 1) + c
        _, first = np.unique(k, return_index=True)
        keep = np.zeros(nnz, bool)
        keep[first] = True
        dupl = np.flatnonzero(~keep)
        seen2 = np.unique(k[dupl], return_index=True)[1]
        keep[dupl[seen2]] = True
        r, c = r[keep], c[keep]
    v = rng.standard_normal(len(r)) * np.exp(rng.uniform(-30, 30, len(r)))
    lines = [f"%%MatrixMarket matrix coordinate real {'symmetric' if symmetric else 'general'}", f"{n} {n} {len(r)}"]
    body = "\n".join(f"{a} {b} {x:.17g}" for a, b, x in zip(r, c, v))
    return "\n".join(lines) + "\n" + body + "\n", len(r)


@pytest.mark.parametrize("symmetric", [False, True])
def test_large_file_multithreaded_parse(ctx, ref, tmp_path, symmetric):
    rng = np.random.default_rng(11 + symmetric)
    text, k = big_text(rng, 200_000, 600_000, symmetric)
    p = tmp_path / "big.mtx"
    p.write_text(text)
    A = ctx.read_matrix_market(str(p), fmt="coo")
    want, rc, _, _ = ref.parse_matrix_market(text)
    assert rc == 0
    r, c, v = ref.get_coo(want)
    gr, gc, gv = coo_arrays(A)
    np.testing.assert_array_equal(gr, r)
    np.testing.assert_array_equal(gc, c)
    np.testing.assert_array_equal(gv, v)
    # an error deep in a later chunk keeps the reference's line number
    lines = text.split("\n")
    lines[500_000] = "17 oops 1.0"
    bad = "\n".join(lines)
    _, rc, msg, line = ref.parse_matrix_market(bad)
    with pytest.raises(kg.ParseError) as ei:
        ctx.parse_matrix_market(bad)
    assert ei.value.line_number == line == 500_001 and str(ei.value) == msg


def test_build_coo_device(ctx, ref):
    rng = np.random.default_rng(5)
    n, nnz = 3000, 40_000
    r = rng.integers(0, n, nnz)
    c = rng.integers(0, n, nnz)
    v = rng.standard_normal(nnz)
    A = ctx.build_coo(n, n, r, c, v, fmt="coo")
    W = ref.build_coo(n, n, r, c, v)
    wr, wc, wv = ref.get_coo(W)
    gr, gc, gv = coo_arrays(A)
    np.testing.assert_array_equal(gr, wr)
    np.testing.assert_array_equal(gc, wc)
    np.testing.assert_allclose(gv, wv, rtol=1e-14, atol=1e-15)  # >2 duplicates: sum order may differ
    csr = ctx.build_coo(n, n, r, c, v, fmt="csr").to_host()
    np.testing.assert_array_equal(csr.col_idx, wc)
    np.testing.assert_array_equal(csr.row_ptr, np.concatenate([[0], np.cumsum(np.bincount(wr, minlength=n))]))
    # the first offending triple is named, as the reference does
    r2 = r.copy()
    r2[[100, 7]] = [n + 5, -1]
    with pytest.raises(kg.IndexOutOfRange) as ei:
        ctx.build_coo(n, n, r2, c, v)
    with pytest.raises(Exception) as er:
        ref.build_coo(n, n, r2, c, v)
    assert er.value.code == kg.IndexOutOfRange.code
    assert str(er.value) == f"[{er.value.code}] {ei.value}"


def test_write_read_round_trip_and_bytes(ctx, ref, tmp_path):
    r = np.array([0, 0, 1, 2, 2])
    c = np.array([0, 2, 1, 0, 2])
    v = np.array([1.0 / 3.0, -7.125e-300, 6.02214076e23, -0.1, 1e-17])
    A = ctx.build_coo(3, 3, r, c, v)
    p1, p2 = tmp_path / "ours.mtx", tmp_path / "ref.mtx"
    A.write_matrix_market(str(p1))
    ref.write_matrix_market(ref.build_coo(3, 3, r, c, v), str(p2))
    assert p1.read_bytes() == p2.read_bytes()
    back = coo_arrays(ctx.read_matrix_market(str(p1)))
    np.testing.assert_array_equal(back[2], v)
    # generated matrices round trip through files (csr source)
    G = ctx.generate("poisson2d", 7)
    G.write_matrix_market(str(p1))
    g = G.to_host()
    back = ctx.read_matrix_market(str(p1), fmt="csr").to_host()
    np.testing.assert_array_equal(back.row_ptr, g.row_ptr)
    np.testing.assert_array_equal(back.col_idx, g.col_idx)
    np.testing.assert_array_equal(back.values, g.values)
