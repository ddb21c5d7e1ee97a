"""Matrix Market ingest and symmetric permutation (matrix_market.hpp:59-152,
matrix.hpp:135-173), checked against the compiled reference's own readers
where available and against known answers.  CPU only: file input is host
work in the reference too."""
import numpy as np
import pytest

import paper_2111_12238_b200 as sf


def _write(tmp_path, name, text):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


def test_symmetric_expansion_and_duplicates(tmp_path):
    path = _write(tmp_path, "a.mtx", """%%MatrixMarket matrix coordinate real symmetric
% comment
3 3 5
1 1 4.0
2 1 -1.0
2 2 4.0
3 3 4.0
2 1 -0.5
""")
    M = sf.read_matrix_market(path)
    D = np.zeros((3, 3))
    for j in range(3):
        for p in range(M.colptr[j], M.colptr[j + 1]):
            D[M.rowidx[p], j] = M.values[p]
    assert np.array_equal(D, np.array([[4.0, -1.5, 0], [-1.5, 4.0, 0], [0, 0, 4.0]]))


@pytest.mark.parametrize("text,err", [
    ("%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n", "coordinate"),
    ("%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n", "complex"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n", "out of bounds"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n", "end of file"),
    ("nothing\n", "banner"),
])
def test_parse_errors(tmp_path, text, err):
    with pytest.raises(sf.ParseError, match=err):
        sf.read_matrix_market(_write(tmp_path, "bad.mtx", text))


def test_round_trip_bit_exact(tmp_path):
    M = sf.config_matrix(3, size=6)  # nonsymmetric values
    path = str(tmp_path / "rt.mtx")
    sf.write_matrix_market(M, path)
    R = sf.read_matrix_market(path)
    assert np.array_equal(R.colptr, M.colptr) and np.array_equal(R.rowidx, M.rowidx)
    assert np.array_equal(R.values, M.values)


def test_permutation_matches_dense(tmp_path):
    M = sf.config_matrix(1, size=5)
    rng = np.random.default_rng(4)
    perm = rng.permutation(M.n).astype(np.int32)
    B = sf.permute_symmetric(M, perm)
    A = np.zeros((M.n, M.n))
    for j in range(M.n):
        for p in range(M.colptr[j], M.colptr[j + 1]):
            A[M.rowidx[p], j] = M.values[p]
    P = np.zeros((M.n, M.n))
    P[perm, np.arange(M.n)] = 1.0  # row/col i -> perm[i]
    Bd = np.zeros((M.n, M.n))
    for j in range(B.n):
        for p in range(B.colptr[j], B.colptr[j + 1]):
            Bd[B.rowidx[p], j] = B.values[p]
    assert np.array_equal(Bd, P @ A @ P.T)
    path = _write(tmp_path, "perm.txt", "\n".join(str(v) for v in perm) + "\n")
    assert np.array_equal(sf.read_permutation(path, M.n), perm)
    with pytest.raises(sf.InvalidMatrixError):
        sf.permute_symmetric(M, np.zeros(M.n, np.int32))


def test_reference_reader_agrees(tmp_path):
    # the same files through the compiled reference's read_matrix_market
    from oracle.oracle import Reference
    if not Reference.available():
        pytest.skip("reference tree not built here")
    ref = Reference()
    rng = np.random.default_rng(9)
    lines = ["%%MatrixMarket matrix coordinate real symmetric", "% random, with duplicates"]
    ent = []
    for _ in range(60):
        i, j = sorted(rng.integers(1, 21, 2))[::-1]
        ent.append(f"{i} {j} {rng.uniform(-1, 1):.17g}")
    lines.append(f"20 20 {len(ent)}")
    path = _write(tmp_path, "r.mtx", "\n".join(lines + ent) + "\n")
    M = sf.config_matrix(2, size=5)
    path2 = str(tmp_path / "g.mtx")
    sf.write_matrix_market(M, path2)
    for p in (path, path2):
        got, want = sf.read_matrix_market(p), ref.read_matrix_market(p)
        assert np.array_equal(got.colptr, want.colptr) and np.array_equal(got.rowidx, want.rowidx)
        assert np.array_equal(got.values, want.values)
