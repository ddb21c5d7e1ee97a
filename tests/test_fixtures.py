"""Product-side generators (paper_2111_12238_b200 fixtures, host C++) against
the reference's own generator outputs (tests/golden) and the BASELINE.json
configuration shapes."""
import numpy as np
import pytest

import paper_2111_12238_b200 as sf
from conftest import golden_matrix


def test_gen_vector_matches_reference(golden):
    assert np.array_equal(sf.gen_vector(4, 7), golden["gen_vector_4_7"])
    assert np.array_equal(sf.gen_vector(1000, 123), golden["gen_vector_1000_123"])


@pytest.mark.parametrize("name,make", [
    ("banded24", lambda: sf.gen_banded_spd(24, 3, 11)),
    ("banded40", lambda: sf.gen_banded_spd(40, 5, 3)),
    ("grid6", lambda: sf.gen_grid_laplacian(6)),
    ("grid10", lambda: sf.gen_grid_laplacian(10)),
])
def test_generators_match_reference(golden, name, make):
    M = make()
    G = golden_matrix(golden, name)
    assert np.array_equal(M.colptr, G.colptr)
    assert np.array_equal(M.rowidx, G.rowidx)
    assert np.array_equal(M.values, G.values)


def _dense(M):
    D = np.zeros((M.n, M.n))
    for j in range(M.n):
        D[M.rowidx[M.colptr[j]:M.colptr[j + 1]], j] = M.values[M.colptr[j]:M.colptr[j + 1]]
    return D


def _check_csc(M):
    assert M.colptr[0] == 0 and np.all(np.diff(M.colptr) >= 0)
    for j in range(M.n):
        r = M.rowidx[M.colptr[j]:M.colptr[j + 1]]
        assert np.all(np.diff(r) > 0) and j in r


@pytest.mark.parametrize("cfg,size", [(1, 7), (2, 5), (3, 5), (4, 300), (5, 5)])
def test_config_shapes_small(cfg, size):
    M = sf.config_matrix(cfg, size=size, halfwidth=20) if cfg == 4 else sf.config_matrix(cfg, size=size)
    _check_csc(M)
    D = _dense(M)
    assert np.array_equal(D != 0, (D != 0).T)  # symmetric pattern
    off = np.abs(D).sum(axis=1) - np.abs(np.diag(D))
    if cfg == 1:
        assert set(np.unique(D)) <= {-1.0, 0.0, 4.0}
    if cfg == 2:
        assert np.all(np.diag(D) == 6.01)
    if cfg == 3:
        assert np.allclose(np.diag(D), off + 0.1)
        L, U = np.tril(D, -1), np.triu(D, 1)
        lo, up = L[L != 0], U.T[U.T != 0]
        assert np.all((lo <= -1.0) & (lo >= -1.5)) and np.all((up >= -1.0) & (up <= -0.5))
    if cfg == 4:
        assert np.allclose(D, D.T) and np.allclose(np.diag(D), off + 1.0)
        assert np.all(D[~np.eye(M.n, dtype=bool)] <= 0)
        i, j = np.nonzero(D)
        assert np.max(np.abs(i - j)) <= 20
    if cfg == 5:
        assert np.all(np.diag(D) == 26.5) and set(np.unique(D)) <= {-1.0, 0.0, 26.5}


def test_config_full_sizes():
    # BASELINE.json configs: n and nnz at full size
    assert (lambda M: (M.n, M.nnz))(sf.config_matrix(1)) == (262_144, 1_308_672)
    assert (lambda M: (M.n, M.nnz))(sf.config_matrix(2)) == (262_144, 1_810_432)
    assert (lambda M: (M.n, M.nnz))(sf.config_matrix(3)) == (884_736, 6_137_856)
    M = sf.config_matrix(4)
    assert M.n == 1_000_000 and 16.5 < M.nnz / M.n < 17.5  # ~16 nnz/row + diagonal


def test_config5_systems_perturbation():
    M, vals = sf.config5_systems(size=6, nsys=3)
    assert vals.shape == (3 * M.nnz,)
    V = vals.reshape(3, M.nnz)
    diag = np.zeros(M.nnz, bool)
    for j in range(M.n):
        for p in range(M.colptr[j], M.colptr[j + 1]):
            diag[p] = M.rowidx[p] == j
    for s in range(3):
        d = V[s][diag] - M.values[diag]
        assert np.all((d >= 0) & (d < 0.1)) and np.array_equal(V[s][~diag], M.values[~diag])
    assert not np.array_equal(V[0], V[1])
