"""The oracle (oracle/sf_oracle.c) pinned against the reference's own outputs
(tests/golden, produced by the unmodified reference) and known answers from
the reference's test-suite (proj/tests/*.cpp)."""
import numpy as np
import pytest

from conftest import GOLDEN_MATS, golden_matrix
from oracle.oracle import Csc, FactorizationError, Reference

ALL_COMBOS = (1, 2, 3, 4, 5, 6, 7)


def csc_from_dense(D):
    D = np.asarray(D, float)
    n = D.shape[0]
    cp, ri, va = [0], [], []
    for j in range(n):
        for i in range(n):
            if D[i, j] != 0.0:
                ri.append(i)
                va.append(D[i, j])
        cp.append(len(ri))
    return Csc(n, np.array(cp, np.int32), np.array(ri, np.int32), np.array(va, float))


def test_gen_vector_known_answer(orc, golden):
    # SURVEY.md 7 step 1 known answer, reproduced by the reference itself
    want = [0.50877060830571597, 0.89860240578528838, -0.76517143793096376,
            0.78382635342495277]
    assert np.array_equal(golden["gen_vector_4_7"], want)
    assert np.array_equal(orc.gen_vector(4, 7), want)
    assert np.array_equal(orc.gen_vector(1000, 123), golden["gen_vector_1000_123"])


@pytest.mark.parametrize("name", GOLDEN_MATS)
@pytest.mark.parametrize("combo", ALL_COMBOS + (8,))
def test_outputs_bit_exact_vs_reference(orc, golden, name, combo):
    M = golden_matrix(golden, name)
    got = orc.run_sequential(combo, M, 7)
    assert np.array_equal(got, golden[f"{name}/c{combo}/outputs"])


@pytest.mark.parametrize("name", GOLDEN_MATS)
@pytest.mark.parametrize("combo", ALL_COMBOS)
def test_dags_levels_reuse_vs_reference(orc, golden, name, combo):
    M = golden_matrix(golden, name)
    key = f"{name}/c{combo}"
    g = {}
    for which in (1, 2):
        g[which] = orc.build_g(combo, which, M)
        assert np.array_equal(g[which].succptr, golden[f"{key}/g{which}_succptr"])
        assert np.array_equal(g[which].succ, golden[f"{key}/g{which}_succ"])
        assert np.array_equal(g[which].cost, golden[f"{key}/g{which}_cost"])
        li = orc.level_info(g[which])
        assert np.array_equal(li.level, golden[f"{key}/g{which}_level"])
        assert li.critical_path == golden[f"{key}/g{which}_P"][0]
    f = orc.inter_dag(combo, M)
    assert np.array_equal(f.rowptr, golden[f"{key}/f_rowptr"])
    assert np.array_equal(f.colidx, golden[f"{key}/f_colidx"])
    j = orc.joint_dag(g[1], g[2], f)
    assert np.array_equal(j.succptr, golden[f"{key}/j_succptr"])
    assert np.array_equal(j.succ, golden[f"{key}/j_succ"])
    assert np.array_equal(j.cost, golden[f"{key}/j_cost"])
    lj = orc.level_info(j)
    assert np.array_equal(lj.level, golden[f"{key}/j_level"])
    assert np.array_equal(lj.height, golden[f"{key}/j_height"])
    assert np.array_equal(lj.slack, golden[f"{key}/j_slack"])
    assert lj.critical_path == golden[f"{key}/j_P"][0]
    assert orc.compute_reuse(combo, M) == golden[f"{key}/reuse"][0]


def test_fixture11_levels(orc, golden):
    # test_dag.cpp:48-55: P = 6, l(3) = 4, l(9) = 5, l(10) = 6
    M = golden_matrix(golden, "fixture11")
    li = orc.level_info(orc.build_g(1, 1, M))
    assert li.critical_path == 6
    assert li.level[3] == 4 and li.level[9] == 5 and li.level[10] == 6


def test_breakdown_index(orc, golden):
    # test_executor.cpp:157-171: IC0 hits a non-positive pivot at column 7
    cp = golden["breakdown/colptr"]
    M = Csc(len(cp) - 1, cp, golden["breakdown/rowidx"], golden["breakdown/values"])
    with pytest.raises(FactorizationError) as e:
        orc.run_sequential(5, M, 1)
    assert e.value.index == golden["breakdown/c5_index"][0] == 7


def test_frozen_examples(orc):
    # test_kernels.cpp:111-119 SpTRSV [[2,0,0],[1,3,0],[0,4,5]] x = [2,4,9] -> 1
    L = csc_from_dense([[2, 0, 0], [1, 3, 0], [0, 4, 5]])
    out = orc.run_sequential(1, L, 7, vin=np.array([2.0, 4.0, 9.0]))
    assert np.allclose(out[:3], 1.0, rtol=0, atol=1e-14)
    # test_kernels.cpp:149-154 IC0 diag(4, 9) -> diag(2, 3)
    out = orc.run_sequential(5, csc_from_dense([[4, 0], [0, 9]]), 7)
    assert list(out[:2]) == [2.0, 3.0]
    # test_kernels.cpp:155-159 tridiagonal: L00 = sqrt(2)
    T = csc_from_dense([[2, -1, 0], [-1, 2, -1], [0, -1, 2]])
    out = orc.run_sequential(5, T, 7)
    assert out[0] == pytest.approx(np.sqrt(2.0), rel=1e-14)
    # test_kernels.cpp:214-223 ILU0 of the tridiagonal = exact LU
    out = orc.run_sequential(6, T, 7)
    assert np.allclose(out[:7], [2, -1, -0.5, 1.5, -1, -2 / 3, 4 / 3], rtol=1e-14)
    # test_kernels.cpp:170-178 negative pivot reported with its column
    with pytest.raises(FactorizationError) as e:
        orc.run_sequential(5, csc_from_dense([[-1, 0], [0, 4]]), 7)
    assert e.value.index == 0
    # test_kernels.cpp:225-236 zero pivot reported with the pivot row
    with pytest.raises(FactorizationError) as e:
        orc.run_sequential(6, csc_from_dense([[0, 1], [1, 0]]), 7)
    assert e.value.index == 0
    # test_kernels.cpp:288-296 DSCAL [[4,2],[2,9]] -> [[1,1/3],[1/3,1]], then IC0
    out = orc.run_sequential(7, csc_from_dense([[4, 2], [2, 9]]), 7)
    fac, d = out[:3], out[3:]
    assert np.allclose(d, [0.5, 1 / 3], rtol=1e-15)
    assert fac[0] == pytest.approx(1.0) and fac[1] == pytest.approx(1 / 3)
    assert fac[2] == pytest.approx(np.sqrt(1 - 1 / 9))


def test_combo8_backward_vs_dense(orc, golden):
    for name in GOLDEN_MATS:
        M = golden_matrix(golden, name)
        out = orc.run_sequential(8, M, 7)
        n = M.n
        D = np.zeros((n, n))
        for j in range(n):
            for p in range(M.colptr[j], M.colptr[j + 1]):
                if M.rowidx[p] >= j:
                    D[M.rowidx[p], j] = M.values[p]
        z = np.linalg.solve(D, orc.gen_vector(n, 7))
        x = np.linalg.solve(D.T, out[:n])
        assert np.max(np.abs(out[:n] - z)) <= 1e-12 * max(1, np.abs(z).max())
        assert np.max(np.abs(out[n:] - x)) <= 1e-12 * max(1, np.abs(x).max())


@pytest.mark.skipif(not Reference.available(), reason="reference tree not built here")
@pytest.mark.parametrize("seed", range(1, 9))
def test_random_sweep_vs_live_reference(orc, seed):
    # dense-oracle style sweep (test_kernels.cpp:416-509) against the live reference
    ref = Reference()
    M = ref.gen_banded_spd(10 + 3 * seed, 1 + seed % 4, seed * 13)
    for combo in ALL_COMBOS:
        want = ref.state(combo, M, seed).execute(0)
        assert np.array_equal(orc.run_sequential(combo, M, seed), want)


@pytest.mark.skipif(not Reference.available(), reason="reference tree not built here")
def test_reference_partitioning_validator_is_discriminating(golden):
    # the validator the GPU schedule is checked with (msp.hpp:1108-1237)
    # accepts a level-ordered partitioning and rejects a reversed one
    from conftest import golden_matrix
    Mo = golden_matrix(golden, "grid6")
    ref = Reference()
    rs = ref.state(1, Mo, 7)
    tags, iters, lp = rs.wavefront()
    # one w-partition per entry, one s-partition per wavefront level
    s_ptr = np.asarray(lp, np.int64)
    w_ptr = np.arange(len(tags) + 1, dtype=np.int64)
    nbad, msg = rs.validate_partitioning(s_ptr, w_ptr, tags, iters)
    assert nbad == 0, msg
    nbad, msg = rs.validate_partitioning(np.array([0, 1]), np.array([0, len(tags)]),
                                         tags[::-1], iters[::-1])
    assert nbad > 0 and "unsatisfied" in msg


needs_ref = pytest.mark.skipif(not Reference.available(), reason="oracle/_ref not built")


@needs_ref
@pytest.mark.parametrize("case", ("cfg5_16", "banded", "grid", "irregular"))
def test_combo8_vs_reference_primitives(orc, case):
    """Combo 8 (fwd L, bwd L^T) restated by the oracle equals the reference's
    primitives composed as SURVEY.md 8(c) prescribes -- sptrsv on L, then on
    permute_symmetric(transpose(L), rev) -- bit for bit, beyond the golden
    matrices: C5's 27-point stencil (8 systems), banded, grid and an irregular
    random pattern."""
    ref = Reference()
    if case == "cfg5_16":
        M, vals = ref.config_matrix(5, 16, nsys_perturb=8)
        systems = [Csc(M.n, M.colptr, M.rowidx, vals[s * M.nnz:(s + 1) * M.nnz]) for s in range(8)]
    elif case == "banded":
        systems = [ref.gen_banded_spd(3000, 40, 5)]
    elif case == "grid":
        systems = [ref.gen_grid_laplacian(40)]
    else:
        rng = np.random.default_rng(3)
        n = 1500
        D = np.zeros((n, n))
        for i in range(n):
            js = rng.integers(0, i + 1, size=rng.integers(0, 12))
            D[i, js] = rng.uniform(-1, 0, size=len(js))
            D[i, i] = 4.0 + rng.uniform(0, 1)
        systems = [csc_from_dense(np.tril(D) + np.tril(D, -1).T)]
    for s, Ms in enumerate(systems):
        b = ref.gen_vector(Ms.n, 7 + s)
        assert np.array_equal(orc.run_sequential(8, Ms, 7, vin=b), ref.fwd_bwd(Ms, b))


@needs_ref
@pytest.mark.parametrize("cfg", (1, 2, 3, 4, 5))
def test_reference_arm_inputs_equal_the_packages(cfg):
    """bench.py's reference arm generates its inputs from oracle/_ref (the
    repo's fixtures.cpp compiled in under renamed symbols), never from
    libsfgpu.so; they must be the very inputs our arm uses."""
    import paper_2111_12238_b200 as sf
    ref = Reference()
    size = {1: 40, 2: 10, 3: 9, 4: 5000, 5: 12}[cfg]
    A, B = ref.config_matrix(cfg, size), sf.config_matrix(cfg, size=size)
    assert np.array_equal(A.colptr, B.colptr) and np.array_equal(A.rowidx, B.rowidx)
    assert np.array_equal(A.values, B.values)
    if cfg == 5:
        _, v1 = ref.config_matrix(5, size, nsys_perturb=8, seed0=1004)
        _, v2 = sf.config5_systems(size=size, nsys=8, seed0=1004)
        assert np.array_equal(v1, v2)
