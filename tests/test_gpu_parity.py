"""CUDA path (libsfgpu.so through the C-ABI) against the reference.

* golden cases: outputs, DAGs, F, joint DAG, levels and reuse produced by the
  unmodified reference (tests/golden) -- compared bit for bit;
* BASELINE.json configurations at full size: compared with the oracle
  (oracle/sf_oracle.c, itself pinned to the reference by test_oracle.py) on
  the same seeded inputs -- bit for bit, and the north_star tolerance
  (max relative error 1e-10) plus solve residuals as a second line;
* error behaviour (FactorizationError index), idempotence, fused vs unfused,
  and the schedule being a linear extension of the joint DAG.
"""
import numpy as np
import pytest

import paper_2111_12238_b200 as sf
from conftest import GOLDEN_MATS, golden_matrix
from oracle.oracle import Csc

pytestmark = pytest.mark.gpu

GPU_COMBOS = (1, 2, 3, 4, 5, 6, 7, 8)
TOL = 1e-10  # north_star: fp64 values within max-relative-error 1e-10


def as_sf(M) -> sf.CscMatrix:
    return sf.CscMatrix(M.n, M.colptr, M.rowidx, M.values)


def max_rel(got, want):
    scale = max(1.0, float(np.max(np.abs(want)))) if want.size else 1.0
    return float(np.max(np.abs(got - want))) / scale if want.size else 0.0


@pytest.fixture(scope="module", autouse=True)
def _device():
    from paper_2111_12238_b200 import abi
    assert abi.device_available(), "B200 required: the -m gpu suite never skips"


@pytest.mark.parametrize("name", GOLDEN_MATS)
@pytest.mark.parametrize("combo", GPU_COMBOS)
def test_golden_outputs_fused_and_unfused(golden, name, combo):
    M = as_sf(golden_matrix(golden, name))
    want = golden[f"{name}/c{combo}/outputs"]
    st = sf.make_state(combo, M, seed=7)
    sched = sf.make_fused_schedule(st)
    sf.execute_fused(sched, st)
    assert np.array_equal(sf.collect_outputs(st), want)
    st.execute_unfused()
    assert np.array_equal(st.collect_outputs(), want)
    # idempotent re-execution (reset semantics, kernels.hpp:497-502)
    st.execute_fused()
    assert np.array_equal(st.collect_outputs(), want)


@pytest.mark.parametrize("name", GOLDEN_MATS)
@pytest.mark.parametrize("combo", (1, 2, 3, 4, 5, 6, 7))
def test_golden_dags_levels(golden, name, combo):
    M = as_sf(golden_matrix(golden, name))
    key = f"{name}/c{combo}"
    st = sf.make_state(combo, M)
    for which in (1, 2):
        g = st.dag(which)
        assert np.array_equal(g.succptr, golden[f"{key}/g{which}_succptr"])
        assert np.array_equal(g.succ, golden[f"{key}/g{which}_succ"])
        assert np.array_equal(g.cost, golden[f"{key}/g{which}_cost"])
        li = st.level_info(which)
        assert np.array_equal(li.level, golden[f"{key}/g{which}_level"])
        assert li.critical_path == golden[f"{key}/g{which}_P"][0]
    f = sf.inter_dag(st)
    assert np.array_equal(f.rowptr, golden[f"{key}/f_rowptr"])
    assert np.array_equal(f.colidx, golden[f"{key}/f_colidx"])
    j = sf.joint_dag(st)
    assert np.array_equal(j.succptr, golden[f"{key}/j_succptr"])
    assert np.array_equal(j.succ, golden[f"{key}/j_succ"])
    assert np.array_equal(j.cost, golden[f"{key}/j_cost"])
    lj = sf.level_info(st, 3)
    assert np.array_equal(lj.level, golden[f"{key}/j_level"])
    assert np.array_equal(lj.height, golden[f"{key}/j_height"])
    assert np.array_equal(lj.slack, golden[f"{key}/j_slack"])
    assert lj.critical_path == golden[f"{key}/j_P"][0]
    assert sf.compute_reuse(st) == golden[f"{key}/reuse"][0]


def _check_linear_extension(st, joint):
    """Every joint-DAG edge u -> v is scheduled with u before v."""
    sch = st.schedule()
    n = st.n
    pos = np.empty(2 * n, np.int64)
    ids = np.where(sch.tags == 1, sch.iters, n + sch.iters)
    assert np.array_equal(np.sort(ids), np.arange(2 * n))
    pos[ids] = np.arange(len(ids))
    src = np.repeat(np.arange(joint.nvert), np.diff(joint.succptr))
    assert np.all(pos[src] < pos[joint.succ])
    assert sch.wave_ptr[0] == 0 and sch.wave_ptr[-1] == len(ids)


@pytest.mark.parametrize("name", GOLDEN_MATS)
@pytest.mark.parametrize("combo", (1, 2, 3, 4, 5, 6, 7))
def test_schedule_is_linear_extension(golden, name, combo):
    M = as_sf(golden_matrix(golden, name))
    st = sf.make_state(combo, M).inspect()
    _check_linear_extension(st, st.dag(3))


@pytest.mark.parametrize("name", GOLDEN_MATS)
def test_combo8_structures_vs_oracle(orc, golden, name):
    Mo = golden_matrix(golden, name)
    st = sf.make_state(8, as_sf(Mo)).inspect()
    for which in (1, 2):
        g, w = st.dag(which), orc.build_g(8, which, Mo)
        assert np.array_equal(g.succptr, w.succptr) and np.array_equal(g.succ, w.succ)
        assert np.array_equal(g.cost, w.cost)
    f, w = st.inter_dag(), orc.inter_dag(8, Mo)
    assert np.array_equal(f.rowptr, w.rowptr) and np.array_equal(f.colidx, w.colidx)
    j = st.dag(3)
    wj = orc.joint_dag(orc.build_g(8, 1, Mo), orc.build_g(8, 2, Mo), w)
    assert np.array_equal(j.succptr, wj.succptr) and np.array_equal(j.succ, wj.succ)
    lj, wl = st.level_info(3), orc.level_info(wj)
    assert np.array_equal(lj.level, wl.level) and np.array_equal(lj.height, wl.height)
    _check_linear_extension(st, j)


def test_breakdown_reports_reference_index(golden):
    cp = golden["breakdown/colptr"]
    M = sf.CscMatrix(len(cp) - 1, cp, golden["breakdown/rowidx"], golden["breakdown/values"])
    st = sf.make_state(5, M, seed=1)
    with pytest.raises(sf.FactorizationError) as e:
        st.execute_fused()
    assert e.value.index == golden["breakdown/c5_index"][0] == 7
    assert "non-positive pivot" in str(e.value)
    with pytest.raises(sf.FactorizationError):
        st.execute_unfused()


@pytest.mark.parametrize("combo", (1, 4, 8))
def test_zero_diagonal_solve_error(orc, combo):
    # a zero diagonal is rejected by lower_triangle (matrix.hpp:106-112)
    M = sf.config_matrix(1, size=6)
    vals = M.values.copy()
    j = 9
    p = M.colptr[j] + list(M.rowidx[M.colptr[j]:M.colptr[j + 1]]).index(j)
    vals[p] = 0.0
    with pytest.raises(sf.InvalidMatrixError, match="zero diagonal entry at column 9"):
        sf.make_state(combo, sf.CscMatrix(M.n, M.colptr, M.rowidx, vals))


def test_combo3_zero_diagonal_is_factorization_error(orc):
    # scaling_vector throws from make_state (kernels.hpp:299-309)
    M = sf.config_matrix(3, size=6)
    vals = M.values.copy()
    j = 11
    p = M.colptr[j] + list(M.rowidx[M.colptr[j]:M.colptr[j + 1]]).index(j)
    vals[p] = 0.0
    Mo = Csc(M.n, M.colptr, M.rowidx, vals)
    from oracle.oracle import FactorizationError as OFE
    with pytest.raises(OFE) as want:
        orc.run_sequential(3, Mo, 7)
    with pytest.raises(sf.FactorizationError) as got:
        sf.make_state(3, as_sf(Mo))
    assert got.value.index == want.value.index == 11
    assert "zero diagonal" in str(got.value)


@pytest.mark.parametrize("combo", (2, 3))
def test_combos_2_3_full_size_vs_oracle(orc, combo):
    # the reference's remaining Table-2 pairs on the BASELINE matrices
    M = sf.config_matrix(1 if combo == 2 else 3)
    Mo = Csc(M.n, M.colptr, M.rowidx, M.values)
    want = orc.run_sequential(combo, Mo, 7)
    st = sf.make_state(combo, M, seed=7)
    st.execute_fused()
    assert np.array_equal(st.collect_outputs(), want)
    st.execute_unfused()
    assert np.array_equal(st.collect_outputs(), want)


def test_ilu0_zero_pivot_index(orc):
    # row 3's pivot U_33 cancels to 0 -> "zero pivot" at the pivot row
    D = np.array([[2.0, 1, 0, 0, 0], [1, 2, 0, 0, 0], [0, 0, 1, 1, 0], [0, 0, 1, 1, 1],
                  [0, 0, 0, 1, 3]])
    cp, ri, va = [0], [], []
    for jj in range(5):
        for ii in range(5):
            if D[ii, jj] != 0:
                ri.append(ii)
                va.append(D[ii, jj])
        cp.append(len(ri))
    Mo = Csc(5, np.array(cp, np.int32), np.array(ri, np.int32), np.array(va))
    from oracle.oracle import FactorizationError as OFE
    with pytest.raises(OFE) as want:
        orc.run_sequential(6, Mo, 7)
    st = sf.make_state(6, as_sf(Mo))
    with pytest.raises(sf.FactorizationError) as got:
        st.execute_fused()
    assert got.value.index == want.value.index == 3
    assert "zero pivot" in str(got.value)


def test_multisystem_golden(golden, orc):
    # nsys systems with distinct values/vectors: each equals its own oracle run
    for name in ("banded40", "grid10"):
        Mo = golden_matrix(golden, name)
        nsys = 4
        rng = np.random.default_rng(3)
        vals = np.concatenate([Mo.values * (1 + 0.01 * s) for s in range(nsys)])
        vin = rng.uniform(-1, 1, nsys * Mo.n)
        for combo in (1, 8):
            st = sf.make_state(combo, as_sf(Mo), nsys=nsys, values=vals, vin=vin)
            st.execute_fused()
            got = st.collect_outputs().reshape(nsys, -1)
            for s in range(nsys):
                Ms = Csc(Mo.n, Mo.colptr, Mo.rowidx, vals[s * Mo.nnz:(s + 1) * Mo.nnz])
                want = orc.run_sequential(combo, Ms, 7, vin=vin[s * Mo.n:(s + 1) * Mo.n])
                assert np.array_equal(got[s], want)


# ---- BASELINE.json configurations at full size --------------------------------
CONFIG_COMBO = {1: 4, 2: 5, 3: 6, 4: 7}


@pytest.mark.parametrize("cfg", (1, 2, 3, 4))
def test_config_full_size_vs_oracle(orc, cfg):
    M = sf.config_matrix(cfg)
    combo = CONFIG_COMBO[cfg]
    Mo = Csc(M.n, M.colptr, M.rowidx, M.values)
    want = orc.run_sequential(combo, Mo, 7)
    st = sf.make_state(combo, M, seed=7)
    st.execute_fused()
    got = st.collect_outputs()
    assert max_rel(got, want) <= TOL
    assert np.array_equal(got, want)  # bit-exact: same order, no FMA
    st.execute_unfused()
    assert np.array_equal(st.collect_outputs(), want)


def test_config5_batch_full_size(orc):
    nsys = 8
    M, vals = sf.config5_systems(nsys=nsys)
    n, nnz = M.n, M.nnz
    vin = np.concatenate([sf.gen_vector(n, 7 + s) for s in range(nsys)])
    for combo in (8, 1):
        st = sf.make_state(combo, M, nsys=nsys, values=vals, vin=vin)
        st.execute_fused()
        got = st.collect_outputs().reshape(nsys, 2 * n)
        for s in range(nsys):  # every system of the batch
            Ms = Csc(n, M.colptr, M.rowidx, vals[s * nnz:(s + 1) * nnz])
            want = orc.run_sequential(combo, Ms, 7, vin=vin[s * n:(s + 1) * n])
            assert max_rel(got[s], want) <= TOL
            assert np.array_equal(got[s], want)
        del st


# ---- inspector structures at the BASELINE sizes -----------------------------
def _same_dag(got, want):
    assert got.nvert == want.nvert
    assert np.array_equal(got.succptr, want.succptr)
    assert np.array_equal(got.succ, want.succ)
    assert np.array_equal(got.cost, want.cost)


def _structures_vs_oracle(orc, st, combo, Mo):
    """G1, G2, F, the joint DAG, level_info of all three (level, height,
    slack, critical path) and compute_reuse, bit for bit against the oracle
    (dag.hpp:150-431 restated in oracle/sf_oracle.c, pinned by test_oracle)."""
    w1, w2 = orc.build_g(combo, 1, Mo), orc.build_g(combo, 2, Mo)
    wf = orc.inter_dag(combo, Mo)
    _same_dag(st.dag(1), w1)
    _same_dag(st.dag(2), w2)
    f = st.inter_dag()
    assert np.array_equal(f.rowptr, wf.rowptr) and np.array_equal(f.colidx, wf.colidx)
    wj = orc.joint_dag(w1, w2, wf)
    _same_dag(st.dag(3), wj)
    for which, wg in ((1, w1), (2, w2), (3, wj)):
        li, wl = st.level_info(which), orc.level_info(wg)
        assert li.critical_path == wl.critical_path
        assert np.array_equal(li.level, wl.level)
        assert np.array_equal(li.height, wl.height)
        assert np.array_equal(li.slack, wl.slack)
    if combo != 8:  # the reference has no combo 8
        assert st.compute_reuse() == orc.compute_reuse(combo, Mo)
    # the joint level sets: ascending vertex id within a level
    # (build_wavefront_schedule, executor.hpp:209-229)
    ws = st.wavefront()
    lv = orc.level_info(wj).level
    order = np.lexsort((np.arange(len(lv)), lv))
    n = st.n
    assert np.array_equal(ws.tags, np.where(order < n, 1, 2))
    assert np.array_equal(ws.iters, np.where(order < n, order, order - n))
    assert np.array_equal(ws.level_ptr, np.concatenate([[0], np.cumsum(np.bincount(lv)[1:])]))


@pytest.mark.parametrize("cfg", (1, 2, 3, 4))
def test_config_structures_full_size(orc, cfg):
    M = sf.config_matrix(cfg)
    combo = CONFIG_COMBO[cfg]
    st = sf.make_state(combo, M, seed=7)
    _structures_vs_oracle(orc, st, combo, Csc(M.n, M.colptr, M.rowidx, M.values))


@pytest.mark.parametrize("combo", (1, 8))
def test_config5_structures_full_size(orc, combo):
    # C5's pattern: 27-point 128^3, 2,097,152 rows, 26.8 M edges per solve DAG
    M, vals = sf.config5_systems(nsys=1)
    st = sf.make_state(combo, M, nsys=1, values=vals)
    _structures_vs_oracle(orc, st, combo, Csc(M.n, M.colptr, M.rowidx, vals))


def test_config1_residuals():
    # ||L z - b||_inf / ||b||_inf (SPEC.md:132 bound 1e-12) and y = A z
    M = sf.config_matrix(1)
    st = sf.make_state(4, M, seed=7)
    st.execute_fused()
    out = st.collect_outputs()
    n = M.n
    z, y = out[:n], out[n:]
    b = sf.gen_vector(n, 7)
    import scipy.sparse as sp
    A = sp.csc_matrix((M.values, M.rowidx, M.colptr), shape=(n, n))
    L = sp.tril(A).tocsr()
    assert np.max(np.abs(L @ z - b)) <= 1e-12 * np.max(np.abs(b))
    assert np.max(np.abs(A @ z - y)) <= 1e-12 * max(1, np.max(np.abs(y)))


def test_division_from_reciprocal_is_ieee():
    # the executors divide with a reciprocal staged off the critical path;
    # it must equal IEEE division bit for bit
    import ctypes as C
    from paper_2111_12238_b200 import abi
    bad = C.c_int64(-1)
    fast = C.c_int64(0)
    n = 1 << 28
    assert abi.load().sfg_selftest_division(n, 12345, C.byref(bad), C.byref(fast)) == 0
    assert bad.value == 0
    assert fast.value > n // 10


@pytest.mark.parametrize("combo", GPU_COMBOS)
def test_set_values_refactorizes(orc, golden, combo):
    # new values, same pattern: equals a fresh state built on those values
    Mo = golden_matrix(golden, "grid10")
    st = sf.make_state(combo, as_sf(Mo), seed=7).inspect()
    st.execute_fused()
    v2 = Mo.values * 1.25
    st.set_values(v2)
    st.execute_fused()
    want = orc.run_sequential(combo, Csc(Mo.n, Mo.colptr, Mo.rowidx, v2), 7)
    assert np.array_equal(st.collect_outputs(), want)
    st.execute_unfused()
    assert np.array_equal(st.collect_outputs(), want)


def test_set_values_full_size_config4(orc):
    M = sf.config_matrix(4)
    st = sf.make_state(7, M, seed=7).inspect()
    v2 = M.values.copy()
    v2[M.rowidx == np.repeat(np.arange(M.n), np.diff(M.colptr))] *= 2.0  # heavier diagonal
    st.set_values(v2)
    st.execute_fused()
    want = orc.run_sequential(7, Csc(M.n, M.colptr, M.rowidx, v2), 7)
    assert np.array_equal(st.collect_outputs(), want)


@pytest.mark.parametrize("combo", (1, 5, 7, 8))
def test_set_values_zero_diagonal(golden, combo):
    Mo = golden_matrix(golden, "grid6")
    st = sf.make_state(combo, as_sf(Mo))
    v2 = Mo.values.copy()
    j = 4
    p = Mo.colptr[j] + list(Mo.rowidx[Mo.colptr[j]:Mo.colptr[j + 1]]).index(j)
    v2[p] = 0.0
    with pytest.raises(sf.InvalidMatrixError, match="zero diagonal entry at column 4"):
        st.set_values(v2)


# ---- alternative executors (SFG_EXECUTOR, read at sfg_inspect) -----------------
@pytest.mark.parametrize("executor", ("levels", "mline"))
@pytest.mark.parametrize("name", GOLDEN_MATS)
def test_alternative_executors_golden(golden, monkeypatch, executor, name):
    monkeypatch.setenv("SFG_EXECUTOR", executor)
    M = as_sf(golden_matrix(golden, name))
    for combo in (1, 8) if executor == "mline" else GPU_COMBOS:
        st = sf.make_state(combo, M, seed=7).inspect()
        st.execute_fused()
        if combo == 8:
            continue  # golden has no combo 8; covered against the oracle below
        assert np.array_equal(st.collect_outputs(), golden[f"{name}/c{combo}/outputs"])
        st.execute_unfused()
        assert np.array_equal(st.collect_outputs(), golden[f"{name}/c{combo}/outputs"])
        _check_linear_extension(st, st.dag(3))


@pytest.mark.parametrize("executor,nsys,rows", (("mline", 1, 0), ("mline", 2, 0), ("mline", 8, 0),
                                                 ("mline", 32, 0), ("chain", 1, 0), ("chain", 1, 1),
                                                 ("chain", 1, 8), ("chain", 2, 2), ("chain", 2, 16),
                                                 ("chain", 4, 8), ("chain", 8, 2), ("chain", 16, 0),
                                                 ("chain", 32, 0)))
def test_mline_executor_vs_oracle(orc, monkeypatch, executor, nsys, rows):
    """The 27-point grid through the multi-line and chain executors at every
    batch size, including non-default chain tile heights (SFG_CHAIN_G)."""
    monkeypatch.setenv("SFG_EXECUTOR", executor)
    if rows:
        monkeypatch.setenv("SFG_CHAIN_G", str(rows))
    M, vals = sf.config5_systems(size=24, nsys=nsys)
    n, nnz = M.n, M.nnz
    vin = np.concatenate([sf.gen_vector(n, 7 + s) for s in range(nsys)])
    for combo in (8, 1):
        st = sf.make_state(combo, M, nsys=nsys, values=vals, vin=vin)
        st.execute_fused()
        got = st.collect_outputs().reshape(nsys, 2 * n)
        for s in range(nsys):
            Ms = Csc(n, M.colptr, M.rowidx, vals[s * nnz:(s + 1) * nnz])
            want = orc.run_sequential(combo, Ms, 7, vin=vin[s * n:(s + 1) * n])
            assert np.array_equal(got[s], want)


@pytest.mark.parametrize("pack", ("0", "8", "16"))
@pytest.mark.parametrize("combo", (3, 6))
def test_ilu0_packing_modes(orc, golden, monkeypatch, pack, combo):
    """The ILU0 executor with 1, 2 or 4 same-level rows per warp
    (SFG_ILU_PACK 0 / 16 / 8): golden matrices and the C3 matrix, bit-exact,
    fused and unfused."""
    monkeypatch.setenv("SFG_ILU_PACK", pack)
    for name in GOLDEN_MATS:
        st = sf.make_state(combo, as_sf(golden_matrix(golden, name)), seed=7)
        want = golden[f"{name}/c{combo}/outputs"]
        st.execute_fused()
        assert np.array_equal(st.collect_outputs(), want)
        st.execute_unfused()
        assert np.array_equal(st.collect_outputs(), want)
    M = sf.config_matrix(3, size=40)
    want = orc.run_sequential(combo, Csc(M.n, M.colptr, M.rowidx, M.values), 7)
    st = sf.make_state(combo, M, seed=7)
    st.execute_fused()
    assert np.array_equal(st.collect_outputs(), want)


# ---- the GPU schedule checked by the reference's own validator ------------------
def _validated_by_reference(st, combo, Mo):
    from oracle.oracle import Reference
    part = st.partitioning()
    assert part.w_ptr[-1] == len(part.tags)
    rs = Reference().state(combo, Mo, 7)
    nbad, msg = rs.validate_partitioning(part.s_ptr, part.w_ptr, part.tags, part.iters)
    assert nbad == 0, msg
    return part


@pytest.mark.parametrize("name", GOLDEN_MATS)
@pytest.mark.parametrize("combo", (1, 2, 3, 5, 6, 7))
def test_partitioning_replayed_by_reference(golden, name, combo):
    """replay_schedule (executor.hpp:518-553): the reference runs the GPU's
    exported partitioning with its w-partitions interleaved in random orders;
    every replay reproduces the reference's sequential outputs (combo 4's CSC
    scatter is order-dependent and is checked by the validator only)."""
    from oracle.oracle import Reference
    Mo = golden_matrix(golden, name)
    st = sf.make_state(combo, as_sf(Mo)).inspect()
    part = st.partitioning()
    rs = Reference().state(combo, Mo, 7)
    want = golden[f"{name}/c{combo}/outputs"]
    for seed in (1, 2, 3):
        got = rs.replay_partitioning(part.s_ptr, part.w_ptr, part.tags, part.iters, seed)
        assert np.array_equal(got, want)


@pytest.mark.parametrize("name", GOLDEN_MATS)
@pytest.mark.parametrize("combo", (1, 2, 3, 4, 5, 6, 7))
def test_partitioning_valid_for_reference(golden, name, combo):
    # validate_fused_partitioning (msp.hpp:1108-1237): coverage, order inside
    # w-partitions, cross-partition dependences -- of the GPU-built schedule
    Mo = golden_matrix(golden, name)
    st = sf.make_state(combo, as_sf(Mo)).inspect()
    _validated_by_reference(st, combo, Mo)


@pytest.mark.parametrize("executor", ("chain", "mline", "levels"))
@pytest.mark.parametrize("combo", (1, 4))
def test_partitioning_valid_all_executors(monkeypatch, executor, combo):
    monkeypatch.setenv("SFG_EXECUTOR", executor)
    M = sf.config_matrix(1, size=40) if combo == 4 else sf.config_matrix(5, size=10)
    Mo = Csc(M.n, M.colptr, M.rowidx, M.values)
    st = sf.make_state(combo, M).inspect()
    part = _validated_by_reference(st, combo, Mo)
    assert part.b() > 1


# ---- batched executions with overlapped transfers (sfg_execute_batch) ----------
@pytest.mark.parametrize("combo,nsys", ((8, 8), (1, 2), (4, 1), (2, 1), (5, 1), (6, 1)))
def test_execute_batch_equals_serial(orc, combo, nsys):
    from paper_2111_12238_b200 import abi
    if combo in (1, 8):
        M, vals = sf.config5_systems(size=12, nsys=nsys)
    else:
        M, vals = sf.config_matrix({4: 1, 2: 1, 5: 2, 6: 3}[combo], size=16), None
    n = M.n
    st = sf.make_state(combo, M, nsys=nsys, values=vals).inspect()
    K = 5
    rng = np.random.default_rng(combo)
    ins = [abi.PinnedArray(nsys * n) for _ in range(K)]
    outs = [abi.PinnedArray(nsys * st.output_len) for _ in range(K)]
    for a in ins:
        a.array[:] = rng.uniform(-1, 1, nsys * n)
    st.execute_batch([a.array for a in ins], [o.array for o in outs])
    finals = [abi.PinnedArray(nsys * n) for _ in range(K)]
    st.execute_batch([a.array for a in ins], [f.array for f in finals], final_only=True)
    for k in range(K):
        st.set_vin(ins[k].array)
        st.execute_fused()
        full = st.collect_outputs()
        assert np.array_equal(outs[k].array, full)
        # SFG_OUTPUTS_FINAL: kernel 2's output of every system, system-major
        assert np.array_equal(finals[k].array, full.reshape(nsys, -1)[:, -n:].ravel())
    for a in ins + outs + finals:
        a.free()


def test_execute_batch_reports_breakdown(golden):
    from paper_2111_12238_b200 import abi
    cp = golden["breakdown/colptr"]
    M = sf.CscMatrix(len(cp) - 1, cp, golden["breakdown/rowidx"], golden["breakdown/values"])
    st = sf.make_state(5, M, seed=1).inspect()
    ins = [abi.PinnedArray(M.n) for _ in range(3)]
    outs = [abi.PinnedArray(st.output_len) for _ in range(3)]
    for a in ins:
        a.array[:] = 1.0
    with pytest.raises(sf.FactorizationError) as e:
        st.execute_batch([a.array for a in ins], [o.array for o in outs])
    assert e.value.index == 7
    for a in ins + outs:
        a.free()


def test_matrix_market_input_end_to_end(orc, tmp_path):
    # a matrix read from a Matrix Market file (symmetric storage) goes
    # through make_state exactly like a generated one
    M = sf.config_matrix(2, size=10)
    lines = ["%%MatrixMarket matrix coordinate real symmetric"]
    ent = []
    for j in range(M.n):
        for p in range(M.colptr[j], M.colptr[j + 1]):
            if M.rowidx[p] >= j:
                ent.append(f"{M.rowidx[p] + 1} {j + 1} {M.values[p]:.17g}")
    lines.append(f"{M.n} {M.n} {len(ent)}")
    path = tmp_path / "c2.mtx"
    path.write_text("\n".join(lines + ent) + "\n")
    R = sf.read_matrix_market(str(path))
    assert np.array_equal(R.values, M.values)
    perm = np.random.default_rng(2).permutation(R.n).astype(np.int32)
    P = sf.permute_symmetric(R, perm)
    for combo in (5, 6):
        st = sf.make_state(combo, P)
        st.execute_fused()
        want = orc.run_sequential(combo, Csc(P.n, P.colptr, P.rowidx, P.values), 7)
        assert np.array_equal(st.collect_outputs(), want)


# ---- PCG driver: IC0 factor (combo 5) + fused forward/backward solve (combo 8) --
def _csc_scipy(M):
    import scipy.sparse as sp
    return sp.csc_matrix((M.values, M.rowidx, M.colptr), shape=(M.n, M.n))


@pytest.mark.parametrize("cfg,size", ((2, 20), (2, 64), (4, 20000)))
def test_pcg_converges_to_true_solution(cfg, size):
    import scipy.sparse.linalg as spla
    M = sf.config_matrix(cfg, size=size, halfwidth=200) if cfg == 4 else sf.config_matrix(cfg, size=size)
    A = _csc_scipy(M)
    b = sf.gen_vector(M.n, 11)
    pcg = sf.PCG(M)
    x, it, rr, ms = pcg.solve(b, rtol=1e-10, maxit=500)
    assert rr <= 1e-10 and 0 < it < 500
    assert np.linalg.norm(A @ x - b) <= 1e-9 * np.linalg.norm(b)
    if M.n <= 10000:
        xd = spla.spsolve(A.tocsc(), b)
        assert np.max(np.abs(x - xd)) <= 1e-8 * np.max(np.abs(xd))
    x2, it2, rr2, _ = pcg.solve(b, rtol=1e-10, maxit=500)
    assert it2 == it and np.array_equal(x2, x)  # deterministic reductions
    pcg.close()


def test_pcg_preconditioner_helps():
    M = sf.config_matrix(2, size=32)
    b = sf.gen_vector(M.n, 3)
    x, it, rr, _ = sf.PCG(M).solve(b, rtol=1e-8, maxit=1000)
    # unpreconditioned CG on this operator needs roughly 3x more iterations
    import scipy.sparse.linalg as spla
    count = [0]
    spla.cg(_csc_scipy(M), b, rtol=1e-8, maxiter=1000, callback=lambda _: count.__setitem__(0, count[0] + 1))
    assert it < count[0]


def test_pcg_ic0_breakdown_reported():
    M = sf.config_matrix(1, size=6)
    vals = M.values.copy()
    cols = np.repeat(np.arange(M.n), np.diff(M.colptr))
    vals[M.rowidx == cols] = 1.0  # diagonal 1 with off-diagonals -1: IC0 breaks down
    with pytest.raises(sf.FactorizationError):
        sf.PCG(sf.CscMatrix(M.n, M.colptr, M.rowidx, vals))


# ---------------------------------------------------------------------------
# config 1 split across ranks: kernel 1 alone, then the row-sharded
# SpMV; on one GPU the shards run back to back and must reproduce combo 4's y
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("size,world", [(64, 1), (64, 3), (512, 4), (512, 7)])
def test_config1_sharded_spmv_matches_fused(size, world):
    import torch
    from paper_2111_12238_b200 import shard
    M = sf.config_matrix(1, size=size)
    st = sf.make_state(4, M, seed=7)
    st.execute_fused()
    want = st.collect_outputs()
    n = M.n
    st2 = sf.make_state(4, M, seed=7)
    torch.cuda.set_device(0)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        st2.set_stream(s.cuda_stream)  # plan and torch share one stream
        solve, spmv = shard.plan_callbacks(st2, n)
        x = solve()
        ys = []
        for r0, r1 in shard.row_shards(n, world):
            y = torch.full((max(r1 - r0, 1),), float("nan"), dtype=torch.float64, device="cuda")
            if r1 > r0:
                spmv(r0, r1, x, y)
            ys.append(y[:r1 - r0])
        got_x = x.cpu().numpy()
        got_y = torch.cat(ys).cpu().numpy()
        # ShardedSpmv at world 1 is the same computation end to end
        S = shard.ShardedSpmv(None, 0, 1, n, *shard.csr_pattern(M.colptr, M.rowidx, n),
                              torch.device("cuda"), solve=solve, spmv=spmv)
        y1 = S.step().cpu().numpy()
    st2.synchronize()
    assert np.array_equal(got_x, want[:n])
    assert np.array_equal(got_y, want[n:2 * n])
    assert np.array_equal(y1, want[n:2 * n])
    st.close()
    st2.close()


def test_execute_kernel_two_halves_equal_unfused(golden):
    """sfg_execute_kernel(1) then (2) == execute_unfused for every combo."""
    M = as_sf(golden_matrix(golden, "grid10"))
    for combo in GPU_COMBOS:
        st = sf.make_state(combo, M, seed=7)
        st.execute_unfused()
        want = st.collect_outputs()
        st2 = sf.make_state(combo, M, seed=7)
        st2.execute_kernel(1)
        st2.execute_kernel(2)
        assert np.array_equal(st2.collect_outputs(), want), combo
        st.close()
        st2.close()


def test_spmv_rows_rejects_bad_ranges():
    M = sf.config_matrix(1, size=16)
    st = sf.make_state(4, M, seed=7)
    st.inspect()
    with pytest.raises(Exception):
        st.spmv_rows(5, 4, 1, 1)
    with pytest.raises(Exception):
        st.spmv_rows(0, M.n + 1, 1, 1)
    st.close()


# ---------------------------------------------------------------------------
# different plans run concurrently on different streams:
# every executor claims tickets only from resident warps, so two launches
# sharing the GPU both progress; results stay bit-exact
# ---------------------------------------------------------------------------
def test_plans_concurrent_on_streams(orc):
    import torch
    torch.cuda.set_device(0)
    cases = [(8, None), (7, sf.config_matrix(4, size=20000, halfwidth=200)),
             (6, sf.config_matrix(3, size=24)), (4, sf.config_matrix(1, size=128))]
    plans, wants = [], []
    Mb, vals = sf.config5_systems(size=16, nsys=4)
    vin = np.concatenate([sf.gen_vector(Mb.n, 7 + s) for s in range(4)])
    for combo, M in cases:
        if combo == 8:
            st = sf.make_state(8, Mb, nsys=4, values=vals, vin=vin)
            want = []
            for s in range(4):
                Ms = Csc(Mb.n, Mb.colptr, Mb.rowidx, vals[s * Mb.nnz:(s + 1) * Mb.nnz])
                want.append(orc.run_sequential(8, Ms, 7, vin=vin[s * Mb.n:(s + 1) * Mb.n]))
            want = np.stack(want).ravel()
        else:
            st = sf.make_state(combo, M, seed=7)
            want = orc.run_sequential(combo, Csc(M.n, M.colptr, M.rowidx, M.values), 7)
        st.inspect()
        plans.append(st)
        wants.append(want)
    streams = [torch.cuda.Stream() for _ in plans]
    for st, s in zip(plans, streams):
        st.set_stream(s.cuda_stream)
    for _ in range(3):
        for st in plans:
            st.execute_fused(sync=False)
        for st, want in zip(plans, wants):
            got = st.collect_outputs()  # batched plan: system-major, like want
            assert np.array_equal(got.ravel(), want), "concurrent execution changed a result"
    for st in plans:
        st.set_stream(None)
        st.close()


# new values for every system of a batched plan (same pattern): the staged
# chain executor re-reads them, fused and unfused, bit-exact
@pytest.mark.parametrize("combo", (1, 8))
def test_set_values_batched(orc, combo):
    nsys = 4
    M, vals = sf.config5_systems(size=12, nsys=nsys)
    vin = np.concatenate([sf.gen_vector(M.n, 7 + s) for s in range(nsys)])
    st = sf.make_state(combo, M, nsys=nsys, values=vals, vin=vin).inspect()
    st.execute_fused()
    rng = np.random.default_rng(combo)
    v2 = vals * (1.0 + 0.05 * rng.uniform(0, 1, vals.size))
    st.set_values(v2)
    for run in (st.execute_fused, st.execute_unfused):
        run()
        got = st.collect_outputs().reshape(nsys, -1)
        for s in range(nsys):
            Ms = Csc(M.n, M.colptr, M.rowidx, v2[s * M.nnz:(s + 1) * M.nnz])
            want = orc.run_sequential(combo, Ms, 7, vin=vin[s * M.n:(s + 1) * M.n])
            assert np.array_equal(got[s], want), (combo, s, run.__name__)
    st.close()
