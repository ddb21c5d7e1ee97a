"""The reference's schedule API on the GPU (-m gpu): the canonical call
sequence of proj/demos/fuse_demo.cpp:15-31 (msp -> validate_fused_partitioning
-> compile_schedule -> execute_fused / execute_unfused /
execute_joint_wavefront / execute_sequential), schedules handed to
execute_fused are verified against the joint DAG, and the wavefront and
sequential executors reproduce the reference's outputs.

Golden outputs come from the unmodified reference (tests/golden); full-size
cases are compared with the oracle (oracle/sf_oracle.c, pinned by
test_oracle.py)."""
import numpy as np
import pytest

import paper_2111_12238_b200 as sf
from conftest import GOLDEN_MATS, golden_matrix
from oracle.oracle import Csc

pytestmark = pytest.mark.gpu

TOL = 1e-10  # north_star: fp64 within max-relative-error 1e-10
CONFIG_COMBO = {1: 4, 2: 5, 3: 6, 4: 7}


def as_sf(M) -> sf.CscMatrix:
    return sf.CscMatrix(M.n, M.colptr, M.rowidx, M.values)


def close_combo4(got, want):
    # spmv_csc_col accumulates with atomic adds in any order
    # (kernels.hpp:162-168; the reference's own tolerance, test_kernels.cpp:395-396)
    scale = max(1.0, float(np.max(np.abs(want))))
    return float(np.max(np.abs(got - want))) <= 1e-13 * scale


@pytest.fixture(scope="module", autouse=True)
def _device():
    from paper_2111_12238_b200 import abi
    assert abi.device_available(), "B200 required: the -m gpu suite never skips"


@pytest.mark.parametrize("name", GOLDEN_MATS)
@pytest.mark.parametrize("combo", (1, 2, 3, 4, 5, 6, 7))
def test_canonical_sequence_golden(golden, name, combo):
    """fuse_demo.cpp's sequence, every executor checked against the
    reference's golden outputs."""
    key = f"{name}/c{combo}"
    want = golden[f"{key}/outputs"]
    st = sf.make_state(combo, as_sf(golden_matrix(golden, name)), seed=7)
    g1, g2 = sf.build_g1(st), sf.build_g2(st)
    f = sf.inter_dag(st)
    reuse = sf.compute_reuse(st)
    V = sf.msp(g1, g2, f, 4, reuse)
    assert sf.validate_fused_partitioning(V, g1, g2, f) == []
    assert V.interleaved == (reuse >= 1.0)
    sched = sf.compile_schedule(V, reuse, g1, g2, 4)
    sf.execute_fused(sched, st, 4)
    assert np.array_equal(sf.collect_outputs(st), want)
    sf.execute_unfused(g1, g2, st, 4)
    assert np.array_equal(sf.collect_outputs(st), want)
    sf.execute_joint_wavefront(g1, g2, f, st, 4)
    got = sf.collect_outputs(st)
    assert close_combo4(got, want) if combo == 4 else np.array_equal(got, want)
    sf.execute_sequential(st)
    assert np.array_equal(sf.collect_outputs(st), want)


@pytest.mark.parametrize("name", GOLDEN_MATS)
@pytest.mark.parametrize("combo", (1, 2, 3, 4, 5, 6, 7))
def test_wavefront_schedule_golden(golden, name, combo):
    """build_wavefront_schedule's level sets (executor.hpp:209-229): the GPU
    inspector's, and those built from the bare DAGs, equal the reference's."""
    key = f"{name}/c{combo}"
    st = sf.make_state(combo, as_sf(golden_matrix(golden, name)))
    for g1, g2, f in ((sf.build_g1(st), sf.build_g2(st), sf.inter_dag(st)),
                      (sf.DepDag(*golden_dag(golden, key, "g1")), sf.DepDag(*golden_dag(golden, key, "g2")),
                       sf.InterDep(st.n, st.n, golden[f"{key}/f_rowptr"], golden[f"{key}/f_colidx"]))):
        ws = sf.build_wavefront_schedule(g1, g2, f)
        assert np.array_equal(ws.tags, golden[f"{key}/wf_tags"])
        assert np.array_equal(ws.iters, golden[f"{key}/wf_iters"])
        assert np.array_equal(ws.level_ptr, golden[f"{key}/wf_ptr"])


def golden_dag(golden, key, g):
    sp = golden[f"{key}/{g}_succptr"]
    return len(sp) - 1, sp, golden[f"{key}/{g}_succ"], golden[f"{key}/{g}_cost"]


@pytest.mark.parametrize("name", GOLDEN_MATS)
@pytest.mark.parametrize("combo", (1, 2, 3, 4, 5, 6, 7))
def test_dag_only_msp_and_structures(golden, name, combo):
    """msp / joint_dag / level_info on DAGs that carry no state (the
    reference's free functions on plain structures)."""
    key = f"{name}/c{combo}"
    g1 = sf.DepDag(*golden_dag(golden, key, "g1"))
    g2 = sf.DepDag(*golden_dag(golden, key, "g2"))
    n = g1.nvert
    f = sf.InterDep(n, n, golden[f"{key}/f_rowptr"], golden[f"{key}/f_colidx"])
    j = sf.joint_dag(g1, g2, f)
    assert np.array_equal(j.succptr, golden[f"{key}/j_succptr"])
    assert np.array_equal(j.succ, golden[f"{key}/j_succ"])
    assert np.array_equal(j.cost, golden[f"{key}/j_cost"])
    li = sf.level_info(j)
    assert np.array_equal(li.level, golden[f"{key}/j_level"])
    assert np.array_equal(li.height, golden[f"{key}/j_height"])
    assert np.array_equal(li.slack, golden[f"{key}/j_slack"])
    assert li.critical_path == golden[f"{key}/j_P"][0]
    reuse = float(golden[f"{key}/reuse"][0])
    V = sf.msp(g1, g2, f, 3, reuse)
    assert sf.validate_fused_partitioning(V, g1, g2, f) == []
    # executed on a state of the same matrix: verified against its joint DAG
    st = sf.make_state(combo, as_sf(golden_matrix(golden, name)), seed=7)
    sched = sf.compile_schedule(V, reuse, g1, g2, 3)
    assert sched.checked_for is None
    sf.execute_fused(sched, st, 3)
    assert np.array_equal(sf.collect_outputs(st), golden[f"{key}/outputs"])


@pytest.mark.parametrize("combo", (1, 4, 5, 6, 7, 8))
def test_invalid_schedule_refused(golden, combo):
    st = sf.make_state(combo, as_sf(golden_matrix(golden, "grid10")), seed=7)
    sched = sf.make_fused_schedule(st)
    bad = sf.FusedSchedule(sched.tags[::-1].copy(), sched.iters[::-1].copy(), sched.wave_ptr)
    assert st.check_schedule(bad.tags, bad.iters) > 0
    with pytest.raises(ValueError):
        sf.execute_fused(bad, st)
    missing = sf.FusedSchedule(sched.tags[1:].copy(), sched.iters[1:].copy(), sched.wave_ptr)
    with pytest.raises(ValueError):
        sf.execute_fused(missing, st)
    assert st.check_schedule(sched.tags, sched.iters) == 0


def test_unfused_rejects_foreign_dags(golden):
    a = sf.make_state(5, as_sf(golden_matrix(golden, "grid6")))
    b = sf.make_state(5, as_sf(golden_matrix(golden, "grid6")))
    with pytest.raises(ValueError):
        sf.execute_unfused(sf.build_g1(a), sf.build_g2(a), b)


@pytest.mark.parametrize("combo", (1, 4, 5, 6, 7, 8))
def test_reset_restores_inputs(golden, combo):
    """reset (kernels.hpp:498-502): fac = fac0, vmid = vout = 0."""
    M = golden_matrix(golden, "grid6")
    st = sf.make_state(combo, as_sf(M), seed=7)
    st.execute_fused()
    sf.reset(st)
    out = st.collect_outputs()
    n = st.n
    if combo in (1, 4, 8):
        assert not out.any()
    elif combo in (5, 7):
        lower = [p for j in range(n) for p in range(M.colptr[j], M.colptr[j + 1]) if M.rowidx[p] >= j]
        assert np.array_equal(out[:-n], M.values[lower])
        if combo == 5:
            assert not out[-n:].any()
    else:  # combo 6: CSR values of A
        assert not out[-n:].any()
        assert np.array_equal(np.sort(out[:-n]), np.sort(M.values))


@pytest.mark.parametrize("cfg", (1, 2, 3, 4))
def test_wavefront_executor_full_size(orc, cfg):
    M = sf.config_matrix(cfg)
    combo = CONFIG_COMBO[cfg]
    want = orc.run_sequential(combo, Csc(M.n, M.colptr, M.rowidx, M.values), 7)
    st = sf.make_state(combo, M, seed=7)
    st.execute_wavefront()
    got = st.collect_outputs()
    if combo == 4:
        assert close_combo4(got, want)
    else:
        assert np.array_equal(got, want)


def test_wavefront_executor_config5_batch(orc):
    nsys = 8
    M, vals = sf.config5_systems(size=48, nsys=nsys)
    n, nnz = M.n, M.nnz
    vin = np.concatenate([sf.gen_vector(n, 7 + s) for s in range(nsys)])
    st = sf.make_state(8, M, nsys=nsys, values=vals, vin=vin)
    st.execute_wavefront()
    got = st.collect_outputs().reshape(nsys, 2 * n)
    for s in range(nsys):
        Ms = Csc(n, M.colptr, M.rowidx, vals[s * nnz:(s + 1) * nnz])
        assert np.array_equal(got[s], orc.run_sequential(8, Ms, 7, vin=vin[s * n:(s + 1) * n]))


def test_wavefront_reports_breakdown(golden):
    cp = golden["breakdown/colptr"]
    M = sf.CscMatrix(len(cp) - 1, cp, golden["breakdown/rowidx"], golden["breakdown/values"])
    st = sf.make_state(5, M, seed=1)
    for run in (st.execute_wavefront, st.execute_sequential):
        with pytest.raises(sf.FactorizationError) as e:
            run()
        assert e.value.index == golden["breakdown/c5_index"][0]
