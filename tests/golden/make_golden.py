"""Regenerates tests/golden/*.npz from the UNMODIFIED reference.

Runs only where /root/reference exists (oracle/_ref/libsfref.so is built from
it by oracle/Makefile).  Every array stored here is produced by the reference
itself -- its generators (fixtures.hpp), make_state + run_sequential_reference
+ collect_outputs (kernels.hpp), build_g1/build_g2/inter_dag/joint_dag/
level_info/compute_reuse (dag.hpp) and build_wavefront_schedule
(executor.hpp) -- and combo 8 (forward L then backward L^T), which the
reference lacks as a pair: its outputs come from the reference's own
primitives composed as SURVEY.md 8(c) prescribes -- sptrsv (kernels.hpp:
335-342) on L, then sptrsv on permute_symmetric(transpose(L), rev)
(matrix.hpp:130-173), oracle/ref_driver.cpp ref_fwd_bwd -- and are checked
here against the C oracle (bit for bit) and a dense backward substitution.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import Csc, Oracle, Reference  # noqa: E402

COMBOS = (1, 2, 3, 4, 5, 6, 7)


def dense_backward(L: np.ndarray, z: np.ndarray) -> np.ndarray:
    n = len(z)
    x = np.zeros(n)
    for i in range(n - 1, -1, -1):
        acc = z[i]
        for j in range(n - 1, i, -1):
            acc -= L[j, i] * x[j]
        x[i] = acc / L[i, i]
    return x


def to_dense(M: Csc) -> np.ndarray:
    D = np.zeros((M.n, M.n))
    for j in range(M.n):
        for p in range(M.colptr[j], M.colptr[j + 1]):
            D[M.rowidx[p], j] += M.values[p]
    return D


def main():
    ref = Reference()
    orc = Oracle()
    mats = {
        "banded24": ref.gen_banded_spd(24, 3, 11),
        "banded40": ref.gen_banded_spd(40, 5, 3),
        "grid6": ref.gen_grid_laplacian(6),
        "grid10": ref.gen_grid_laplacian(10),
        "fixture11": ref.fixture11_lower(),
        "dense12": ref.gen_dense_spd(12, 3),
    }
    out = {
        "gen_vector_4_7": ref.gen_vector(4, 7),
        "gen_vector_1000_123": ref.gen_vector(1000, 123),
    }
    for name, M in mats.items():
        out[f"{name}/colptr"] = M.colptr
        out[f"{name}/rowidx"] = M.rowidx
        out[f"{name}/values"] = M.values
        for combo in COMBOS:
            st = ref.state(combo, M, 7)
            key = f"{name}/c{combo}"
            out[f"{key}/outputs"] = st.execute(0)
            for which in (1, 2):
                g = st.build_g(which)
                out[f"{key}/g{which}_succptr"] = g.succptr
                out[f"{key}/g{which}_succ"] = g.succ
                out[f"{key}/g{which}_cost"] = g.cost
            f = st.inter_dag()
            out[f"{key}/f_rowptr"] = f.rowptr
            out[f"{key}/f_colidx"] = f.colidx
            j = st.joint_dag()
            out[f"{key}/j_succptr"] = j.succptr
            out[f"{key}/j_succ"] = j.succ
            out[f"{key}/j_cost"] = j.cost
            li = ref.level_info(j)
            out[f"{key}/j_level"] = li.level
            out[f"{key}/j_height"] = li.height
            out[f"{key}/j_slack"] = li.slack
            out[f"{key}/j_P"] = np.array([li.critical_path], np.int32)
            for which in (1, 2):
                lg = ref.level_info(st.build_g(which))
                out[f"{key}/g{which}_level"] = lg.level
                out[f"{key}/g{which}_P"] = np.array([lg.critical_path], np.int32)
            out[f"{key}/reuse"] = np.array([st.compute_reuse()])
            tags, iters, lp = st.wavefront()
            out[f"{key}/wf_tags"] = tags
            out[f"{key}/wf_iters"] = iters
            out[f"{key}/wf_ptr"] = lp
        # combo 8 (Deviation 1): the reference's primitives composed
        # (ref_fwd_bwd); the oracle must agree bit for bit, and the backward
        # half must match a dense substitution
        got8 = ref.fwd_bwd(M, ref.gen_vector(M.n, 7))
        assert np.array_equal(got8, orc.run_sequential(8, M, 7))
        z = ref.state(1, M, 7).execute(0)[: M.n]
        D = np.tril(to_dense(M))
        x_dense = dense_backward(D, z)
        assert np.array_equal(got8[: M.n], z)
        assert np.max(np.abs(got8[M.n:] - x_dense)) <= 1e-12 * max(1.0, np.max(np.abs(x_dense)))
        out[f"{name}/c8/outputs"] = got8
    # numeric breakdown pin (test_executor.cpp:157-171): column 7 made indefinite
    A = ref.gen_banded_spd(16, 2, 3)
    vals = A.values.copy()
    for p in range(A.colptr[7], A.colptr[8]):
        if A.rowidx[p] == 7:
            vals[p] = -vals[p]
    out["breakdown/colptr"] = A.colptr
    out["breakdown/rowidx"] = A.rowidx
    out["breakdown/values"] = vals
    try:
        ref.state(5, Csc(A.n, A.colptr, A.rowidx, vals), 1).execute(0)
        raise AssertionError("expected breakdown")
    except Exception as e:  # FactorizationError
        out["breakdown/c5_index"] = np.array([e.index], np.int32)
    np.savez_compressed(os.path.join(HERE, "reference_golden.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
