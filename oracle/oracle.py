"""ctypes bindings for the test-infrastructure libraries in oracle/.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py -- always as the checker or
the CPU baseline, never as the product path.

* ``Oracle``     -- liboracle.so, the plain-C restatement (oracle/sf_oracle.c).
* ``Reference``  -- _ref/libsfref.so, the unmodified reference headers compiled
                    where they lie under /root/reference (oracle/Makefile).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

ERR_NAMES = {
    1: "zero diagonal in triangular solve",
    2: "non-positive pivot",
    3: "zero pivot",
    4: "invalid matrix",
    5: "zero diagonal",
    6: "bad argument",
}

_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)


def _p(a, t):
    return a.ctypes.data_as(t) if a is not None else None


@dataclass
class Csc:
    """CscMatrix (matrix.hpp:18-26): square, int32 indices, fp64 values."""

    n: int
    colptr: np.ndarray
    rowidx: np.ndarray
    values: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.colptr[-1])

    def arrays(self):
        return (np.ascontiguousarray(self.colptr, np.int32),
                np.ascontiguousarray(self.rowidx, np.int32),
                np.ascontiguousarray(self.values, np.float64))


@dataclass
class Dag:
    """DepDag (dag.hpp:17-30)."""

    nvert: int
    succptr: np.ndarray
    succ: np.ndarray
    cost: np.ndarray


@dataclass
class InterDep:
    """InterDep F (dag.hpp:34-41)."""

    nrows: int
    ncols: int
    rowptr: np.ndarray
    colidx: np.ndarray


@dataclass
class Levels:
    """LevelInfo (dag.hpp:43-48)."""

    level: np.ndarray
    height: np.ndarray
    slack: np.ndarray
    critical_path: int


class FactorizationError(RuntimeError):
    """Mirror of sparsefuse::FactorizationError (types.hpp:17-26)."""

    def __init__(self, what: str, index: int, code: int = 0):
        super().__init__(f"{what} at index {index}")
        self.index = index
        self.code = code


class _OrcDag(C.Structure):
    _fields_ = [("nvert", C.c_int32), ("nedges", C.c_int64),
                ("succptr", _i32p), ("succ", _i32p), ("cost", _i64p)]


class _OrcInter(C.Structure):
    _fields_ = [("nrows", C.c_int32), ("ncols", C.c_int32), ("nnz", C.c_int64),
                ("rowptr", _i32p), ("colidx", _i32p)]


def _ensure_built(path: str):
    if not os.path.exists(path):
        import subprocess
        subprocess.check_call(["make", "-s", "-C", HERE])


class Oracle:
    """The plain-C restatement (oracle/sf_oracle.c)."""

    def __init__(self, path: str | None = None):
        path = path or os.path.join(HERE, "liboracle.so")
        _ensure_built(path)
        L = C.CDLL(path)
        L.orc_gen_vector.argtypes = [C.c_int32, C.c_uint64, _f64p]
        L.orc_output_len.argtypes = [C.c_int, C.c_int32, _i32p, _i32p]
        L.orc_output_len.restype = C.c_int64
        L.orc_run_sequential.argtypes = [C.c_int, C.c_int32, _i32p, _i32p, _f64p,
                                         C.c_uint64, _f64p, _f64p, C.c_int64,
                                         _i32p, _i32p]
        L.orc_run_sequential.restype = C.c_int64
        L.orc_build_g.argtypes = [C.c_int, C.c_int, C.c_int32, _i32p, _i32p, _f64p,
                                  C.POINTER(_OrcDag)]
        L.orc_inter_dag.argtypes = [C.c_int, C.c_int32, _i32p, _i32p, _f64p,
                                    C.POINTER(_OrcInter)]
        L.orc_joint_dag.argtypes = [C.POINTER(_OrcDag), C.POINTER(_OrcDag),
                                    C.POINTER(_OrcInter), C.POINTER(_OrcDag)]
        L.orc_level_info.argtypes = [C.POINTER(_OrcDag), _i32p, _i32p, _i32p, _i32p]
        L.orc_compute_reuse.argtypes = [C.c_int, C.c_int32, _i32p, _i32p, _f64p]
        L.orc_compute_reuse.restype = C.c_double
        L.orc_free_dag.argtypes = [C.POINTER(_OrcDag)]
        L.orc_free_interdep.argtypes = [C.POINTER(_OrcInter)]
        self.lib = L

    def gen_vector(self, n: int, seed: int) -> np.ndarray:
        out = np.empty(n, np.float64)
        self.lib.orc_gen_vector(n, seed, _p(out, _f64p))
        return out

    def run_sequential(self, combo: int, M: Csc, seed: int = 7, vin=None) -> np.ndarray:
        """make_state + run_sequential_reference + collect_outputs."""
        cp, ri, va = M.arrays()
        cap = self.lib.orc_output_len(combo, M.n, _p(cp, _i32p), _p(ri, _i32p))
        if cap < 0:
            raise ValueError("bad combo id")
        out = np.empty(max(cap, 1), np.float64)
        code = C.c_int32(0)
        idx = C.c_int32(-1)
        vin_a = None if vin is None else np.ascontiguousarray(vin, np.float64)
        got = self.lib.orc_run_sequential(combo, M.n, _p(cp, _i32p), _p(ri, _i32p),
                                          _p(va, _f64p), seed, _p(vin_a, _f64p),
                                          _p(out, _f64p), cap, C.byref(code),
                                          C.byref(idx))
        if got < 0:
            if code.value in (1, 2, 3, 5):
                raise FactorizationError(ERR_NAMES[code.value], idx.value, code.value)
            raise ValueError(f"{ERR_NAMES.get(code.value, 'error')} at {idx.value}")
        return out[:got]

    @staticmethod
    def _dag(d: _OrcDag) -> Dag:
        nv, ne = d.nvert, d.nedges
        sp = np.ctypeslib.as_array(d.succptr, (nv + 1,)).copy()
        su = (np.ctypeslib.as_array(d.succ, (ne,)).copy() if ne
              else np.zeros(0, np.int32))
        co = (np.ctypeslib.as_array(d.cost, (nv,)).copy() if nv
              else np.zeros(0, np.int64))
        return Dag(nv, sp, su, co)

    def build_g(self, combo: int, which: int, M: Csc) -> Dag:
        cp, ri, va = M.arrays()
        d = _OrcDag()
        rc = self.lib.orc_build_g(combo, which, M.n, _p(cp, _i32p), _p(ri, _i32p),
                                  _p(va, _f64p), C.byref(d))
        if rc:
            raise ValueError(f"build_g failed: {ERR_NAMES.get(rc)}")
        try:
            return self._dag(d)
        finally:
            self.lib.orc_free_dag(C.byref(d))

    def inter_dag(self, combo: int, M: Csc) -> InterDep:
        cp, ri, va = M.arrays()
        f = _OrcInter()
        rc = self.lib.orc_inter_dag(combo, M.n, _p(cp, _i32p), _p(ri, _i32p),
                                    _p(va, _f64p), C.byref(f))
        if rc:
            raise ValueError(f"inter_dag failed: {ERR_NAMES.get(rc)}")
        try:
            rp = np.ctypeslib.as_array(f.rowptr, (f.nrows + 1,)).copy()
            ci = (np.ctypeslib.as_array(f.colidx, (f.nnz,)).copy() if f.nnz
                  else np.zeros(0, np.int32))
            return InterDep(f.nrows, f.ncols, rp, ci)
        finally:
            self.lib.orc_free_interdep(C.byref(f))

    @staticmethod
    def _to_c_dag(g: Dag):
        keep = [np.ascontiguousarray(g.succptr, np.int32),
                np.ascontiguousarray(g.succ if len(g.succ) else np.zeros(1, np.int32), np.int32),
                np.ascontiguousarray(g.cost if len(g.cost) else np.zeros(1, np.int64), np.int64)]
        d = _OrcDag(g.nvert, int(g.succptr[-1]), _p(keep[0], _i32p),
                    _p(keep[1], _i32p), _p(keep[2], _i64p))
        return d, keep

    def joint_dag(self, g1: Dag, g2: Dag, f: InterDep) -> Dag:
        d1, k1 = self._to_c_dag(g1)
        d2, k2 = self._to_c_dag(g2)
        rp = np.ascontiguousarray(f.rowptr, np.int32)
        ci = np.ascontiguousarray(f.colidx if len(f.colidx) else np.zeros(1, np.int32), np.int32)
        cf = _OrcInter(f.nrows, f.ncols, int(f.rowptr[-1]), _p(rp, _i32p), _p(ci, _i32p))
        out = _OrcDag()
        self.lib.orc_joint_dag(C.byref(d1), C.byref(d2), C.byref(cf), C.byref(out))
        try:
            return self._dag(out)
        finally:
            self.lib.orc_free_dag(C.byref(out))

    def level_info(self, g: Dag) -> Levels:
        d, keep = self._to_c_dag(g)
        n = g.nvert
        lv = np.empty(max(n, 1), np.int32)
        ht = np.empty(max(n, 1), np.int32)
        sl = np.empty(max(n, 1), np.int32)
        P = C.c_int32(0)
        rc = self.lib.orc_level_info(C.byref(d), _p(lv, _i32p), _p(ht, _i32p),
                                     _p(sl, _i32p), C.byref(P))
        if rc:
            raise ValueError("dependence cycle: edge does not ascend")
        return Levels(lv[:n], ht[:n], sl[:n], P.value)

    def compute_reuse(self, combo: int, M: Csc) -> float:
        cp, ri, va = M.arrays()
        return self.lib.orc_compute_reuse(combo, M.n, _p(cp, _i32p), _p(ri, _i32p),
                                          _p(va, _f64p))


class Reference:
    """The unmodified reference, compiled from /root/reference (oracle/_ref)."""

    PATH = os.path.join(HERE, "_ref", "libsfref.so")

    @classmethod
    def available(cls) -> bool:
        return os.path.exists(cls.PATH)

    def __init__(self):
        if not self.available():
            raise FileNotFoundError(self.PATH)
        L = C.CDLL(self.PATH)
        vp = C.c_void_p
        L.ref_gen_vector.argtypes = [C.c_int32, C.c_uint64, _f64p]
        L.ref_mat_gen.argtypes = [C.c_int, C.c_int32, C.c_int32, C.c_uint64]
        L.ref_mat_gen.restype = vp
        L.ref_mat_dims.argtypes = [vp, _i32p, _i32p]
        L.ref_mat_copy.argtypes = [vp, _i32p, _i32p, _f64p]
        L.ref_mat_free.argtypes = [vp]
        L.ref_state_new.argtypes = [C.c_int, C.c_int32, _i32p, _i32p, _f64p, C.c_uint64,
                                    _f64p, _i32p, C.c_char_p, C.c_int]
        L.ref_state_new.restype = vp
        L.ref_state_fixture11.argtypes = [C.c_uint64]
        L.ref_state_fixture11.restype = vp
        L.ref_state_free.argtypes = [vp]
        L.ref_output_len.argtypes = [vp]
        L.ref_output_len.restype = C.c_int64
        L.ref_execute.argtypes = [vp, C.c_int, C.c_int32, _f64p, C.c_int64, _i32p,
                                  C.c_char_p, C.c_int]
        L.ref_bench.argtypes = [vp, C.c_int, C.c_int32, C.c_int, C.c_int, _f64p, _f64p,
                                _i32p, C.c_char_p, C.c_int]
        L.ref_build_g.argtypes = [vp, C.c_int]
        L.ref_build_g.restype = vp
        L.ref_inter_dag.argtypes = [vp]
        L.ref_inter_dag.restype = vp
        L.ref_joint_dag.argtypes = [vp, vp, vp]
        L.ref_joint_dag.restype = vp
        L.ref_dag_from_csr.argtypes = [C.c_int32, _i32p, _i32p, _i64p]
        L.ref_dag_from_csr.restype = vp
        L.ref_dag_dims.argtypes = [vp, _i32p, _i64p]
        L.ref_dag_copy.argtypes = [vp, _i32p, _i32p, _i64p]
        L.ref_dag_free.argtypes = [vp]
        L.ref_inter_dims.argtypes = [vp, _i32p, _i32p, _i64p]
        L.ref_inter_copy.argtypes = [vp, _i32p, _i32p]
        L.ref_inter_free.argtypes = [vp]
        L.ref_level_info.argtypes = [vp, _i32p, _i32p, _i32p, _i32p]
        L.ref_compute_reuse.argtypes = [vp]
        L.ref_compute_reuse.restype = C.c_double
        L.ref_wavefront.argtypes = [vp, C.POINTER(C.c_uint8), _i32p, _i32p, _i32p]
        L.ref_wavefront.restype = C.c_int64
        L.ref_validate_partitioning.argtypes = [vp, C.c_int32, _i64p, _i64p,
                                                C.POINTER(C.c_uint8), _i32p, C.c_char_p, C.c_int]
        L.ref_validate_partitioning.restype = C.c_int64
        L.ref_replay_partitioning.argtypes = [vp, C.c_int32, _i64p, _i64p, C.POINTER(C.c_uint8), _i32p,
                                              C.c_uint64, _f64p, C.c_int64, _i32p, C.c_char_p, C.c_int]
        L.ref_read_mm.argtypes = [C.c_char_p, C.c_char_p, C.c_int]
        L.ref_read_mm.restype = vp
        L.ref_fwd_bwd.argtypes = [C.c_int32, _i32p, _i32p, _f64p, _f64p, _f64p, _i32p,
                                  C.c_char_p, C.c_int]
        L.ref_backward_matrix.argtypes = [C.c_int32, _i32p, _i32p, _f64p]
        L.ref_backward_matrix.restype = vp
        L.ref_solver_new.argtypes = [C.c_int32, _i32p, _i32p, _f64p, C.c_int32, _f64p]
        L.ref_solver_new.restype = vp
        L.ref_solver_run.argtypes = [vp, _f64p, _f64p, _f64p, _i32p, C.c_char_p, C.c_int]
        L.ref_solver_free.argtypes = [vp]
        L.ref_solver_clone_diag.argtypes = [vp, _f64p]
        L.ref_solver_clone_diag.restype = vp
        # the repo's BASELINE generators (fixtures.cpp compiled in, renamed)
        L.refgen_matrix_gen.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_uint64,
                                        C.POINTER(vp)]
        L.refgen_matrix_dims.argtypes = [vp, _i32p, _i64p]
        L.refgen_matrix_copy.argtypes = [vp, _i32p, _i32p, _f64p]
        L.refgen_matrix_free.argtypes = [vp]
        L.refgen_matrix_perturb_diag.argtypes = [vp, C.c_int32, C.c_uint64, _f64p]
        self.lib = L

    # ---- fixtures.hpp
    def gen_vector(self, n: int, seed: int) -> np.ndarray:
        out = np.empty(n, np.float64)
        self.lib.ref_gen_vector(n, seed, _p(out, _f64p))
        return out

    def _mat(self, kind, a, b=0, seed=0) -> Csc:
        h = self.lib.ref_mat_gen(kind, a, b, seed)
        if not h:
            raise ValueError("generator failed")
        n = C.c_int32()
        nnz = C.c_int32()
        self.lib.ref_mat_dims(h, C.byref(n), C.byref(nnz))
        cp = np.empty(n.value + 1, np.int32)
        ri = np.empty(max(nnz.value, 1), np.int32)
        va = np.empty(max(nnz.value, 1), np.float64)
        self.lib.ref_mat_copy(h, _p(cp, _i32p), _p(ri, _i32p), _p(va, _f64p))
        self.lib.ref_mat_free(h)
        return Csc(n.value, cp, ri[:nnz.value], va[:nnz.value])

    # ---- BASELINE.json configurations (the repo's generators, not libsfgpu)
    FULL_SIZE = {1: 512, 2: 64, 3: 96, 4: 1_000_000, 5: 128}

    def config_matrix(self, cfg: int, size: int | None = None, seed: int = 7,
                      halfwidth: int = 2000, nsys_perturb: int = 0, seed0: int = 1000):
        """The same inputs as paper_2111_12238_b200.config_matrix /
        config5_systems, generated by fixtures.cpp compiled into libsfref.so."""
        a = size or self.FULL_SIZE[cfg]
        b = halfwidth if cfg == 4 else 0
        h = C.c_void_p()
        if self.lib.refgen_matrix_gen(9 + cfg, a, b, seed, C.byref(h)) != 0:
            raise ValueError("bad generator parameters")
        try:
            n = C.c_int32()
            nnz = C.c_int64()
            self.lib.refgen_matrix_dims(h, C.byref(n), C.byref(nnz))
            cp = np.empty(n.value + 1, np.int32)
            ri = np.empty(max(nnz.value, 1), np.int32)
            va = np.empty(max(nnz.value, 1), np.float64)
            self.lib.refgen_matrix_copy(h, _p(cp, _i32p), _p(ri, _i32p), _p(va, _f64p))
            M = Csc(n.value, cp, ri[:nnz.value], va[:nnz.value])
            if nsys_perturb:
                vals = np.empty(nsys_perturb * nnz.value, np.float64)
                self.lib.refgen_matrix_perturb_diag(h, nsys_perturb, seed0, _p(vals, _f64p))
                return M, vals
            return M
        finally:
            self.lib.refgen_matrix_free(h)

    def fwd_bwd(self, M: Csc, b: np.ndarray) -> np.ndarray:
        """Config 5's pair from the reference's primitives:
        z = sptrsv(L, b); x from sptrsv on permute_symmetric(transpose(L), rev).
        Returns z ++ x."""
        out = np.empty(2 * M.n, np.float64)
        ei = C.c_int32(-1)
        msg = C.create_string_buffer(256)
        b = np.ascontiguousarray(b, np.float64)
        rc = self.lib.ref_fwd_bwd(M.n, _p(M.colptr, _i32p), _p(M.rowidx, _i32p),
                                  _p(M.values, _f64p), _p(b, _f64p), _p(out, _f64p),
                                  C.byref(ei), msg, 256)
        if rc:
            raise RuntimeError(msg.value.decode())
        return out

    def backward_matrix(self, M: Csc) -> Csc:
        """permute_symmetric(transpose(lower_triangle(M)), rev)."""
        h = self.lib.ref_backward_matrix(M.n, _p(M.colptr, _i32p), _p(M.rowidx, _i32p),
                                         _p(M.values, _f64p))
        if not h:
            raise ValueError("backward_matrix failed")
        n = C.c_int32()
        nnz = C.c_int32()
        self.lib.ref_mat_dims(h, C.byref(n), C.byref(nnz))
        cp = np.empty(n.value + 1, np.int32)
        ri = np.empty(max(nnz.value, 1), np.int32)
        va = np.empty(max(nnz.value, 1), np.float64)
        self.lib.ref_mat_copy(h, _p(cp, _i32p), _p(ri, _i32p), _p(va, _f64p))
        self.lib.ref_mat_free(h)
        return Csc(n.value, cp, ri[:nnz.value], va[:nnz.value])

    def solver(self, M: Csc, nthreads: int) -> "RefSolver":
        return RefSolver(self, M, nthreads)

    def read_matrix_market(self, path: str) -> Csc:
        """The reference's read_matrix_market (matrix_market.hpp:59-121).
        Runs in a child interpreter without numpy: the reference's iostream
        parsing crashed in a process that had imported numpy (not analysed
        further -- test infrastructure only)."""
        import json
        import subprocess
        import sys
        code = (
            "import ctypes as C, json, sys\n"
            f"L = C.CDLL({self.PATH!r})\n"
            "L.ref_read_mm.argtypes = [C.c_char_p, C.c_char_p, C.c_int]\n"
            "L.ref_read_mm.restype = C.c_void_p\n"
            "L.ref_mat_dims.argtypes = [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]\n"
            "L.ref_mat_copy.argtypes = [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_double)]\n"
            "msg = C.create_string_buffer(512)\n"
            "h = L.ref_read_mm(sys.argv[1].encode(), msg, 512)\n"
            "if not h:\n"
            "    print(json.dumps({'error': msg.value.decode()})); sys.exit(0)\n"
            "n = C.c_int32(); nnz = C.c_int32()\n"
            "L.ref_mat_dims(h, C.byref(n), C.byref(nnz))\n"
            "cp = (C.c_int32 * (n.value + 1))(); ri = (C.c_int32 * max(nnz.value, 1))()\n"
            "va = (C.c_double * max(nnz.value, 1))()\n"
            "L.ref_mat_copy(h, cp, ri, va)\n"
            "print(json.dumps({'n': n.value, 'cp': list(cp), 'ri': list(ri)[:nnz.value],"
            " 'va': [v.hex() for v in list(va)[:nnz.value]]}))\n")
        r = subprocess.run([sys.executable, "-c", code, path], capture_output=True, text=True,
                           check=True)
        d = json.loads(r.stdout)
        if "error" in d:
            raise ValueError(d["error"])
        return Csc(d["n"], np.array(d["cp"], np.int32), np.array(d["ri"], np.int32),
                   np.array([float.fromhex(v) for v in d["va"]], np.float64))

    def gen_grid_laplacian(self, k: int) -> Csc:
        return self._mat(0, k)

    def gen_banded_spd(self, n: int, bw: int, seed: int) -> Csc:
        return self._mat(1, n, bw, seed)

    def gen_dense_spd(self, n: int, seed: int) -> Csc:
        return self._mat(2, n, 0, seed)

    def fixture11_lower(self) -> Csc:
        return self._mat(3, 0)

    def fixture11_spmv(self) -> Csc:
        return self._mat(4, 0)

    # ---- state
    def state(self, combo: int, M: Csc, seed: int = 7, vin=None) -> "RefState":
        cp, ri, va = M.arrays()
        vin_a = None if vin is None else np.ascontiguousarray(vin, np.float64)
        ei = C.c_int32(-1)
        msg = C.create_string_buffer(256)
        h = self.lib.ref_state_new(combo, M.n, _p(cp, _i32p), _p(ri, _i32p), _p(va, _f64p),
                                   seed, _p(vin_a, _f64p), C.byref(ei), msg, 256)
        if not h:
            raise ValueError(msg.value.decode())
        return RefState(self, h)

    def state_fixture11(self, seed: int = 3) -> "RefState":
        return RefState(self, self.lib.ref_state_fixture11(seed))

    def _dag(self, h) -> Dag:
        nv = C.c_int32()
        ne = C.c_int64()
        self.lib.ref_dag_dims(h, C.byref(nv), C.byref(ne))
        sp = np.empty(nv.value + 1, np.int32)
        su = np.empty(max(ne.value, 1), np.int32)
        co = np.empty(max(nv.value, 1), np.int64)
        self.lib.ref_dag_copy(h, _p(sp, _i32p), _p(su, _i32p), _p(co, _i64p))
        return Dag(nv.value, sp, su[:ne.value], co[:nv.value])

    def _inter(self, h) -> InterDep:
        nr = C.c_int32()
        nc = C.c_int32()
        nnz = C.c_int64()
        self.lib.ref_inter_dims(h, C.byref(nr), C.byref(nc), C.byref(nnz))
        rp = np.empty(nr.value + 1, np.int32)
        ci = np.empty(max(nnz.value, 1), np.int32)
        self.lib.ref_inter_copy(h, _p(rp, _i32p), _p(ci, _i32p))
        return InterDep(nr.value, nc.value, rp, ci[:nnz.value])

    def _dag_handle(self, g: Dag):
        sp = np.ascontiguousarray(g.succptr, np.int32)
        su = np.ascontiguousarray(g.succ if len(g.succ) else np.zeros(1, np.int32), np.int32)
        co = np.ascontiguousarray(g.cost if len(g.cost) else np.zeros(1, np.int64), np.int64)
        return self.lib.ref_dag_from_csr(g.nvert, _p(sp, _i32p), _p(su, _i32p), _p(co, _i64p))

    def level_info(self, g: Dag) -> Levels:
        h = self._dag_handle(g)
        try:
            n = g.nvert
            lv = np.empty(max(n, 1), np.int32)
            ht = np.empty(max(n, 1), np.int32)
            sl = np.empty(max(n, 1), np.int32)
            P = C.c_int32()
            rc = self.lib.ref_level_info(h, _p(lv, _i32p), _p(ht, _i32p), _p(sl, _i32p),
                                         C.byref(P))
            if rc:
                raise ValueError("dependence cycle: edge does not ascend")
            return Levels(lv[:n], ht[:n], sl[:n], P.value)
        finally:
            self.lib.ref_dag_free(h)


class RefSolver:
    """L x = b with the reference's own parallel executor (kernel 1 of a
    combo-1 state under its LBC schedule, execute_unfused with an empty
    kernel-2 schedule; the schedule is built once)."""

    def __init__(self, ref: "Reference", M: Csc | None, nthreads: int, _handle=None):
        self.ref = ref
        if _handle is not None:
            self.h, self.n, self.inspector_s = _handle
            return
        self.n = M.n
        insp = C.c_double()
        self.h = ref.lib.ref_solver_new(M.n, _p(M.colptr, _i32p), _p(M.rowidx, _i32p),
                                        _p(M.values, _f64p), nthreads, C.byref(insp))
        if not self.h:
            raise RuntimeError("ref_solver_new failed")
        self.inspector_s = insp.value

    def with_diagonal(self, diag: np.ndarray) -> "RefSolver":
        """The same pattern and schedule, row i's diagonal set to diag[i]."""
        diag = np.ascontiguousarray(diag, np.float64)
        h = self.ref.lib.ref_solver_clone_diag(self.h, _p(diag, _f64p))
        if not h:
            raise RuntimeError("ref_solver_clone_diag failed")
        return RefSolver(self.ref, None, 0, _handle=(h, self.n, 0.0))

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.ref_solver_free(self.h)
            self.h = None

    def run(self, b: np.ndarray, x: np.ndarray | None = None) -> float:
        """x = L^-1 b; returns the executor's wall seconds."""
        b = np.ascontiguousarray(b, np.float64)
        wall = C.c_double()
        ei = C.c_int32(-1)
        msg = C.create_string_buffer(256)
        rc = self.ref.lib.ref_solver_run(self.h, _p(b, _f64p), _p(x, _f64p) if x is not None else None,
                                         C.byref(wall), C.byref(ei), msg, 256)
        if rc:
            raise RuntimeError(msg.value.decode())
        return wall.value


class RefState:
    """A reference KernelState (kernels.hpp:409-427) behind a handle."""

    def __init__(self, ref: Reference, h):
        self.ref = ref
        self.h = h

    def __del__(self):
        try:
            self.ref.lib.ref_state_free(self.h)
        except Exception:
            pass

    def execute(self, executor: int = 0, nthreads: int = 1) -> np.ndarray:
        """0 sequential, 1 fused (msp), 2 unfused, 3 joint wavefront."""
        L = self.ref.lib
        cap = max(L.ref_output_len(self.h), 1)
        out = np.empty(cap, np.float64)
        ei = C.c_int32(-1)
        msg = C.create_string_buffer(256)
        rc = L.ref_execute(self.h, executor, nthreads, _p(out, _f64p), cap, C.byref(ei), msg, 256)
        if rc == 1:
            text = msg.value.decode()
            raise FactorizationError(text.rsplit(" at index", 1)[0], ei.value)
        if rc:
            raise ValueError(msg.value.decode())
        return out[:L.ref_output_len(self.h)]

    def validate_partitioning(self, s_ptr, w_ptr, tags, iters) -> tuple:
        """validate_fused_partitioning (msp.hpp:1108-1237) of an external
        partitioning in flat form; returns (violations, first message)."""
        sp = np.ascontiguousarray(s_ptr, np.int64)
        wp = np.ascontiguousarray(w_ptr, np.int64)
        tg = np.ascontiguousarray(tags, np.uint8)
        it = np.ascontiguousarray(iters, np.int32)
        msg = C.create_string_buffer(512)
        nbad = self.ref.lib.ref_validate_partitioning(
            self.h, len(sp) - 1, _p(sp, _i64p), _p(wp, _i64p),
            tg.ctypes.data_as(C.POINTER(C.c_uint8)), _p(it, _i32p), msg, 512)
        return int(nbad), msg.value.decode()

    def replay_partitioning(self, s_ptr, w_ptr, tags, iters, seed: int) -> np.ndarray:
        """replay_schedule (executor.hpp:518-553) of an external partitioning
        in flat form; returns collect_outputs."""
        sp = np.ascontiguousarray(s_ptr, np.int64)
        wp = np.ascontiguousarray(w_ptr, np.int64)
        tg = np.ascontiguousarray(tags, np.uint8)
        it = np.ascontiguousarray(iters, np.int32)
        n = int(self.ref.lib.ref_output_len(self.h))
        out = np.empty(max(n, 1), np.float64)
        ei = C.c_int32(-1)
        msg = C.create_string_buffer(512)
        rc = self.ref.lib.ref_replay_partitioning(
            self.h, len(sp) - 1, _p(sp, _i64p), _p(wp, _i64p),
            tg.ctypes.data_as(C.POINTER(C.c_uint8)), _p(it, _i32p), seed, _p(out, _f64p), len(out),
            C.byref(ei), msg, 512)
        if rc:
            raise RuntimeError(msg.value.decode())
        return out[:n]

    def bench(self, executor: int, nthreads: int, warmups: int = 2, repeats: int = 5):
        """Returns (per-repeat seconds, inspector seconds, s-partitions)."""
        times = np.zeros(repeats, np.float64)
        insp = C.c_double()
        nsp = C.c_int32()
        msg = C.create_string_buffer(256)
        rc = self.ref.lib.ref_bench(self.h, executor, nthreads, warmups, repeats,
                                    _p(times, _f64p), C.byref(insp), C.byref(nsp), msg, 256)
        if rc:
            raise RuntimeError(msg.value.decode())
        return times, insp.value, nsp.value

    def build_g(self, which: int) -> Dag:
        h = self.ref.lib.ref_build_g(self.h, which)
        try:
            return self.ref._dag(h)
        finally:
            self.ref.lib.ref_dag_free(h)

    def inter_dag(self) -> InterDep:
        h = self.ref.lib.ref_inter_dag(self.h)
        try:
            return self.ref._inter(h)
        finally:
            self.ref.lib.ref_inter_free(h)

    def joint_dag(self) -> Dag:
        L = self.ref.lib
        g1 = L.ref_build_g(self.h, 1)
        g2 = L.ref_build_g(self.h, 2)
        f = L.ref_inter_dag(self.h)
        j = L.ref_joint_dag(g1, g2, f)
        try:
            return self.ref._dag(j)
        finally:
            for h in (g1, g2, j):
                L.ref_dag_free(h)
            L.ref_inter_free(f)

    def compute_reuse(self) -> float:
        return self.ref.lib.ref_compute_reuse(self.h)

    def wavefront(self):
        """Level sets of the joint DAG (executor.hpp:209-229)."""
        L = self.ref.lib
        nl = C.c_int32()
        ne = L.ref_wavefront(self.h, None, None, None, C.byref(nl))
        tags = np.empty(max(ne, 1), np.uint8)
        iters = np.empty(max(ne, 1), np.int32)
        lp = np.empty(nl.value + 1, np.int32)
        L.ref_wavefront(self.h, tags.ctypes.data_as(C.POINTER(C.c_uint8)), _p(iters, _i32p),
                        _p(lp, _i32p), C.byref(nl))
        return tags[:ne], iters[:ne], lp
