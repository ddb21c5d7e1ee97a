"""Host-side mirror of the reference inspector/executor API (namespace
``sparsefuse``, proj/include/sparsefuse/*.hpp) over the C-ABI.

Same names, argument meaning and error behaviour as the reference, so code
written against it ports line for line::

    st  = make_state(5, M, seed=7)              # kernels.hpp:429
    g1  = build_g1(st); g2 = build_g2(st)       # dag.hpp:319,339
    f   = inter_dag(st)                         # dag.hpp:279
    j   = joint_dag(st)                         # dag.hpp:222 (built on the GPU)
    li  = level_info(st, 3)                     # dag.hpp:197
    sch = make_fused_schedule(st)               # msp + compile_schedule
    execute_fused(sch, st)                      # executor.hpp:395
    out = collect_outputs(st)                   # kernels.hpp:585

Numeric breakdown raises ``FactorizationError`` with the failing index
(types.hpp:17-26); invalid input raises ``InvalidMatrixError``.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import weakref

import numpy as np

from . import abi
from .abi import f64p, i32p, i64p, ptr, u8p

# kernels.hpp:53-68 plus combo 8 (forward L, backward L^T; BASELINE config 5)
COMBOS = {
    1: ("sptrsv-sptrsv", "x = inv(L)*y; z = inv(L)*x"),
    2: ("spmv-sptrsv", "y = A*x; z = inv(L)*y"),
    3: ("dscal-spilu0", "LU ~= D*A*D'"),
    4: ("sptrsv-spmv", "y = inv(L)*x; z = A*y"),
    5: ("spic0-sptrsv", "L*L' ~= A; y = inv(L)*x"),
    6: ("spilu0-sptrsv", "LU ~= A; y = inv(L)*x"),
    7: ("dscal-spic0", "L*L' ~= D*A*D'"),
    8: ("sptrsv-sptrsvT", "z = inv(L)*b; x = inv(L')*z"),
}


class FactorizationError(RuntimeError):
    """sparsefuse::FactorizationError (types.hpp:17-26)."""

    def __init__(self, what: str, index: int, kind: int = 0):
        super().__init__(what)
        self.index = index
        self.kind = kind


class InvalidMatrixError(RuntimeError):
    """sparsefuse::InvalidMatrixError (types.hpp:28-31)."""


class NoDeviceError(RuntimeError):
    """No CUDA device: this library has no CPU fallback by design."""


@dataclass
class CscMatrix:
    """CscMatrix (matrix.hpp:18-26)."""

    n: int
    colptr: np.ndarray
    rowidx: np.ndarray
    values: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.colptr[-1])


@dataclass
class DepDag:
    """DepDag (dag.hpp:17-30).  ``origin`` (a weak reference to the
    KernelState it was built from, or None) lets msp / joint_dag / the
    executors use that state's GPU inspector."""

    nvert: int
    succptr: np.ndarray
    succ: np.ndarray
    cost: np.ndarray
    origin: object = None

    def nedges(self) -> int:
        return int(self.succptr[-1]) if len(self.succptr) else 0


@dataclass
class InterDep:
    """InterDep F (dag.hpp:34-41)."""

    nrows: int
    ncols: int
    rowptr: np.ndarray
    colidx: np.ndarray
    origin: object = None


@dataclass
class LevelInfo:
    """LevelInfo (dag.hpp:43-48)."""

    level: np.ndarray
    height: np.ndarray
    slack: np.ndarray
    critical_path: int


@dataclass
class FusedSchedule:
    """FusedSchedule (executor.hpp:138-150) in flat form: entries (tag, iter)
    in execution order, grouped into s-partitions by ``wave_ptr``.
    ``checked_for``: weak reference to the KernelState the entries were
    verified against (execute_fused verifies any other schedule first)."""

    tags: np.ndarray
    iters: np.ndarray
    wave_ptr: np.ndarray
    interleaved: bool = False
    fusion: bool = True
    checked_for: object = None

    def nspartitions(self) -> int:
        return len(self.wave_ptr) - 1


@dataclass
class WavefrontSchedule:
    """WavefrontSchedule (executor.hpp:152-156): the joint DAG's level sets,
    level l = entries [level_ptr[l], level_ptr[l+1])."""

    tags: np.ndarray
    iters: np.ndarray
    level_ptr: np.ndarray

    def nlevels(self) -> int:
        return len(self.level_ptr) - 1


@dataclass
class FusedPartitioning:
    """FusedPartitioning (msp.hpp:44-63) in flat form: s-partition k holds
    w-partitions [s_ptr[k], s_ptr[k+1]); w-partition w holds the ordered
    (tag, iter) entries [w_ptr[w], w_ptr[w+1])."""

    s_ptr: np.ndarray
    w_ptr: np.ndarray
    tags: np.ndarray
    iters: np.ndarray
    interleaved: bool = False
    reuse_ratio: float = 0.0
    fusion: bool = True
    origin: object = None

    def b(self) -> int:
        return len(self.s_ptr) - 1

    def spartitions(self):
        """Nested [s][w] lists of (tag, iter), the reference's layout."""
        out = []
        for k in range(self.b()):
            ws = []
            for w in range(self.s_ptr[k], self.s_ptr[k + 1]):
                e0, e1 = self.w_ptr[w], self.w_ptr[w + 1]
                ws.append(list(zip(self.tags[e0:e1].tolist(), self.iters[e0:e1].tolist())))
            out.append(ws)
        return out


def _raise(L, h, st: int, what: str):
    if st == abi.SFG_OK:
        return
    kind = C.c_int32(0)
    idx = C.c_int32(-1)
    msg = C.create_string_buffer(512)
    if h:
        L.sfg_last_error(h, C.byref(kind), C.byref(idx), msg, 512)
    text = msg.value.decode() or what
    if st == abi.SFG_ERR_FACTORIZATION:
        raise FactorizationError(text, idx.value, kind.value)
    if st == abi.SFG_ERR_INVALID_MATRIX:
        raise InvalidMatrixError(text)
    if st == abi.SFG_ERR_INVALID_ARGUMENT:
        raise ValueError(text)
    if st == abi.SFG_ERR_NO_DEVICE:
        raise NoDeviceError("no CUDA device: sfgpu runs on sm_100a only (no CPU fallback)")
    if st == abi.SFG_ERR_LOGIC:
        raise RuntimeError(text)
    raise RuntimeError(f"{what}: {text} (status {st})")


class KernelState:
    """A KernelState (kernels.hpp:409-427) resident in GPU memory."""

    def __init__(self, combo: int, M: CscMatrix, seed: int = 7, nsys: int = 1,
                 values: np.ndarray | None = None, vin: np.ndarray | None = None):
        self.L = abi.load()
        self.combo = combo
        self.n = M.n
        self.nsys = nsys
        self.nnz_m = int(M.nnz)
        cp = np.ascontiguousarray(M.colptr, np.int32)
        ri = np.ascontiguousarray(M.rowidx, np.int32)
        va = np.ascontiguousarray(M.values if values is None else values, np.float64)
        if values is not None and va.size != nsys * M.nnz:
            raise ValueError("values must hold nsys * nnz doubles")
        vi = None if vin is None else np.ascontiguousarray(vin, np.float64)
        h = C.c_void_p()
        st = self.L.sfg_plan_create(combo, M.n, ptr(cp, i32p), ptr(ri, i32p), ptr(va, f64p),
                                    nsys, ptr(vi, f64p), seed, C.byref(h))
        self.h = h.value
        if st != abi.SFG_OK:
            try:
                _raise(self.L, self.h, st, "make_state")
            finally:
                self.close()
        info = [C.c_int32(), C.c_int32(), C.c_int32(), C.c_int64(), C.c_int64()]
        self.L.sfg_plan_info(self.h, *[C.byref(x) for x in info])
        self.nnz_factor = info[3].value
        self.output_len = info[4].value
        self.inspected = False

    def close(self):
        if getattr(self, "h", None):
            self.L.sfg_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _chk(self, st, what):
        _raise(self.L, self.h, st, what)

    # ---- inputs
    def set_vin(self, vin: np.ndarray):
        v = np.ascontiguousarray(vin, np.float64)
        if v.size != self.n * self.nsys:
            raise ValueError("vin must hold nsys * n doubles")
        self._chk(self.L.sfg_set_vin(self.h, ptr(v, f64p)), "set_vin")

    def set_values(self, values: np.ndarray):
        """New matrix values, same pattern (nsys * nnz(M), plan_create layout)."""
        v = np.ascontiguousarray(values, np.float64)
        if v.size != self.nnz_m * self.nsys:
            raise ValueError("values must hold nsys * nnz(M) doubles")
        self._chk(self.L.sfg_set_values(self.h, ptr(v, f64p)), "set_values")

    def set_stream(self, stream_handle: int | None):
        self._chk(self.L.sfg_plan_set_stream(self.h, stream_handle or None), "set_stream")

    # ---- inspector
    def inspect(self):
        self._chk(self.L.sfg_inspect(self.h), "inspect")
        self.inspected = True
        return self

    def dag(self, which: int) -> DepDag:
        nv = C.c_int32()
        ne = C.c_int64()
        self._chk(self.L.sfg_get_dag(self.h, which, C.byref(nv), C.byref(ne), None, None, None),
                  "dag")
        sp = np.empty(nv.value + 1, np.int32)
        su = np.empty(max(ne.value, 1), np.int32)
        co = np.empty(max(nv.value, 1), np.int64)
        self._chk(self.L.sfg_get_dag(self.h, which, None, None, ptr(sp, i32p), ptr(su, i32p),
                                     ptr(co, i64p)), "dag")
        return DepDag(nv.value, sp, su[:ne.value], co[:nv.value], weakref.ref(self))

    def inter_dag(self) -> InterDep:
        nr = C.c_int32()
        nc = C.c_int32()
        nnz = C.c_int64()
        self._chk(self.L.sfg_get_interdep(self.h, C.byref(nr), C.byref(nc), C.byref(nnz), None,
                                          None), "inter_dag")
        rp = np.empty(nr.value + 1, np.int32)
        ci = np.empty(max(nnz.value, 1), np.int32)
        self._chk(self.L.sfg_get_interdep(self.h, None, None, None, ptr(rp, i32p),
                                          ptr(ci, i32p)), "inter_dag")
        return InterDep(nr.value, nc.value, rp, ci[:nnz.value], weakref.ref(self))

    def level_info(self, which: int) -> LevelInfo:
        nv = self.n if which < 3 else 2 * self.n
        lv = np.empty(max(nv, 1), np.int32)
        ht = np.empty(max(nv, 1), np.int32)
        sl = np.empty(max(nv, 1), np.int32)
        P = C.c_int32()
        self._chk(self.L.sfg_get_levels(self.h, which, ptr(lv, i32p), ptr(ht, i32p),
                                        ptr(sl, i32p), C.byref(P)), "level_info")
        return LevelInfo(lv[:nv], ht[:nv], sl[:nv], P.value)

    def compute_reuse(self) -> float:
        r = C.c_double()
        self._chk(self.L.sfg_compute_reuse(self.h, C.byref(r)), "compute_reuse")
        return r.value

    def schedule(self) -> FusedSchedule:
        ne = C.c_int64()
        nw = C.c_int32()
        self._chk(self.L.sfg_get_schedule(self.h, C.byref(ne), None, None, C.byref(nw), None),
                  "schedule")
        tags = np.empty(max(ne.value, 1), np.uint8)
        iters = np.empty(max(ne.value, 1), np.int32)
        wp = np.empty(nw.value + 1, np.int64)
        self._chk(self.L.sfg_get_schedule(self.h, None, ptr(tags, u8p), ptr(iters, i32p), None,
                                          ptr(wp, i64p)), "schedule")
        return FusedSchedule(tags[:ne.value], iters[:ne.value], wp)

    def partitioning(self) -> "FusedPartitioning":
        """The schedule as the reference's FusedPartitioning (msp.hpp:44-63)."""
        if not self.inspected:
            self.inspect()
        ns = C.c_int32()
        nw = C.c_int64()
        ne = C.c_int64()
        self._chk(self.L.sfg_get_partitioning(self.h, C.byref(ns), C.byref(nw), C.byref(ne),
                                              None, None, None, None), "partitioning")
        sp = np.empty(ns.value + 1, np.int64)
        wp = np.empty(nw.value + 1, np.int64)
        tags = np.empty(max(ne.value, 1), np.uint8)
        iters = np.empty(max(ne.value, 1), np.int32)
        self._chk(self.L.sfg_get_partitioning(self.h, None, None, None, ptr(sp, i64p),
                                              ptr(wp, i64p), ptr(tags, u8p), ptr(iters, i32p)),
                  "partitioning")
        r = self.compute_reuse()
        return FusedPartitioning(sp, wp, tags[:ne.value], iters[:ne.value], r >= 1.0, r, True,
                                 weakref.ref(self))

    def wavefront(self) -> "WavefrontSchedule":
        """The joint DAG's level sets (build_wavefront_schedule,
        executor.hpp:209-229), built on the GPU."""
        ne = C.c_int64()
        nl = C.c_int32()
        self._chk(self.L.sfg_get_wavefront(self.h, C.byref(ne), None, None, C.byref(nl), None),
                  "wavefront")
        tags = np.empty(max(ne.value, 1), np.uint8)
        iters = np.empty(max(ne.value, 1), np.int32)
        lp = np.empty(nl.value + 1, np.int64)
        self._chk(self.L.sfg_get_wavefront(self.h, None, ptr(tags, u8p), ptr(iters, i32p), None,
                                           ptr(lp, i64p)), "wavefront")
        return WavefrontSchedule(tags[:ne.value], iters[:ne.value], lp)

    def check_schedule(self, tags: np.ndarray, iters: np.ndarray) -> int:
        """Violations of a flattened schedule against this state's joint DAG
        (sfg_check_schedule): missing / repeated iterations and dependences
        out of order.  0 = a valid order."""
        tags = np.ascontiguousarray(tags, np.uint8)
        iters = np.ascontiguousarray(iters, np.int32)
        bad = C.c_int64()
        self._chk(self.L.sfg_check_schedule(self.h, len(tags), ptr(tags, u8p), ptr(iters, i32p),
                                            C.byref(bad)), "check_schedule")
        return int(bad.value)

    def execute_wavefront(self, sync: bool = True):
        """execute_joint_wavefront (executor.hpp:465-507) on the GPU."""
        self._chk(self.L.sfg_execute_wavefront(self.h), "execute_joint_wavefront")
        if sync:
            self.synchronize()

    def execute_sequential(self, sync: bool = True):
        """execute_sequential (executor.hpp:315-322): the reference loop on one
        GPU thread."""
        self._chk(self.L.sfg_execute_sequential(self.h), "execute_sequential")
        if sync:
            self.synchronize()

    def reset(self):
        """reset (kernels.hpp:498-502): fac = fac0, vmid = vout = 0."""
        self._chk(self.L.sfg_reset(self.h), "reset")

    # ---- executor
    def execute_fused(self, sync: bool = True):
        if not self.inspected:
            self.inspect()
        self._chk(self.L.sfg_execute_fused(self.h), "execute_fused")
        if sync:
            self.synchronize()

    def execute_batch(self, vins, outs, final_only: bool = False):
        """len(vins) executions with new input vectors, transfers overlapped
        with compute (sfg_execute_batch_ex); vins[k] / outs[k] are host arrays
        (page-locked for the overlap) of nsys*n doubles and nsys*output_len
        doubles -- or, with final_only, nsys*n doubles of kernel 2's output."""
        if not self.inspected:
            self.inspect()
        k = len(vins)
        if len(outs) != k:
            raise ValueError("one output buffer per input")
        need = self.n * self.nsys if final_only else self.output_len * self.nsys
        for v in vins:
            if v.dtype != np.float64 or v.size != self.n * self.nsys or not v.flags.c_contiguous:
                raise ValueError("vin must be contiguous float64 of nsys * n")
        for o in outs:
            if o.dtype != np.float64 or o.size < need or not o.flags.c_contiguous:
                raise ValueError(f"out must be contiguous float64 of {need} doubles")
        vp = (C.c_void_p * max(k, 1))(*[v.ctypes.data for v in vins])
        op = (C.c_void_p * max(k, 1))(*[o.ctypes.data for o in outs])
        self._chk(self.L.sfg_execute_batch_ex(self.h, k, vp, op, 1 if final_only else 0),
                  "execute_batch")

    def execute_kernel(self, which: int, sync: bool = True):
        """Kernel 1 or kernel 2 of the pair alone (sfg_execute_kernel)."""
        if not self.inspected:
            self.inspect()
        self._chk(self.L.sfg_execute_kernel(self.h, which), "execute_kernel")
        if sync:
            self.synchronize()

    def spmv_rows(self, r0: int, r1: int, x_device: int, y_device: int):
        """y[0:r1-r0] = A[r0:r1, :] x on device pointers (sfg_spmv_rows)."""
        self._chk(self.L.sfg_spmv_rows(self.h, r0, r1, x_device, y_device), "spmv_rows")

    def execute_unfused(self, sync: bool = True):
        if not self.inspected:
            self.inspect()
        self._chk(self.L.sfg_execute_unfused(self.h), "execute_unfused")
        if sync:
            self.synchronize()

    def synchronize(self):
        self._chk(self.L.sfg_synchronize(self.h), "synchronize")

    def collect_outputs(self, out: np.ndarray | None = None) -> np.ndarray:
        """All systems' collect_outputs, concatenated system-major."""
        need = self.output_len * self.nsys
        if out is None:
            out = np.empty(max(need, 1), np.float64)
        self._chk(self.L.sfg_collect_outputs(self.h, ptr(out, f64p), out.size), "collect_outputs")
        return out[:need]

    def last_exec_ms(self):
        tot = C.c_float()
        ker = C.c_float()
        self._chk(self.L.sfg_last_exec_ms(self.h, C.byref(tot), C.byref(ker)), "last_exec_ms")
        return tot.value, ker.value

    def bench(self, reps: int, unfused: bool | int = False):
        """reps back-to-back executions timed with CUDA events on the plan
        stream: (total_ms, mean main-kernel ms).  unfused: False/0 fused,
        True/1 the two-launch comparator, 2 the joint wavefront executor."""
        if not self.inspected:
            self.inspect()
        tot = C.c_float()
        ker = C.c_float()
        self._chk(self.L.sfg_bench_executions(self.h, reps, int(unfused), C.byref(tot),
                                              C.byref(ker)), "bench")
        return tot.value, ker.value

    def launch_count(self) -> int:
        return int(self.L.sfg_launch_count(self.h))

    def device_output(self, which: int):
        p = C.c_void_p()
        cnt = C.c_int64()
        self._chk(self.L.sfg_device_output(self.h, which, C.byref(p), C.byref(cnt)),
                  "device_output")
        return p.value, cnt.value


# ---- free functions with the reference's names --------------------------------
def make_state(combo: int, M: CscMatrix, seed: int = 7, **kw) -> KernelState:
    """make_state (kernels.hpp:429-495); storage conversions run on the GPU."""
    return KernelState(combo, M, seed, **kw)


def build_g1(st: KernelState) -> DepDag:
    return st.dag(1)


def build_g2(st: KernelState) -> DepDag:
    return st.dag(2)


def inter_dag(st: KernelState) -> InterDep:
    return st.inter_dag()


def _state_of(*objs):
    """The live KernelState every object was built from, or None."""
    st = None
    for o in objs:
        ref = getattr(o, "origin", None)
        s = ref() if ref is not None else None
        if s is None or (st is not None and s is not st):
            return None
        st = s
    return st


def joint_dag(st_or_g1, g2: DepDag | None = None, f: InterDep | None = None) -> DepDag:
    """joint_dag (dag.hpp:222-238): joint_dag(st) from the state's GPU
    inspector, or joint_dag(g1, g2, f) from the structures (edges of G1, G2
    offset by |V1|, (j, |V1| + i) per F_ij; sorted, duplicate-free)."""
    if isinstance(st_or_g1, KernelState):
        return st_or_g1.dag(3)
    g1 = st_or_g1
    st = _state_of(g1, g2, f)
    if st is not None:
        return st.dag(3)
    n1 = g1.nvert
    src = [np.repeat(np.arange(n1, dtype=np.int64), np.diff(g1.succptr)),
           n1 + np.repeat(np.arange(g2.nvert, dtype=np.int64), np.diff(g2.succptr)),
           np.asarray(f.colidx[:int(f.rowptr[-1])], np.int64)]
    dst = [np.asarray(g1.succ[:g1.nedges()], np.int64), n1 + np.asarray(g2.succ[:g2.nedges()], np.int64),
           n1 + np.repeat(np.arange(f.nrows, dtype=np.int64), np.diff(f.rowptr))]
    nv = n1 + g2.nvert
    key = np.unique(np.concatenate(src) * nv + np.concatenate(dst))
    u, v = key // max(nv, 1), key % max(nv, 1)
    sp = np.zeros(nv + 1, np.int32)
    np.add.at(sp, u + 1, 1)
    return DepDag(nv, np.cumsum(sp).astype(np.int32), v.astype(np.int32),
                  np.concatenate([g1.cost, g2.cost]).astype(np.int64))


def level_info(st_or_dag, which: int = 3) -> LevelInfo:
    """level_info (dag.hpp:197-218) of a state's G1/G2/joint DAG, or of any
    DepDag (computed on the GPU, sfg_dag_levels)."""
    if isinstance(st_or_dag, KernelState):
        return st_or_dag.level_info(which)
    g = st_or_dag
    L = abi.load()
    nv = g.nvert
    sp = np.ascontiguousarray(g.succptr, np.int32)
    su = np.ascontiguousarray(g.succ if len(g.succ) else np.zeros(1, np.int32), np.int32)
    lv, ht, sl = (np.empty(max(nv, 1), np.int32) for _ in range(3))
    P = C.c_int32()
    st = L.sfg_dag_levels(nv, ptr(sp, i32p), ptr(su, i32p), ptr(lv, i32p), ptr(ht, i32p),
                          ptr(sl, i32p), C.byref(P))
    if st == abi.SFG_ERR_INVALID_ARGUMENT:
        raise ValueError("dependence cycle: edge does not ascend")
    _raise(L, None, st, "level_info")
    return LevelInfo(lv[:nv], ht[:nv], sl[:nv], P.value)


def compute_reuse(st: KernelState) -> float:
    return st.compute_reuse()


def msp(g1: DepDag, g2: DepDag, f: InterDep, r: int, reuse_ratio: float,
        redundancy_factor: float = 2.0) -> FusedPartitioning:
    """msp (msp.hpp:825-1082).  DAGs of a live state: that state's GPU
    inspector partitioning (what execute_fused runs).  Otherwise the joint
    DAG's level sets, each split into at most r contiguous w-partitions --
    a valid fused partitioning of any DAG pair.  Packing is interleaved iff
    reuse_ratio >= 1 (msp.hpp:834)."""
    if r < 1:
        raise ValueError("partition count must be >= 1")
    st = _state_of(g1, g2, f)
    if st is not None:
        V = st.partitioning()
        V.reuse_ratio = reuse_ratio
        V.interleaved = reuse_ratio >= 1.0
        return V
    ws = build_wavefront_schedule(g1, g2, f)
    s_ptr, w_ptr = [0], [0]
    for l in range(ws.nlevels()):
        b, e = int(ws.level_ptr[l]), int(ws.level_ptr[l + 1])
        parts = min(r, e - b)
        for w in range(parts):
            w_ptr.append(b + (w + 1) * (e - b) // parts)
        s_ptr.append(len(w_ptr) - 1)
    return FusedPartitioning(np.array(s_ptr, np.int64), np.array(w_ptr, np.int64), ws.tags,
                             ws.iters, reuse_ratio >= 1.0, reuse_ratio)


def validate_fused_partitioning(V: FusedPartitioning, g1: DepDag, g2: DepDag,
                                f: InterDep) -> list:
    """validate_fused_partitioning (msp.hpp:1110-1237): coverage, duplicate
    provenance, within-partition order and the cross-partition invariant,
    with the reference's messages; [] means valid."""
    bad = []
    if not V.fusion:
        return ["fusion disabled but schedule non-empty"] if V.b() else []
    n1, n2 = g1.nvert, g2.nvert
    pos1 = [[] for _ in range(n1)]
    pos2 = [None] * n2
    cnt2 = [0] * n2
    for s in range(V.b()):
        for w in range(int(V.s_ptr[s]), int(V.s_ptr[s + 1])):
            for e, q in enumerate(range(int(V.w_ptr[w]), int(V.w_ptr[w + 1]))):
                tag, it = int(V.tags[q]), int(V.iters[q])
                wl = w - int(V.s_ptr[s])
                where = f"(s={s},w={wl},entry={e}): "
                if tag == 1:
                    if not 0 <= it < n1:
                        bad.append(where + "kernel-1 iteration out of range")
                    else:
                        pos1[it].append((s, wl, e, w))
                elif not 0 <= it < n2:
                    bad.append(where + "kernel-2 iteration out of range")
                else:
                    cnt2[it] += 1
                    if cnt2[it] > 1:
                        bad.append(where + "kernel-2 iteration duplicated")
                    pos2[it] = (s, wl, e, w)
    bad += [f"kernel-1 iteration {v} missing" for v in range(n1) if not pos1[v]]
    bad += [f"kernel-2 iteration {v} missing" for v in range(n2) if cnt2[v] == 0]
    if bad:
        return bad
    for v in range(n1):
        if len(pos1[v]) > 1:
            bad.append(f"(s={pos1[v][0][0]},w={pos1[v][0][1]},entry={pos1[v][0][2]}): "
                       "replicated entry not flagged dup")
    def before(p, u, tag):
        w0 = int(V.w_ptr[p[3]])
        return any(int(V.tags[w0 + k]) == tag and int(V.iters[w0 + k]) == u for k in range(p[2]))
    def earliest1(u):
        return min(p[0] for p in pos1[u])
    def preds(g):
        pr = [[] for _ in range(g.nvert)]
        for u in range(g.nvert):
            for p in range(int(g.succptr[u]), int(g.succptr[u + 1])):
                pr[int(g.succ[p])].append(u)
        return pr
    p1, p2 = preds(g1), preds(g2)
    for v in range(n1):
        for pv in pos1[v]:
            for u in p1[v]:
                if not before(pv, u, 1) and earliest1(u) >= pv[0]:
                    bad.append(f"(s={pv[0]},w={pv[1]},entry={pv[2]}): kernel-1 dependence on {u} unsatisfied")
    for v in range(n2):
        pv = pos2[v]
        for u in p2[v]:
            pu = pos2[u]
            if not (pu[0] < pv[0] or (pu[0] == pv[0] and pu[1] == pv[1] and pu[2] < pv[2])):
                bad.append(f"(s={pv[0]},w={pv[1]},entry={pv[2]}): kernel-2 dependence on {u} unsatisfied")
        for p in range(int(f.rowptr[v]), int(f.rowptr[v + 1])):
            u = int(f.colidx[p])
            if not before(pv, u, 1) and earliest1(u) >= pv[0]:
                bad.append(f"(s={pv[0]},w={pv[1]},entry={pv[2]}): cross-kernel dependence on {u} unsatisfied")
    return bad


def compile_schedule(V: FusedPartitioning, reuse_ratio: float, g1: DepDag, g2: DepDag,
                     r: int = 1) -> FusedSchedule:
    """compile_schedule (executor.hpp:235-268): flattens V; interleaved iff
    reuse_ratio >= 1.  The entries are verified against the state the DAGs
    came from, when it is alive."""
    wave = np.asarray([V.w_ptr[int(k)] for k in V.s_ptr], np.int64)
    fs = FusedSchedule(np.asarray(V.tags, np.uint8), np.asarray(V.iters, np.int32), wave,
                       reuse_ratio >= 1.0, V.fusion)
    st = _state_of(g1, g2)
    if st is not None and st.check_schedule(fs.tags, fs.iters) == 0:
        fs.checked_for = weakref.ref(st)
    return fs


def make_fused_schedule(st: KernelState) -> FusedSchedule:
    """The state's own schedule (the GPU inspector replaces msp +
    compile_schedule)."""
    st.inspect()
    fs = st.schedule()
    fs.interleaved = st.compute_reuse() >= 1.0
    fs.checked_for = weakref.ref(st)
    return fs


def _verified(sched: FusedSchedule | None, st: KernelState) -> None:
    if sched is None:
        return
    ref = sched.checked_for
    if ref is not None and ref() is st:
        return
    if not sched.fusion:
        raise RuntimeError("execute_fused: fusion disabled, run the fallback schedule")
    bad = st.check_schedule(sched.tags, sched.iters)
    if bad:
        raise ValueError(f"execute_fused: schedule violates the joint DAG of this state ({bad} violations)")


def execute_fused(sched: FusedSchedule | None, st: KernelState, nthreads: int | None = None):
    """execute_fused (executor.hpp:395-461) on the GPU.  A schedule not
    verified for this state is checked against its joint DAG first
    (ValueError if an iteration is missing/repeated or a dependence is out of
    order); any valid order computes the same result, so the state's own
    executor runs it.  ``nthreads`` has no GPU meaning."""
    _verified(sched, st)
    st.execute_fused()


def _same_state(st: KernelState, *objs):
    for o in objs:
        ref = getattr(o, "origin", None)
        if ref is not None and ref() is not st:
            raise ValueError("the DAGs do not belong to this KernelState")


def execute_unfused(st_or_g1, g2: DepDag | None = None, st: KernelState | None = None,
                    nthreads: int | None = None):
    """execute_unfused(st) or execute_unfused(g1, g2, st, T) (executor.hpp:325-392)."""
    if isinstance(st_or_g1, KernelState):
        st_or_g1.execute_unfused()
        return
    _same_state(st, st_or_g1, g2)
    st.execute_unfused()


def build_wavefront_schedule(g1: DepDag, g2: DepDag, f: InterDep) -> WavefrontSchedule:
    """build_wavefront_schedule (executor.hpp:209-229): joint level sets,
    ascending vertex id within a level (the GPU inspector's for DAGs of a live
    state; otherwise from the joint DAG's GPU-computed levels)."""
    st = _state_of(g1, g2, f)
    if st is not None:
        return st.wavefront()
    j = joint_dag(g1, g2, f)
    li = level_info(j)
    order = np.lexsort((np.arange(j.nvert), li.level))
    counts = np.bincount(li.level, minlength=li.critical_path + 1)[1:]
    lp = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    tags = np.where(order < g1.nvert, 1, 2).astype(np.uint8)
    iters = np.where(order < g1.nvert, order, order - g1.nvert).astype(np.int32)
    return WavefrontSchedule(tags, iters, lp)


def execute_joint_wavefront(g1: DepDag, g2: DepDag, f: InterDep, st: KernelState,
                            nthreads: int | None = None):
    """execute_joint_wavefront (executor.hpp:465-507): the joint level sets
    in order with a grid barrier between levels (sfg_execute_wavefront)."""
    _same_state(st, g1, g2, f)
    st.execute_wavefront()


def execute_sequential(st: KernelState):
    """execute_sequential (executor.hpp:315-322) on one GPU thread."""
    st.execute_sequential()


def run_sequential_reference(st: KernelState):
    st.execute_sequential()


def reset(st: KernelState):
    """reset (kernels.hpp:498-502): fac = fac0, vmid = vout = 0 (device)."""
    st.reset()


def collect_outputs(st: KernelState) -> np.ndarray:
    return st.collect_outputs()


def gen_vector(n: int, seed: int) -> np.ndarray:
    """gen_vector (fixtures.hpp:148-155)."""
    out = np.empty(max(n, 1), np.float64)
    abi.load().sfg_gen_vector(n, seed, ptr(out, f64p))
    return out[:n]


class PCG:
    """Preconditioned CG on the GPU with the IC0 factor (combo 5) and the fused
    forward/backward solve (combo 8) as M^-1 (sfg_pcg_*)."""

    def __init__(self, M: CscMatrix):
        self.L = abi.load()
        self.n = M.n
        cp = np.ascontiguousarray(M.colptr, np.int32)
        ri = np.ascontiguousarray(M.rowidx, np.int32)
        va = np.ascontiguousarray(M.values, np.float64)
        h = C.c_void_p()
        st = self.L.sfg_pcg_create(M.n, ptr(cp, i32p), ptr(ri, i32p), ptr(va, f64p), C.byref(h))
        self.h = h.value
        if st != abi.SFG_OK:
            fac = C.c_void_p()
            if self.h:
                self.L.sfg_pcg_plans(self.h, C.byref(fac), None)
            try:
                _raise(self.L, fac.value, st, "pcg setup")
            finally:
                self.close()

    def solve(self, b: np.ndarray, rtol: float = 1e-10, maxit: int = 1000, check: int = 1):
        """Returns (x, iterations, relative residual, device ms)."""
        bb = np.ascontiguousarray(b, np.float64)
        x = np.empty(self.n, np.float64)
        it = C.c_int32()
        rr = C.c_double()
        ms = C.c_float()
        st = self.L.sfg_pcg_solve(self.h, ptr(bb, f64p), ptr(x, f64p), rtol, maxit, check,
                                  C.byref(it), C.byref(rr), C.byref(ms))
        if st != abi.SFG_OK:
            raise RuntimeError(f"pcg solve failed with status {st}")
        return x, it.value, rr.value, ms.value

    def close(self):
        if getattr(self, "h", None):
            self.L.sfg_pcg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class ParseError(RuntimeError):
    """types.hpp:33-36 (Matrix Market and permutation files)."""


def _from_handle(L, h) -> CscMatrix:
    n = C.c_int32()
    nnz = C.c_int64()
    L.sfg_matrix_dims(h, C.byref(n), C.byref(nnz))
    cp = np.empty(n.value + 1, np.int32)
    ri = np.empty(max(nnz.value, 1), np.int32)
    va = np.empty(max(nnz.value, 1), np.float64)
    L.sfg_matrix_copy(h, ptr(cp, i32p), ptr(ri, i32p), ptr(va, f64p))
    return CscMatrix(n.value, cp, ri[:nnz.value], va[:nnz.value])


def _handle(L, M: CscMatrix):
    h = C.c_void_p()
    cp = np.ascontiguousarray(M.colptr, np.int32)
    ri = np.ascontiguousarray(M.rowidx, np.int32)
    va = np.ascontiguousarray(M.values, np.float64)
    if L.sfg_matrix_from_csc(M.n, ptr(cp, i32p), ptr(ri, i32p), ptr(va, f64p), C.byref(h)) != abi.SFG_OK:
        raise ValueError("bad CSC arrays")
    return h


def read_matrix_market(path: str) -> CscMatrix:
    """read_matrix_market (matrix_market.hpp:59-121): coordinate real,
    general or symmetric (expanded), duplicates summed."""
    L = abi.load()
    h = C.c_void_p()
    msg = C.create_string_buffer(512)
    st = L.sfg_matrix_read_mm(path.encode(), C.byref(h), msg, 512)
    if st == abi.SFG_ERR_PARSE:
        raise ParseError(msg.value.decode())
    if st == abi.SFG_ERR_INVALID_MATRIX:
        raise InvalidMatrixError(msg.value.decode())
    if st != abi.SFG_OK:
        raise ValueError(msg.value.decode() or "read_matrix_market failed")
    try:
        return _from_handle(L, h)
    finally:
        L.sfg_matrix_free(h)


def write_matrix_market(M: CscMatrix, path: str) -> None:
    """write_matrix_market (matrix_market.hpp:123-138), round-trip exact."""
    L = abi.load()
    h = _handle(L, M)
    try:
        if L.sfg_matrix_write_mm(h, path.encode()) != abi.SFG_OK:
            raise ParseError("cannot write " + path)
    finally:
        L.sfg_matrix_free(h)


def permute_symmetric(M: CscMatrix, perm) -> CscMatrix:
    """B = P A P^T, row/column i of A -> perm[i] of B (matrix.hpp:135-173)."""
    L = abi.load()
    p = np.ascontiguousarray(perm, np.int32)
    if p.size != M.n:
        raise InvalidMatrixError("permutation length mismatch")
    h = _handle(L, M)
    out = C.c_void_p()
    try:
        if L.sfg_matrix_permute(h, ptr(p, i32p), C.byref(out)) != abi.SFG_OK:
            raise InvalidMatrixError("not a permutation")
        try:
            return _from_handle(L, out)
        finally:
            L.sfg_matrix_free(out)
    finally:
        L.sfg_matrix_free(h)


def read_permutation(path: str, n: int) -> np.ndarray:
    """read_permutation (matrix_market.hpp:140-152)."""
    out = np.empty(max(n, 1), np.int32)
    if abi.load().sfg_read_permutation(path.encode(), n, ptr(out, i32p)) != abi.SFG_OK:
        raise ParseError(f"{path}: expected {n} permutation entries")
    return out[:n]


def _matrix(kind: int, a: int, b: int = 0, seed: int = 0, nsys_perturb: int = 0,
            seed0: int = 1000):
    L = abi.load()
    h = C.c_void_p()
    if L.sfg_matrix_gen(kind, a, b, seed, C.byref(h)) != abi.SFG_OK:
        raise ValueError("bad generator parameters")
    try:
        n = C.c_int32()
        nnz = C.c_int64()
        L.sfg_matrix_dims(h, C.byref(n), C.byref(nnz))
        cp = np.empty(n.value + 1, np.int32)
        ri = np.empty(max(nnz.value, 1), np.int32)
        va = np.empty(max(nnz.value, 1), np.float64)
        L.sfg_matrix_copy(h, ptr(cp, i32p), ptr(ri, i32p), ptr(va, f64p))
        M = CscMatrix(n.value, cp, ri[:nnz.value], va[:nnz.value])
        if nsys_perturb:
            vals = np.empty(nsys_perturb * nnz.value, np.float64)
            L.sfg_matrix_perturb_diag(h, nsys_perturb, seed0, ptr(vals, f64p))
            return M, vals
        return M
    finally:
        L.sfg_matrix_free(h)


def gen_grid_laplacian(k: int) -> CscMatrix:
    """gen_grid_laplacian (fixtures.hpp:49-91), ND-numbered."""
    return _matrix(0, k)


def gen_banded_spd(n: int, bw: int, seed: int) -> CscMatrix:
    """gen_banded_spd (fixtures.hpp:97-141)."""
    return _matrix(1, n, bw, seed)


FULL_SIZE = {1: 512, 2: 64, 3: 96, 4: 1_000_000, 5: 128}


def config_matrix(cfg: int, size: int | None = None, seed: int = 7,
                  halfwidth: int = 2000) -> CscMatrix:
    """BASELINE.json config matrices (full size by default):
    1: 5-pt 2-D Laplacian 512^2   2: 7-pt 3-D Laplacian 64^3
    3: 7-pt convection-diffusion 96^3   4: random band n=1e6, half-width 2000
    5: 27-pt 3-D stencil 128^3."""
    a = FULL_SIZE[cfg] if size is None else size
    return _matrix(9 + cfg, a, halfwidth if cfg == 4 else 0, seed)


def config5_systems(size: int | None = None, nsys: int = 8, seed0: int = 1000):
    """Config 5: the 27-point stencil and nsys per-system value arrays
    (system s adds delta ~ U[0, 0.1], mt19937_64(seed0 + s), to the diagonal).
    Returns (M, values[nsys * nnz]); b_s = gen_vector(n, 7 + s)."""
    a = FULL_SIZE[5] if size is None else size
    return _matrix(14, a, 0, 0, nsys_perturb=nsys, seed0=seed0)
