"""ctypes bindings of the C-ABI in include/sfgpu.h (libsfgpu.so, in-tree).

This is the product path: every call goes to the sm_100a CUDA library.  There
is no CPU fallback -- if the library is missing the import fails, and if no
CUDA device is present plan creation raises ``NoDeviceError``.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# SFG_LIB: an alternative build of the same library (A/B measurements)
LIB_PATH = os.environ.get("SFG_LIB") or os.path.join(HERE, "libsfgpu.so")

SFG_OK = 0
SFG_ERR_FACTORIZATION = 1
SFG_ERR_INVALID_MATRIX = 2
SFG_ERR_INVALID_ARGUMENT = 3
SFG_ERR_CUDA = 4
SFG_ERR_LOGIC = 5
SFG_ERR_NO_DEVICE = 6
SFG_ERR_PARSE = 7

# Every function include/sfgpu.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "sfg_device_check", "sfg_version", "sfg_set_device", "sfg_host_alloc",
    "sfg_host_free", "sfg_bench_executions", "sfg_selftest_division", "sfg_plan_create", "sfg_plan_destroy",
    "sfg_plan_set_stream", "sfg_plan_info", "sfg_set_vin", "sfg_set_values", "sfg_inspect",
    "sfg_get_dag", "sfg_get_interdep", "sfg_get_levels", "sfg_compute_reuse",
    "sfg_get_schedule", "sfg_get_partitioning", "sfg_execute_fused", "sfg_execute_batch", "sfg_execute_batch_ex", "sfg_execute_kernel", "sfg_spmv_rows", "sfg_set_vin_device", "sfg_pcg_create", "sfg_pcg_solve", "sfg_pcg_plans", "sfg_pcg_destroy", "sfg_execute_unfused",
    "sfg_synchronize", "sfg_collect_outputs", "sfg_device_output",
    "sfg_last_error", "sfg_launch_count", "sfg_last_exec_ms", "sfg_matrix_gen",
    "sfg_matrix_dims", "sfg_matrix_copy", "sfg_matrix_free", "sfg_matrix_read_mm",
    "sfg_matrix_write_mm", "sfg_matrix_from_csc", "sfg_matrix_permute", "sfg_read_permutation",
    "sfg_matrix_perturb_diag", "sfg_gen_vector", "sfg_execute_wavefront", "sfg_get_wavefront",
    "sfg_execute_sequential", "sfg_check_schedule", "sfg_dag_levels", "sfg_reset",
)

i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)
u8p = C.POINTER(C.c_uint8)
vp = C.c_void_p


def ptr(a, t):
    return None if a is None else a.ctypes.data_as(t)


_lib = None


def load(path: str | None = None):
    """Load libsfgpu.so (raises OSError if it was not built)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or LIB_PATH
    if not os.path.exists(p):
        raise OSError(f"{p} not built: run `make -C {HERE}` (or __graft_entry__.build())")
    L = C.CDLL(p)
    st = C.c_int
    L.sfg_version.restype = C.c_char_p
    L.sfg_device_check.argtypes = [i32p, i32p]
    L.sfg_device_check.restype = st
    L.sfg_set_device.argtypes = [C.c_int32]
    L.sfg_set_device.restype = st
    L.sfg_host_alloc.argtypes = [C.c_size_t, C.POINTER(vp)]
    L.sfg_host_alloc.restype = st
    L.sfg_host_free.argtypes = [vp]
    L.sfg_host_free.restype = st
    L.sfg_bench_executions.argtypes = [vp, C.c_int32, C.c_int32, C.POINTER(C.c_float),
                                       C.POINTER(C.c_float)]
    L.sfg_bench_executions.restype = st
    L.sfg_selftest_division.argtypes = [C.c_int64, C.c_uint64, i64p, i64p]
    L.sfg_selftest_division.restype = st
    L.sfg_plan_create.argtypes = [C.c_int32, C.c_int32, i32p, i32p, f64p, C.c_int32, f64p,
                                  C.c_uint64, C.POINTER(vp)]
    L.sfg_plan_create.restype = st
    L.sfg_plan_destroy.argtypes = [vp]
    L.sfg_plan_destroy.restype = st
    L.sfg_plan_set_stream.argtypes = [vp, vp]
    L.sfg_plan_set_stream.restype = st
    L.sfg_plan_info.argtypes = [vp, i32p, i32p, i32p, i64p, i64p]
    L.sfg_plan_info.restype = st
    L.sfg_set_vin.argtypes = [vp, f64p]
    L.sfg_set_vin.restype = st
    L.sfg_set_values.argtypes = [vp, f64p]
    L.sfg_set_values.restype = st
    L.sfg_inspect.argtypes = [vp]
    L.sfg_inspect.restype = st
    L.sfg_get_dag.argtypes = [vp, C.c_int32, i32p, i64p, i32p, i32p, i64p]
    L.sfg_get_dag.restype = st
    L.sfg_get_interdep.argtypes = [vp, i32p, i32p, i64p, i32p, i32p]
    L.sfg_get_interdep.restype = st
    L.sfg_get_levels.argtypes = [vp, C.c_int32, i32p, i32p, i32p, i32p]
    L.sfg_get_levels.restype = st
    L.sfg_compute_reuse.argtypes = [vp, f64p]
    L.sfg_compute_reuse.restype = st
    L.sfg_get_schedule.argtypes = [vp, i64p, u8p, i32p, i32p, i64p]
    L.sfg_get_schedule.restype = st
    L.sfg_get_partitioning.argtypes = [vp, i32p, i64p, i64p, i64p, i64p, u8p, i32p]
    L.sfg_get_partitioning.restype = st
    L.sfg_execute_batch.argtypes = [vp, C.c_int32, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]
    L.sfg_execute_batch.restype = st
    L.sfg_execute_batch_ex.argtypes = [vp, C.c_int32, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
                                       C.c_int32]
    L.sfg_execute_batch_ex.restype = st
    L.sfg_execute_kernel.argtypes = [vp, C.c_int32]
    L.sfg_execute_kernel.restype = st
    L.sfg_spmv_rows.argtypes = [vp, C.c_int32, C.c_int32, vp, vp]
    L.sfg_spmv_rows.restype = st
    L.sfg_set_vin_device.argtypes = [vp, vp]
    L.sfg_set_vin_device.restype = st
    L.sfg_pcg_create.argtypes = [C.c_int32, i32p, i32p, f64p, C.POINTER(vp)]
    L.sfg_pcg_create.restype = st
    L.sfg_pcg_solve.argtypes = [vp, f64p, f64p, C.c_double, C.c_int32, C.c_int32,
                                C.POINTER(C.c_int32), C.POINTER(C.c_double), C.POINTER(C.c_float)]
    L.sfg_pcg_solve.restype = st
    L.sfg_pcg_plans.argtypes = [vp, C.POINTER(vp), C.POINTER(vp)]
    L.sfg_pcg_plans.restype = st
    L.sfg_pcg_destroy.argtypes = [vp]
    L.sfg_pcg_destroy.restype = st
    L.sfg_execute_fused.argtypes = [vp]
    L.sfg_execute_fused.restype = st
    L.sfg_execute_unfused.argtypes = [vp]
    L.sfg_execute_unfused.restype = st
    L.sfg_execute_wavefront.argtypes = [vp]
    L.sfg_execute_wavefront.restype = st
    L.sfg_execute_sequential.argtypes = [vp]
    L.sfg_execute_sequential.restype = st
    L.sfg_get_wavefront.argtypes = [vp, i64p, u8p, i32p, i32p, i64p]
    L.sfg_get_wavefront.restype = st
    L.sfg_check_schedule.argtypes = [vp, C.c_int64, u8p, i32p, i64p]
    L.sfg_check_schedule.restype = st
    L.sfg_dag_levels.argtypes = [C.c_int32, i32p, i32p, i32p, i32p, i32p, i32p]
    L.sfg_dag_levels.restype = st
    L.sfg_reset.argtypes = [vp]
    L.sfg_reset.restype = st
    L.sfg_synchronize.argtypes = [vp]
    L.sfg_synchronize.restype = st
    L.sfg_collect_outputs.argtypes = [vp, f64p, C.c_int64]
    L.sfg_collect_outputs.restype = st
    L.sfg_device_output.argtypes = [vp, C.c_int32, C.POINTER(vp), i64p]
    L.sfg_device_output.restype = st
    L.sfg_last_error.argtypes = [vp, i32p, i32p, C.c_char_p, C.c_int32]
    L.sfg_last_error.restype = st
    L.sfg_launch_count.argtypes = [vp]
    L.sfg_launch_count.restype = C.c_int64
    L.sfg_last_exec_ms.argtypes = [vp, C.POINTER(C.c_float), C.POINTER(C.c_float)]
    L.sfg_last_exec_ms.restype = st
    L.sfg_matrix_gen.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_uint64, C.POINTER(vp)]
    L.sfg_matrix_gen.restype = st
    L.sfg_matrix_dims.argtypes = [vp, i32p, i64p]
    L.sfg_matrix_dims.restype = st
    L.sfg_matrix_copy.argtypes = [vp, i32p, i32p, f64p]
    L.sfg_matrix_copy.restype = st
    L.sfg_matrix_free.argtypes = [vp]
    L.sfg_matrix_free.restype = st
    L.sfg_matrix_perturb_diag.argtypes = [vp, C.c_int32, C.c_uint64, f64p]
    L.sfg_matrix_perturb_diag.restype = st
    L.sfg_gen_vector.argtypes = [C.c_int32, C.c_uint64, f64p]
    L.sfg_gen_vector.restype = st
    L.sfg_matrix_read_mm.argtypes = [C.c_char_p, C.POINTER(vp), C.c_char_p, C.c_int32]
    L.sfg_matrix_read_mm.restype = st
    L.sfg_matrix_write_mm.argtypes = [vp, C.c_char_p]
    L.sfg_matrix_write_mm.restype = st
    L.sfg_matrix_from_csc.argtypes = [C.c_int32, i32p, i32p, f64p, C.POINTER(vp)]
    L.sfg_matrix_from_csc.restype = st
    L.sfg_matrix_permute.argtypes = [vp, i32p, C.POINTER(vp)]
    L.sfg_matrix_permute.restype = st
    L.sfg_read_permutation.argtypes = [C.c_char_p, C.c_int32, i32p]
    L.sfg_read_permutation.restype = st
    if path is None:
        _lib = L
    return L


def device_available() -> bool:
    L = load()
    cnt = C.c_int32(0)
    sms = C.c_int32(0)
    return L.sfg_device_check(C.byref(cnt), C.byref(sms)) == SFG_OK and cnt.value > 0


class PinnedArray:
    """A page-locked host float64 buffer (sfg_host_alloc) viewed as numpy."""

    def __init__(self, count: int):
        L = load()
        self._L = L
        self._p = C.c_void_p()
        st = L.sfg_host_alloc(max(count, 1) * 8, C.byref(self._p))
        if st != SFG_OK:
            raise RuntimeError(f"sfg_host_alloc failed (status {st})")
        buf = (C.c_double * max(count, 1)).from_address(self._p.value)
        self.array = np.frombuffer(buf, dtype=np.float64, count=count)

    def free(self):
        if self._p:
            self._L.sfg_host_free(self._p)
            self._p = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def set_device(dev: int):
    st = load().sfg_set_device(dev)
    if st != SFG_OK:
        raise RuntimeError(f"sfg_set_device({dev}) failed (status {st})")
