"""ctypes binding of libgapsafe_b200.so (the C ABI in include/gapsafe_b200.h).

The library is built in-tree by ``__graft_entry__.build()``.  There is no
CPU fallback: a missing library or a missing CUDA device raises.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

LIB_NAME = "libgapsafe_b200.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

GS_OK = 0
GS_ERR_CUDA = -1
GS_ERR_VALUE = -2
GS_ERR_INDEX = -3
GS_ERR_RUNTIME = -4
GS_ERR_INFEASIBLE = -5
GS_ERR_NUMERICAL = -6
GS_ERR_NODEVICE = -7

GS_DTYPE_F64 = 0
GS_DTYPE_F32 = 1
GS_RULE_NONE = 0
GS_RULE_GAP_SPHERE = 1
GS_RULE_STATIC = 2
GS_RULE_DYNAMIC = 3
GS_RULE_ST3 = 4
GS_RULE_GAP_DOME = 5

c_i64 = ctypes.c_int64
c_i32 = ctypes.c_int32
c_dbl = ctypes.c_double
c_vp = ctypes.c_void_p
P_f64 = ctypes.POINTER(ctypes.c_double)
P_i64 = ctypes.POINTER(ctypes.c_int64)
P_i32 = ctypes.POINTER(ctypes.c_int32)

CKPT_CB = ctypes.CFUNCTYPE(None, P_i64, c_i64, c_vp)


class SolveConfig(ctypes.Structure):
    _fields_ = [("epsilon", c_dbl), ("max_passes", c_i64), ("screen_every", c_i64),
                ("rule", c_i32), ("certify", c_i32), ("on_checkpoint", CKPT_CB),
                ("user", c_vp)]


class SolveResult(ctypes.Structure):
    _fields_ = [("beta", P_f64), ("residual", P_f64), ("theta", P_f64), ("active", P_i64),
                ("trace_passes", P_i64), ("trace_active", P_i64), ("trace_gap", P_f64),
                ("trace_radius", P_f64), ("trace_cap", c_i64),
                ("n_active", c_i64), ("n_trace", c_i64), ("passes_done", c_i64),
                ("converged", c_i32), ("interpolating", c_i32), ("lambda_max_shortcut", c_i32),
                ("pad_", c_i32),
                ("margin", c_dbl), ("primal", c_dbl), ("dual", c_dbl), ("gap", c_dbl),
                ("cd_visits", ctypes.c_uint64), ("cd_uncertified", ctypes.c_uint64),
                ("cd_nonzero", ctypes.c_uint64), ("checkpoints", c_i64), ("device_ms", c_dbl),
                ("screen_ms", c_dbl), ("ckpt_ms", c_dbl), ("refresh_ms", c_dbl), ("cd_ms", c_dbl),
                ("n_screen", c_i64), ("n_refresh", c_i64), ("launches", c_i64),
                ("cd_candidates", c_i64), ("cd_skipped", c_i64), ("cd_requeues", c_i64)]


# every symbol declared in include/gapsafe_b200.h with its ctypes signature
SIGNATURES = {
    "gs_init": (c_i32, [ctypes.c_int]),
    "gs_device_count": (c_i32, [ctypes.POINTER(ctypes.c_int)]),
    "gs_last_error": (ctypes.c_char_p, []),
    "gs_version": (ctypes.c_char_p, []),
    "gs_launch_count": (c_i64, []),
    "gs_matrix_dense": (c_i32, [c_vp, ctypes.c_int, c_i64, c_i64, c_i64, P_f64, ctypes.POINTER(c_vp)]),
    "gs_matrix_csc": (c_i32, [P_f64, P_i32, P_i64, c_i64, c_i64, P_f64, ctypes.POINTER(c_vp)]),
    "gs_matrix_norms_sq": (c_i32, [c_vp, P_f64]),
    "gs_matrix_device_bytes": (c_i64, [c_vp]),
    "gs_matrix_free": (None, [c_vp]),
    "gs_tdot": (c_i32, [c_vp, P_f64, P_i64, c_i64, c_dbl, P_f64, ctypes.c_int]),
    "gs_matvec": (c_i32, [c_vp, P_f64, P_f64]),
    "gs_max_abs_correlation": (c_i32, [c_vp, P_f64, P_i64, c_i64, P_f64, P_i64]),
    "gs_axpy_col": (c_i32, [c_vp, c_i64, c_dbl, P_f64]),
    "gs_cd_pass": (c_i32, [c_vp, P_f64, P_f64, P_i64, c_i64, c_dbl, P_f64, c_dbl, ctypes.c_int]),
    "gs_screen_sphere": (c_i32, [c_vp, P_f64, c_dbl, P_i64, c_i64, c_dbl, P_f64, P_i64, P_i64]),
    "gs_vec_stats": (c_i32, [P_f64, P_f64, c_i64, P_f64, P_f64]),
    "gs_solver_create": (c_i32, [c_vp, P_f64, ctypes.POINTER(c_vp)]),
    "gs_solver_lambda_max": (c_i32, [c_vp, P_f64, P_i64, P_f64]),
    "gs_solver_set_lambda_max": (c_i32, [c_vp, c_dbl]),
    "gs_solver_set_beta": (c_i32, [c_vp, P_f64]),
    "gs_solver_seq_screen": (c_i32, [c_vp, c_dbl, P_i64]),
    "gs_solver_solve": (c_i32, [c_vp, c_dbl, ctypes.POINTER(SolveConfig), P_i64, c_i64,
                                ctypes.c_int, ctypes.POINTER(SolveResult)]),
    "gs_solver_free": (None, [c_vp]),
    "gs_solver_timer": (c_i32, [c_vp, ctypes.c_int, P_f64]),
    "gs_matrix_dense_alloc": (c_i32, [c_i32, c_i64, c_i64, ctypes.POINTER(c_vp)]),
    "gs_matrix_dense_set_columns": (c_i32, [c_vp, c_i64, c_i64, c_vp, c_i64]),
    "gs_matrix_dense_finalize": (c_i32, [c_vp]),
    "gs_matrix_dense_dev": (c_i32, [c_vp, c_i32, c_i64, c_i64, c_i64, ctypes.POINTER(c_vp)]),
    "gs_matrix_gather_columns_dev": (c_i32, [c_vp, P_i64, c_i64, c_vp, c_i64]),
    "gs_screen_timed": (c_i32, [c_vp, P_f64, c_dbl, ctypes.c_int, P_f64, P_i64, P_i32]),
    "gs_host_alloc": (c_i32, [c_i64, ctypes.POINTER(c_vp)]),
    "gs_host_free": (None, [c_vp]),
    "gs_batch_create": (c_i32, [c_vp, P_f64, P_i32, c_i64, c_i64, ctypes.POINTER(c_vp)]),
    "gs_batch_lambda_max": (c_i32, [c_vp, P_f64]),
    "gs_batch_run_paths": (c_i32, [c_vp, P_f64, c_i64, ctypes.POINTER(SolveConfig), P_f64, P_f64, P_i64, P_f64,
                                   P_i32, P_i64, P_f64]),
    "gs_batch_free": (None, [c_vp]),
}

_lib = None


class GapSafeDeviceError(RuntimeError):
    """CUDA device missing or CUDA runtime failure (never a silent fallback)."""


def load():
    """Load (once) and return the native library; raises if it is absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise GapSafeDeviceError(
                f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; "
                f"g.build()'` (nvcc, sm_100a).  There is no CPU fallback.")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(rc: int) -> None:
    """Map a GS_* return code onto the reference's exception types."""
    if rc == GS_OK:
        return
    msg = load().gs_last_error().decode(errors="replace")
    if rc == GS_ERR_VALUE:
        raise ValueError(msg)
    if rc == GS_ERR_INDEX:
        raise IndexError(msg)
    if rc == GS_ERR_INFEASIBLE:
        from .problem import InfeasibleDualError
        raise InfeasibleDualError(msg)
    if rc == GS_ERR_NUMERICAL:
        from .regions import NumericalInconsistencyError
        raise NumericalInconsistencyError(msg)
    if rc == GS_ERR_RUNTIME:
        raise RuntimeError(msg)
    raise GapSafeDeviceError(f"gapsafe_b200 error {rc}: {msg}")


def f64p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(P_f64)


def i64p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(P_i64)


def i32p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(P_i32)


def launch_count() -> int:
    """Kernels launched by libgapsafe_b200 in this process so far."""
    return int(load().gs_launch_count())


def init_device(index: int) -> None:
    """Bind the library to CUDA device ``index`` (one process per GPU)."""
    check(load().gs_init(int(index)))


def vec_stats(a: np.ndarray, b: np.ndarray | None = None) -> tuple[float, float]:
    """(a.b, sum|a|) reduced on the device."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    if b is not None:
        b = np.ascontiguousarray(b, dtype=np.float64)
    dot = c_dbl()
    asum = c_dbl()
    check(load().gs_vec_stats(f64p(a), f64p(b), a.size, ctypes.byref(dot), ctypes.byref(asum)))
    return dot.value, asum.value


class PinnedArray:
    """A numpy view of page-locked host memory (freed with the object)."""

    def __init__(self, shape, dtype=np.float64, order="C"):
        self.nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
        ptr = c_vp()
        check(load().gs_host_alloc(self.nbytes, ctypes.byref(ptr)))
        self._ptr = ptr
        buf = (ctypes.c_char * self.nbytes).from_address(ptr.value)
        self.array = np.ndarray(shape, dtype=dtype, buffer=buf, order=order)

    def __del__(self):
        if getattr(self, "_ptr", None) is not None and self._ptr.value:
            load().gs_host_free(self._ptr)
            self._ptr = None
