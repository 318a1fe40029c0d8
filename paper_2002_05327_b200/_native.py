"""ctypes binding of the C-ABI (`include/diagsweep_b200.h`).

The shared library is built in-tree (`csrc/build.sh` -> `lib/`).  There is
no fallback: if the library or a CUDA device is missing, every GPU entry
point raises `SolverError` (the product path never routes through a CPU
implementation).  Status codes map onto the reference's exception types
(`diagsweep/errors.py:4-13`): < 0 -> ConfigurationError, > 0 -> SolverError.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

from .errors import ConfigurationError, ModelError, SolverError

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libdiagsweep_b200.so"

i32 = C.c_int32
i64 = C.c_int64
vp = C.c_void_p
P_i32 = C.POINTER(C.c_int32)
P_i64 = C.POINTER(C.c_int64)
P_f64 = C.POINTER(C.c_double)


class OpDesc(C.Structure):
    _fields_ = [
        ("dim", i32),
        ("shape", i32 * 3),
        ("c_lo", vp * 3),
        ("c_hi", vp * 3),
        ("kappa2_kind", i32),
        ("kappa2_axis", i32),
        ("kappa2", vp),
    ]


class PlanDesc(C.Structure):
    _fields_ = [
        ("dim", i32), ("nsub", i32), ("nsweeps", i32), ("nsteps", i32), ("ndir", i32),
        ("nrhs_max", i32),
        ("grid_counts", i32 * 3),
        ("part_counts", i32 * 3),
        ("win_lo", vp), ("win_shape", vp),
        ("own_lo", vp), ("own_shape", vp),
        ("sup_lo", vp), ("sup_shape", vp),
        ("beta00", vp), ("beta00_off", vp),
        ("nops", i32),
        ("ops", vp),
        ("op_of_sub", vp),
        ("fact_of_sub", vp),
        ("fact_index", vp),
        ("visit_sub", vp),
        ("step_off", vp),
        ("directions", vp),
        ("xfer_use", vp),
        ("band_lo", vp), ("band_shape", vp), ("ext_lo", vp), ("ext_shape", vp),
        ("xfac", vp),
        ("xfac_off", vp),
        ("nlaunch", i32),
        ("launch_off", vp),
        ("launch_visits", vp),
        ("nranks", i32),
        ("rank", i32),
        ("owner", vp),
        ("visit_slot", vp),
    ]


class ModalDesc(C.Structure):
    _fields_ = [
        ("block_axis", i32),
        ("naxes", i32),
        ("v", vp * 2),
        ("vinv", vp * 2),
        ("lambda_", vp * 2),
    ]


# (name, restype, argtypes) — must match include/diagsweep_b200.h
_SIGNATURES = [
    ("ds_abi_version", C.c_int, []),
    ("ds_last_error", C.c_char_p, []),
    ("ds_ctx_create", C.c_int, [C.c_int, vp, C.POINTER(vp)]),
    ("ds_ctx_set_stream", C.c_int, [vp, vp]),
    ("ds_ctx_synchronize", C.c_int, [vp]),
    ("ds_ctx_launches", i64, [vp]),
    ("ds_ctx_work", C.c_int, [vp, vp, i32]),
    ("ds_ctx_set_option", C.c_int, [vp, C.c_char_p, i32]),
    ("ds_ctx_get_option", C.c_int, [vp, C.c_char_p, P_i32]),
    ("ds_ctx_destroy", C.c_int, [vp]),
    ("ds_op_create", C.c_int, [vp, C.POINTER(OpDesc), C.POINTER(vp)]),
    ("ds_op_destroy", C.c_int, [vp]),
    ("ds_op_apply", C.c_int, [vp, vp, vp, vp, i32, P_i32, P_i32, i32]),
    ("ds_fact_create", C.c_int, [vp, C.POINTER(vp), i32, C.POINTER(vp)]),
    ("ds_fact_info", C.c_int, [vp, i32, P_i32, P_i32, P_i32, P_i64]),
    ("ds_fact_solve", C.c_int, [vp, vp, i32, vp, vp, i32]),
    ("ds_fact_destroy", C.c_int, [vp]),
    ("ds_fact_create_modal", C.c_int, [vp, C.POINTER(vp), i32, C.POINTER(ModalDesc), C.POINTER(vp)]),
    ("ds_fact_kind", C.c_int, [vp, i32]),
    ("ds_fact_create_pool", C.c_int, [vp, C.POINTER(vp), i32, i32, C.POINTER(vp)]),
    ("ds_fact_pool_load", C.c_int, [vp, vp, i32, i32]),
    ("ds_fact_pool_load_many", C.c_int, [vp, vp, i32, P_i32, P_i32]),
    ("ds_fact_pool_state", C.c_int, [vp, P_i32, P_i64, P_i32, P_i64]),
    ("ds_plan_create", C.c_int, [vp, C.POINTER(PlanDesc), C.POINTER(vp)]),
    ("ds_plan_workspace_bytes", i64, [vp]),
    ("ds_plan_destroy", C.c_int, [vp]),
    ("ds_ddm_apply", C.c_int, [vp, vp, vp, vp, i32, vp]),
    ("ds_ddm_apply_host", C.c_int, [vp, vp, vp, vp, i32]),
    ("ds_ddm_apply_outer", C.c_int, [vp, vp, vp, vp, i32]),
    ("ds_ddm_apply_host_groups", C.c_int, [vp, C.POINTER(vp), i32, vp, vp, i32]),
    ("ds_ddm_counters", C.c_int, [vp, vp, i32, P_i32, P_i32, P_i32, P_i32, P_i32, P_i32]),
    ("ds_ddm_enable_graph", C.c_int, [vp, vp, i32]),
    ("ds_plan_last_launches", i64, [vp]),
    ("ds_plan_shard_info", C.c_int, [vp, C.POINTER(vp), P_i64, C.POINTER(vp), P_i64]),
    ("ds_plan_set_peers", C.c_int, [vp, vp, i32, C.POINTER(vp), C.POINTER(vp)]),
    ("ds_plan_nlaunch", i32, [vp]),
    ("ds_plan_slot", C.c_int, [vp, vp, i32, i32, i32, P_i32, P_i32, vp, i64, i32]),
    ("ds_ddm_apply_range", C.c_int, [vp, vp, vp, vp, i32, i32, i32, i32]),
    ("ds_plan_set_profiling", C.c_int, [vp, i32]),
    ("ds_plan_kernel_times", C.c_int, [vp, P_f64, P_i64, i32]),
    ("ds_barrier_create", C.c_int, [vp, i32, i32, C.POINTER(vp)]),
    ("ds_barrier_info", C.c_int, [vp, C.POINTER(vp), P_i64]),
    ("ds_barrier_set_peers", C.c_int, [vp, i32, C.POINTER(vp)]),
    ("ds_barrier_wait", C.c_int, [vp, vp]),
    ("ds_barrier_generation", i64, [vp]),
    ("ds_barrier_destroy", C.c_int, [vp]),
    ("ds_vec_dot", C.c_int, [vp, i64, i32, vp, vp, vp]),
    ("ds_vec_norm", C.c_int, [vp, i64, i32, vp, vp]),
    ("ds_vec_axpy", C.c_int, [vp, i64, i32, vp, C.c_double, vp, vp]),
    ("ds_vec_axpy_dot", C.c_int, [vp, i64, i32, vp, vp, vp, vp, vp]),
    ("ds_vec_combine", C.c_int, [vp, i64, i32, i32, C.POINTER(vp), vp, vp]),
    ("ds_vec_scale", C.c_int, [vp, i64, i32, vp, vp, vp]),
    ("ds_vec_sub_norm", C.c_int, [vp, i64, i32, vp, vp, vp, vp]),
    ("ds_vec_rows", C.c_int, [vp, i64, i32, vp, vp, vp]),
    ("ds_layout_to_minor", C.c_int, [vp, i64, i32, vp, vp]),
    ("ds_layout_to_outer", C.c_int, [vp, i64, i32, vp, vp]),
    ("ds_raster_kappa2", C.c_int, [vp, i32, vp, vp, vp, vp, vp, C.c_double, vp]),
    ("ds_gaussian_fields", C.c_int, [vp, i32, vp, i32, vp, vp, vp, i32, vp]),
]

ABI_VERSION = 7

EXPORTED_SYMBOLS = [name for name, _, _ in _SIGNATURES]

_lib = None
_lock = threading.Lock()


def load_library(path: Path | None = None):
    """Load and bind the shared library (no CUDA calls are made)."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path or os.environ.get("DIAGSWEEP_B200_LIB", LIB_PATH))
        if not p.exists():
            raise SolverError(
                f"CUDA library {p} is missing: run __graft_entry__.build() "
                "(there is no CPU fallback)")
        lib = C.CDLL(str(p))
        for name, res, args in _SIGNATURES:
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.ds_abi_version() != ABI_VERSION:
            raise SolverError("diagsweep_b200 ABI version mismatch")
        if path is None:
            _lib = lib
        return lib


def check(status: int, what: str = "") -> None:
    if status == 0:
        return
    msg = _lib.ds_last_error().decode(errors="replace") if _lib else "unknown error"
    text = f"{what}: {msg}" if what else msg
    if status == -2:
        raise ModelError(text)
    if status < 0:
        raise ConfigurationError(text)
    raise SolverError(text)


def ptr(t) -> int:
    """Raw data pointer of a torch tensor or a NumPy array (0 for None)."""
    if t is None:
        return 0
    if hasattr(t, "data_ptr"):
        return t.data_ptr()
    return t.ctypes.data


def i32_array(values):
    import numpy as np

    arr = np.ascontiguousarray(values, dtype=np.int32)
    return arr, arr.ctypes.data_as(P_i32)
