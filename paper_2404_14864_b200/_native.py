"""ctypes binding of the C ABI in ``include/kfbi_b200.h``.

The shared library ``libkfbi_b200.so`` is built in-tree by
``__graft_entry__.build()`` (sm_100a).  There is no fallback: if the library
is missing, importing anything that needs it raises immediately.
"""

from __future__ import annotations

import ctypes as C
import os
import re

from .errors import ConfigError, ConvergenceError, DispatchError, GridError, InstabilityError

LIB_NAME = "libkfbi_b200.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

OK, E_CONFIG, E_GRID, E_NOCONV, E_INSTABILITY, E_CUDA = range(6)
F64, C128 = 0, 1

# index order of the per-kernel timing arrays (engine.py:23-35 names)
KERNEL_ORDER = (
    "classify-nodes",
    "edge-intersections",
    "jumps-and-corrections",
    "transform-rows",
    "transform-cols",
    "diagonal-scale",
    "extract-traces",
    "density-update",
    "rhs-update",
)

vp = C.c_void_p
i32 = C.c_int32
i64 = C.c_int64
f64 = C.c_double


class GridDesc(C.Structure):
    _fields_ = [("m", i32), ("h", f64), ("device", i32)]


class Slab(C.Structure):
    _fields_ = [("nranks", i32), ("rank", i32)]


class TriDist(C.Structure):
    _fields_ = [("nranks", i32), ("rank", i32), ("virt", i32), ("pad", i32),
                ("epoch", C.c_uint64), ("max_spins", C.c_int64), ("timed_out", vp),
                ("panels", vp * 8), ("agg", vp * 8), ("flags", vp * 8)]


class Geometry(C.Structure):
    _fields_ = [
        ("n_ctl", i32), ("n_edges", i32), ("n_rec", i32), ("n_groups", i32),
        ("w_edges", vp), ("edge_axis", vp), ("rec_edge", vp), ("rec_d", vp),
        ("rec_sigma", vp), ("group_start", vp), ("group_node", vp), ("row_group", vp),
        ("deriv_col", vp), ("speed", vp), ("tangent", vp), ("normal", vp),
        ("dtan_ds", vp), ("inv3", vp), ("stencil", vp), ("ainv_rows", vp), ("jcoef", vp),
        ("edge_theta", vp), ("ctl_theta", vp),
    ]


class Bvp(C.Structure):
    _fields_ = [
        ("dtype", i32), ("kappa_re", f64), ("kappa_im", f64),
        ("F", vp), ("F_sign", f64), ("f_gamma", vp), ("f_gamma_sign", f64),
        ("g", vp), ("density", vp), ("gamma", f64), ("tol", f64),
        ("max_iter", i32), ("sweeps_hint", i32),
        ("u", vp), ("trace_u", vp), ("trace_un", vp), ("use_operator", i32),
        ("log_slot", i32), ("bc_kind", i32), ("box_bc", i32), ("field_chunks", i32),
    ]


class StepLog(C.Structure):
    _fields_ = [("iterations", i32), ("status", i32), ("residual", f64), ("norm", f64),
                ("newton", f64)]


class BvpResult(C.Structure):
    _fields_ = [("iterations", i32), ("converged", i32), ("residual", f64),
                ("history", C.POINTER(C.c_double))]


_SIGNATURES = {
    "kfbi_last_error": ([], C.c_char_p),
    "kfbi_version": ([], C.c_char_p),
    "kfbi_plan_create": ([C.POINTER(GridDesc), C.POINTER(vp)], i32),
    "kfbi_plan_destroy": ([vp], i32),
    "kfbi_box_solve": ([vp, i32, f64, f64, vp, vp, vp], i32),
    "kfbi_plan_set_geometry": ([vp, C.POINTER(Geometry)], i32),
    "kfbi_jumps": ([vp, i32, f64, f64, vp, vp, vp, f64, vp, vp], i32),
    "kfbi_corrections": ([vp, i32, vp, vp, vp], i32),
    "kfbi_interface_solve": ([vp, i32, f64, f64, vp, vp, vp, vp], i32),
    "kfbi_extract": ([vp, i32, vp, vp, vp, vp], i32),
    "kfbi_richardson": ([vp, C.POINTER(Bvp), C.POINTER(BvpResult), vp], i32),
    "kfbi_gmres": ([vp, C.POINTER(Bvp), i32, C.POINTER(BvpResult), vp], i32),
    "kfbi_slab_tri_bytes": ([vp, i32, i32, C.POINTER(C.c_int64), C.POINTER(C.c_int64)], i32),
    "kfbi_slab_cols_tri": ([vp, i32, i32, i32, C.c_double, C.c_double, vp, C.POINTER(TriDist), vp], i32),
    "kfbi_classify_nodes": ([i32, i32, vp, vp, vp, i32, C.c_double, vp, C.POINTER(i32), vp, i32], i32),
    "kfbi_build_trace_operator": ([vp, i32, f64, f64, vp], i32),
    "kfbi_build_trace_operator_bc": ([vp, i32, i32, i32, f64, f64, vp], i32),
    "kfbi_box_solve_bc": ([vp, i32, i32, f64, f64, vp, vp, vp], i32),
    "kfbi_interface_solve_bc": ([vp, i32, i32, f64, f64, vp, vp, vp, vp], i32),
    "kfbi_plan_set_onesided": ([vp, i32, vp, vp, vp], i32),
    "kfbi_extract_onesided": ([vp, i32, vp, vp, vp, vp], i32),
    "kfbi_log_reserve": ([vp, i32], i32),
    "kfbi_log_norm": ([vp, i32, i32, vp], i32),
    "kfbi_log_fetch": ([vp, i32, i32, vp, vp], i32),
    "kfbi_log_clear": ([vp, i32, i32, vp], i32),
    "kfbi_plan_set_exterior_zero": ([vp, i32], i32),
    "kfbi_plan_set_interior_list": ([vp, vp, i64], i32),
    "kfbi_plan_set_field_chunks": ([vp, vp, i64], i32),
    "kfbi_plan_work_fractions": ([vp, C.POINTER(f64)], i32),
    "kfbi_log_copy": ([vp, i32, i32, i32, vp], i32),
    "kfbi_heat_rhs": ([vp, i64, vp, vp, vp, vp, f64, C.POINTER(f64), vp], i32),
    "kfbi_wave_rhs": ([vp, i64, vp, vp, vp, vp, vp, vp, f64, f64, C.POINTER(f64), vp], i32),
    "kfbi_schr_ustar": ([vp, i64, i32, vp, vp, f64, vp, vp], i32),
    "kfbi_nonlinear_phase": ([vp, i64, vp, vp, f64, f64, vp, vp, f64, f64, vp,
                              C.POINTER(f64), vp], i32),
    "kfbi_strang_phase": ([vp, i64, i32, vp, vp, f64, vp, f64, f64, vp, vp, f64, f64, vp,
                           C.POINTER(f64), vp], i32),
    "kfbi_mask_norm": ([vp, i32, i64, vp, vp, C.POINTER(f64), vp], i32),
    "kfbi_gather": ([vp, i32, i64, vp, vp, vp, vp], i32),
    "kfbi_edge_values": ([vp, i32, vp, vp, vp], i32),
    "kfbi_slab_stencil_values": ([vp, i32, i32, vp, vp, vp, vp], i32),
    "kfbi_rich_begin": ([vp, i32, f64, vp], i32),
    "kfbi_slab_update": ([vp, i32, i32, vp, vp, vp, vp, vp, vp, f64, vp], i32),
    "kfbi_rich_state": ([vp, C.POINTER(i32), C.POINTER(i32), C.POINTER(f64), vp, vp], i32),
    "kfbi_plan_copy_w": ([vp, i32, i32, vp], i32),
    "kfbi_slab_panel_bytes": ([vp, i32, i32, C.POINTER(i64)], i32),
    "kfbi_slab_rows_fwd": ([vp, i32, vp, vp, f64, vp, vp, vp], i32),
    "kfbi_slab_cols": ([vp, i32, vp, f64, f64, vp, vp], i32),
    "kfbi_slab_rows_inv": ([vp, i32, vp, vp, vp, vp], i32),
    "kfbi_plan_set_interp": ([vp, i32], i32),
    "kfbi_plan_set_colsolver": ([vp, i32], i32),
    "kfbi_plan_set_trace_sweep": ([vp, i32], i32),
    "kfbi_plan_set_facr": ([vp, i32], i32),
    "kfbi_plan_facr_for": ([vp, C.c_double, C.c_double, C.POINTER(i32)], i32),
    "kfbi_operator_max_controls": ([vp, C.POINTER(i32)], i32),
    "kfbi_plan_colsolver_for": ([vp, C.c_double, C.c_double, C.POINTER(i32), C.POINTER(C.c_double)], i32),
    "kfbi_plan_get_colsolver": ([vp, C.POINTER(i32)], i32),
    "kfbi_plan_get_interp": ([vp, C.POINTER(i32)], i32),
    "kfbi_slab_rows_fwd_p2p": ([vp, i32, vp, vp, f64, vp, vp, vp], i32),
    "kfbi_slab_cols_p2p": ([vp, i32, vp, f64, f64, vp, vp, vp], i32),
    "kfbi_ipc_alloc": ([i64, C.POINTER(vp), vp], i32),
    "kfbi_ipc_free": ([vp], i32),
    "kfbi_ipc_open": ([vp, C.POINTER(vp)], i32),
    "kfbi_ipc_close": ([vp], i32),
    "kfbi_p2p_barrier": ([vp, i32, i32, i64, i64, vp, vp], i32),
    "kfbi_kernel_times": ([vp, C.POINTER(f64), C.POINTER(i64)], i32),
    "kfbi_reset_kernel_times": ([vp], i32),
    "kfbi_set_timing": ([vp, i32], i32),
    "kfbi_launch_count": ([vp], i64),
}

EXPORTED_SYMBOLS = tuple(_SIGNATURES)

_lib = None


def lib():
    """Load the library once; raise (never fall back) if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_NAME} is not built (expected at {LIB_PATH}); run "
                "`python -c 'import __graft_entry__ as g; g.build()'` from the repo root")
        handle = C.CDLL(LIB_PATH)
        for name, (args, res) in _SIGNATURES.items():
            fn = getattr(handle, name)
            fn.argtypes = args
            fn.restype = res
        _lib = handle
    return _lib


def last_error():
    return lib().kfbi_last_error().decode("utf-8", "replace")


_KERNEL_RE = re.compile(r"kernel '([^']+)'")


def check(status, iterations=None, last_residual=None):
    """Map a kfbi_status onto the reference exception classes."""
    if status == OK:
        return
    msg = last_error()
    if status == E_CONFIG:
        raise ConfigError(msg)
    if status == E_GRID:
        raise GridError(msg)
    if status == E_NOCONV:
        raise ConvergenceError(msg, iterations=iterations, last_residual=last_residual)
    if status == E_INSTABILITY:
        raise InstabilityError(0, 0.0, float("nan"), float("nan"))
    m = _KERNEL_RE.search(msg)
    raise DispatchError(m.group(1) if m else "unknown", msg)


def ptr(t):
    """Raw device (or host) address of a torch tensor / numpy array, or None."""
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        return t.data_ptr()
    return t.ctypes.data
