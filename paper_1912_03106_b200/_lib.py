"""ctypes binding of libpintgpu.so (include/pintgpu.h).

The library is built in-tree (`paper_1912_03106_b200/lib/libpintgpu.so`,
see build.py).  There is no CPU fallback: loading fails loudly when the
library is missing, and pg_create fails without a CUDA device.
"""

import ctypes
import os

from .errors import InnerSolveError, NewtonConvergenceError, PintGpuError

# PINTGPU_LIB: dev override for A/B builds of the library
LIB_PATH = os.environ.get("PINTGPU_LIB") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "lib", "libpintgpu.so")

PG_OK, PG_EINVAL, PG_ECUDA, PG_ENEWTON, PG_ENOCONV = 0, 1, 2, 3, 4
PG_INNER_PCG, PG_INNER_CHOLESKY = 0, 1
PG_PROFILE_KINDS = 11           # pintgpu.h

c_int, c_int32, c_int64, c_double = (ctypes.c_int, ctypes.c_int32,
                                     ctypes.c_int64, ctypes.c_double)
c_void_p = ctypes.c_void_p
P_int32 = ctypes.POINTER(ctypes.c_int32)
P_double = ctypes.POINTER(ctypes.c_double)


class LevelDesc(ctypes.Structure):
    _fields_ = [
        ("n", c_int32), ("nnz", c_int32),
        ("row_ptr", P_int32), ("col_idx", P_int32),
        ("m_val", P_double), ("k_val", P_double),
        ("n_src", c_int32), ("shapes", P_double), ("weights", P_double),
        ("side", c_int32),
        ("n_elem", c_int32), ("elem_dof", P_int32), ("elem_geo", P_double),
        ("node_elem_ptr", P_int32), ("node_elem", P_int32),
        ("k_pre_val", P_double),
    ]


class SolverOpts(ctypes.Structure):
    _fields_ = [
        ("inner", c_int32), ("rtol", c_double), ("max_iters", c_int32), ("check_every", c_int32),
        ("newton_tol", c_double), ("newton_max_iters", c_int32),
        ("damping", c_double), ("max_halvings", c_int32),
        ("nu0", c_double), ("k1", c_double), ("k2", c_double), ("k3", c_double),
        ("dt_merge_rtol", c_double),
        ("strips", c_int32),
    ]


class PhiStats(ctypes.Structure):
    _fields_ = [
        ("columns", c_int64), ("column_iters", c_int64), ("batch_iters", c_int64),
        ("newton_iters", c_int64), ("failed", c_int64), ("launches", c_int64),
    ]


class KernelProfile(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 16), ("total_ms", c_double), ("launches", c_int64),
                ("alg_bytes", c_double), ("alg_flops", c_double), ("column_iters", c_int64)]


EXPORTS = {
    "pg_create": (c_int, [ctypes.POINTER(c_void_p), c_int]),
    "pg_destroy": (None, [c_void_p]),
    "pg_last_error": (ctypes.c_char_p, [c_void_p]),
    "pg_add_level": (c_int, [c_void_p, ctypes.POINTER(LevelDesc)]),
    "pg_set_options": (c_int, [c_void_p, ctypes.POINTER(SolverOpts)]),
    "pg_phi_batch": (c_int, [c_void_p, c_int, c_int, c_void_p, c_void_p, c_void_p,
                             c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "pg_phi_batch_h": (c_int, [c_void_p, c_int, c_int, c_void_p, c_void_p, c_void_p, c_void_p,
                               c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "pg_prefactor": (c_int, [c_void_p, c_int, c_int, c_void_p, c_void_p]),
    "pg_last_stats": (c_int, [c_void_p, ctypes.POINTER(PhiStats)]),
    "pg_total_stats": (c_int, [c_void_p, ctypes.POINTER(PhiStats), c_int]),
    "pg_newton_failure": (c_int, [c_void_p, ctypes.POINTER(c_int), ctypes.POINTER(c_int)]),
    "pg_restrict": (c_int, [c_void_p, c_int, c_int, c_void_p, c_void_p, c_int, c_void_p]),
    "pg_prolong_add": (c_int, [c_void_p, c_int, c_int, c_void_p, c_void_p, c_void_p,
                               c_double, c_int, c_void_p]),
    "pg_c_residual": (c_int, [c_void_p, c_int, c_int, c_void_p, c_void_p, c_void_p,
                              c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                              c_void_p, c_void_p, c_void_p]),
    "pg_fas_rhs": (c_int, [c_void_p, c_int, c_int, c_int, c_void_p, c_void_p,
                           c_void_p, c_void_p, c_int, c_void_p]),
    "pg_rows_axpby": (c_int, [c_void_p, c_int, c_int, c_void_p, c_void_p, c_int, c_int,
                              c_void_p, c_void_p, c_int, c_int, c_int,
                              c_void_p, c_void_p, c_int, c_int, c_void_p]),
    "pg_launch_count": (c_int64, [c_void_p]),
    "pg_profile": (c_int, [c_void_p, c_int]),
    "pg_profile_read": (c_int, [c_void_p, ctypes.POINTER(KernelProfile), c_int, c_int]),
}

_LIB = None


def load():
    """Load the library once; raises PintGpuError when it is missing."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise PintGpuError(
            f"{LIB_PATH} is missing: build it with "
            "`python -m paper_1912_03106_b200.build` (no CPU fallback exists)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in EXPORTS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


def check(ctx, rc, what):
    if rc == PG_OK:
        return
    lib = load()
    msg = lib.pg_last_error(ctx)
    msg = msg.decode() if msg else ""
    if rc == PG_EINVAL:
        raise ValueError(f"{what}: {msg}")
    if rc == PG_ENEWTON:
        raise NewtonConvergenceError(f"{what}: {msg}")
    if rc == PG_ENOCONV:
        raise InnerSolveError(f"{what}: {msg}")
    raise PintGpuError(f"{what} failed with code {rc}: {msg}")


def ptr(t):
    """Device/host pointer of a torch tensor (or None)."""
    return None if t is None else ctypes.c_void_p(t.data_ptr())
