"""ctypes binding of ``libparaexp.so`` (the C ABI in ``include/paraexp.h``).

This is the binding a maintainer of the (pure-Python) reference would add for
``backend="cuda"``; see INTEGRATION.md. The library is built in-tree by
``__graft_entry__.build()`` (nvcc, sm_100a). There is no CPU fallback: if the
library or a CUDA device is missing, :class:`NativeUnavailable` is raised.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_int, c_size_t, c_uint64, c_void_p

from .errors import NativeUnavailable, raise_for_status

LIB_NAME = "libparaexp.so"
# PX_LIB: developer override (kernel-variant experiments); the default is the in-tree build
LIB_PATH = os.environ.get("PX_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

PX_KIND_ADVDIFF, PX_KIND_BURGERS = 0, 1
PX_EXP_CHEBYSHEV, PX_EXP_KRYLOV = 0, 1
PX_MEM_HOST, PX_MEM_DEVICE = 0, 1
PX_PLAN_SLICE, PX_PLAN_LONG_DIRECT, PX_PLAN_LONG_ADJOINT, PX_PLAN_FROZEN, PX_PLAN_NL_SLICE, PX_PLAN_NL_STEP = range(6)
PX_PLAN_BLOCK_LONG = 6
PX_MAX_LOCAL_BLOCKS = 16
(PX_FIELD_J, PX_FIELD_GRAD, PX_FIELD_UT, PX_FIELD_QDAG0, PX_FIELD_G, PX_FIELD_UBND,
 PX_FIELD_FROZEN_BOUNDS, PX_FIELD_VEND, PX_FIELD_WEND, PX_FIELD_TRAJ) = range(10)
PX_FLAG_BOUNDARY_STATES, PX_FLAG_Z_ACCUM, PX_FLAG_FIELD_CONTROL = 1, 2, 4
ABI_VERSION = 5
# kernel-variant keys (px_set_variant)
VARIANTS = {"march2": 0, "march_cols": 1, "march_band": 2, "cheb_terms": 3, "cheb_strip": 4, "cheb_band": 5,
            "scan1d_cluster": 6, "burgers_cluster": 7, "cheb_terms_phi": 8, "krylov_ortho": 9}
PX_ADJOINT_ABSORBED, PX_ADJOINT_FROZEN_SPAN = 0, 1


class ProblemDesc(ctypes.Structure):
    _fields_ = [
        ("kind", c_int),
        ("nx", c_int),
        ("ny", c_int),
        ("stencil", c_double * 5),
        ("D", c_double),
        ("hx", c_double),
        ("T", c_double),
        ("P", c_int),
        ("nsteps", c_int),
        ("p_begin", c_int),
        ("p_end", c_int),
        ("batch", c_int),
        ("K", c_int),
        ("basis_rows_x", c_int),
        ("basis_rows_y", c_int),
        ("expaction", c_int),
        ("krylov_m", c_int),
        ("flags", c_int),
    ]


class ChebPlanC(ctypes.Structure):
    _fields_ = [
        ("span", c_double),
        ("substeps", c_int),
        ("degree", c_int),
        ("center", c_double),
        ("scale", c_double),
        ("sigma", c_int),
        ("coef_exp", POINTER(c_double)),
        ("coef_phi", POINTER(c_double)),
    ]


class HybridDesc(ctypes.Structure):
    _fields_ = [
        ("nx", c_int),
        ("D", c_double),
        ("hx", c_double),
        ("T", c_double),
        ("batch", c_int),
        ("nslices", c_int),
        ("offsets", POINTER(c_int)),
        ("law", c_double * 4),
        ("target_batched", c_int),
        ("ny", c_int),
        ("hy", c_double),
    ]


(PX_HFIELD_J, PX_HFIELD_GRAD, PX_HFIELD_UT, PX_HFIELD_QDAG0, PX_HFIELD_TRAJ, PX_HFIELD_AEND, PX_HFIELD_ZL,
 PX_HFIELD_UBAR) = range(8)


class Stats(ctypes.Structure):
    _fields_ = [
        ("rk4_lane_steps", c_uint64),
        ("exp_terms", c_uint64),
        ("arnoldi_steps", c_uint64),
        ("kernel_launches", c_uint64),
        ("algorithmic_bytes", c_double),
        ("rk4_bytes", c_double),
        ("exp_bytes", c_double),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


PX_PHASES = ("rk4_direct", "rk4_adjoint", "exp_direct", "exp_adjoint", "other")
PX_KCLASS_MARCH2, PX_KCLASS_CHEB = 0, 1


class Timing(ctypes.Structure):
    _fields_ = [("ms", c_double * 5), ("launches", c_uint64 * 5), ("bytes", c_double * 5)]

    def as_dict(self) -> dict:
        return {ph: {"ms": self.ms[i], "launches": int(self.launches[i]), "bytes": self.bytes[i]}
                for i, ph in enumerate(PX_PHASES)}


# exported symbols and their prototypes: (restype, argtypes)
SIGNATURES = {
    "px_abi_version": (c_int, []),
    "px_build_info": (ctypes.c_char_p, []),
    "px_create": (c_int, [POINTER(ProblemDesc), POINTER(c_void_p)]),
    "px_destroy": (None, [c_void_p]),
    "px_last_error": (ctypes.c_char_p, [c_void_p]),
    "px_set_basis": (c_int, [c_void_p, POINTER(c_double), POINTER(c_double), POINTER(c_int), POINTER(c_int)]),
    "px_set_cheb_plan": (c_int, [c_void_p, c_int, POINTER(ChebPlanC)]),
    "px_set_krylov_plan": (c_int, [c_void_p, c_int, c_double, c_int]),
    "px_set_cheb_plan_law": (c_int, [c_void_p, c_int, POINTER(c_double), POINTER(c_double)]),
    "px_set_time_law": (c_int, [c_void_p, POINTER(c_double)]),
    "px_set_tracking_target": (c_int, [c_void_p, c_void_p, c_int, c_int, c_void_p]),
    "px_set_local_blocks": (c_int, [c_void_p, c_int]),
    "px_set_local_block_sizes": (c_int, [c_void_p, c_int, POINTER(c_int)]),
    "px_set_variant": (c_int, [c_void_p, c_int, c_int]),
    "px_get_variant": (c_int, [c_void_p, c_int, POINTER(c_int)]),
    "px_set_adjoint_mode": (c_int, [c_void_p, c_int]),
    "px_set_inputs": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_void_p]),
    "px_direct": (c_int, [c_void_p, c_void_p]),
    "px_finish_direct": (c_int, [c_void_p, c_void_p]),
    "px_set_adjoint_terminal": (c_int, [c_void_p, c_void_p, c_int, c_void_p]),
    "px_nl_init": (c_int, [c_void_p, c_void_p]),
    "px_nl_prepare": (c_int, [c_void_p, c_void_p]),
    "px_nl_sweep": (c_int, [c_void_p, POINTER(c_double), c_void_p]),
    "px_nl_finish": (c_int, [c_void_p, c_void_p]),
    "px_adjoint": (c_int, [c_void_p, c_void_p]),
    "px_finish_adjoint": (c_int, [c_void_p, c_void_p]),
    "px_gradient": (c_int, [c_void_p, c_void_p]),
    "px_set_graphs": (c_int, [c_void_p, c_int]),
    "px_buffer": (c_int, [c_void_p, c_int, POINTER(c_void_p), POINTER(c_size_t)]),
    "px_get": (c_int, [c_void_p, c_int, c_void_p, c_size_t, c_int, c_void_p]),
    "px_set_timing": (c_int, [c_void_p, c_int]),
    "px_get_timing": (c_int, [c_void_p, POINTER(Timing)]),
    "px_get_kernel_timing": (c_int, [c_void_p, c_int, POINTER(c_double), POINTER(c_uint64)]),
    "px_get_stats": (c_int, [c_void_p, POINTER(Stats)]),
    "px_reset_stats": (c_int, [c_void_p]),
    # the reference's hybrid with its tracking objective (a separate handle)
    "px_hybrid_create": (c_int, [POINTER(HybridDesc), POINTER(c_void_p)]),
    "px_hybrid_destroy": (None, [c_void_p]),
    "px_hybrid_last_error": (ctypes.c_char_p, [c_void_p]),
    "px_hybrid_set_inputs": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_void_p]),
    "px_hybrid_direct": (c_int, [c_void_p, c_int, c_void_p]),
    "px_hybrid_bounds": (c_int, [c_void_p, POINTER(c_double), c_void_p]),
    "px_hybrid_set_slice_plan": (c_int, [c_void_p, c_int, POINTER(ChebPlanC), POINTER(c_double), POINTER(c_double)]),
    "px_hybrid_adjoint": (c_int, [c_void_p, c_void_p]),
    "px_hybrid_nl_init": (c_int, [c_void_p, c_void_p]),
    "px_hybrid_nl_set_plans": (c_int, [c_void_p, POINTER(ChebPlanC), POINTER(ChebPlanC)]),
    "px_hybrid_nl_sweep": (c_int, [c_void_p, POINTER(c_double), c_void_p]),
    "px_hybrid_nl_finish": (c_int, [c_void_p, c_void_p]),
    "px_hybrid_get": (c_int, [c_void_p, c_int, c_void_p, c_size_t, c_int, c_void_p]),
    "px_hybrid_get_timing": (c_int, [c_void_p, POINTER(c_double)]),
}

_lib = None


def load(path: str | None = None):
    """Load the library (idempotent). Raises NativeUnavailable if absent."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or LIB_PATH
    if not os.path.exists(p):
        raise NativeUnavailable(
            f"{p} not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the Paraexp path has no CPU fallback)")
    lib = ctypes.CDLL(p)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.px_abi_version() != ABI_VERSION:
        raise NativeUnavailable("libparaexp.so ABI version mismatch")
    if path is None:
        _lib = lib
    return lib


def check(lib, rc: int, handle=None, t: float = float("nan"), hybrid: bool = False) -> None:
    if rc != 0:
        msg = (lib.px_hybrid_last_error if hybrid else lib.px_last_error)(handle)
        raise_for_status(rc, msg.decode() if msg else "", t)


def dptr(a) -> ctypes.POINTER(c_double):
    import numpy as np
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a.ctypes.data_as(POINTER(c_double)), a


def iptr(a):
    import numpy as np
    a = np.ascontiguousarray(a, dtype=np.int32)
    return a.ctypes.data_as(POINTER(c_int)), a
