"""ctypes binding of libpint_b200.so (include/pint_abi.h).

This is the Python side of the C ABI: the exact stub a maintainer of the
reference would add. It loads the in-tree library built
by ``paper_2110_10762_b200.build`` and fails loudly if it is missing — there
is no CPU fallback anywhere in the product path.
"""
from __future__ import annotations

import ctypes
import os
import threading

from . import errors

PKG = os.path.dirname(os.path.abspath(__file__))
# PINT_LIB_PATH selects an alternative build (e.g. the phase-timing debug library)
LIB_PATH = os.environ.get("PINT_LIB_PATH") or os.path.join(PKG, "libpint_b200.so")

PINT_OK = 0
PINT_EDIM = 1
PINT_EARG = 2
PINT_ENONFINITE = 3
PINT_ENOCONV = 4
PINT_ESINGULAR = 5
PINT_ECUDA = 6
PINT_EUNSUPPORTED = 7

PINT_F32 = 0
PINT_F64 = 1

RULE_BACKWARD_EULER = 0
RULE_TRAPEZOIDAL = 1
RULE_FORWARD_EULER = 2

c_void_p = ctypes.c_void_p
c_int = ctypes.c_int
c_i32 = ctypes.c_int32
c_i64 = ctypes.c_int64
c_double = ctypes.c_double


class OpDesc(ctypes.Structure):
    _fields_ = [
        ("ndim", c_i32), ("rule", c_i32), ("dtype", c_i32), ("nd_solver", c_i32),
        ("shape", c_i64 * 3), ("h", c_double), ("span", c_double), ("steps", c_i64),
        ("a_diag", c_double), ("a_off", c_double), ("c_first", c_double), ("c_last", c_double),
        ("cg_rtol", c_double), ("cg_maxit", c_i64), ("layout_ch", c_i32), ("reserved1", c_i32),
    ]


class OpInfo(ctypes.Structure):
    _fields_ = [
        ("dim", c_i64), ("steps", c_i64), ("dtype", c_i32), ("rule", c_i32),
        ("threads_per_slice", c_i32), ("points_per_thread", c_i32),
        ("batch_cluster", c_i32), ("sweep_cluster", c_i32),
        ("dt", c_double), ("diag", c_double), ("offdiag", c_double), ("min_pivot", c_double),
        ("batch_wave_slices", c_i32), ("fused_sweep", c_i32),
        ("general", c_i32), ("reserved0", c_i32),
    ]


# name -> (restype, argtypes); every symbol declared in include/pint_abi.h
SIGNATURES = {
    "pint_abi_version": (c_int, []),
    "pint_ctx_create": (c_int, [c_int, ctypes.POINTER(c_void_p)]),
    "pint_ctx_destroy": (c_int, [c_void_p]),
    "pint_last_error": (ctypes.c_char_p, [c_void_p]),
    "pint_last_error_value": (c_double, [c_void_p]),
    "pint_op_create": (c_int, [c_void_p, ctypes.POINTER(OpDesc), ctypes.POINTER(c_void_p)]),
    "pint_op_destroy": (c_int, [c_void_p]),
    "pint_op_get_info": (c_int, [c_void_p, ctypes.POINTER(OpInfo)]),
    "pint_op_apply_batch": (c_int, [c_void_p, c_void_p, c_void_p, c_i64, c_i64, c_void_p]),
    "pint_correct": (c_int, [c_void_p, c_i32, c_i64, c_i64, c_void_p, c_void_p, c_void_p, c_void_p,
                             c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "pint_coarse_init": (c_int, [c_void_p, c_void_p, c_i64, c_void_p, c_void_p]),
    "pint_sync_sweep": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_i64, c_i64,
                                c_void_p, c_void_p, c_void_p]),
    "pint_sync_sweep_chain": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_i64, c_i64,
                                      c_void_p, c_void_p, c_void_p]),
    "pint_async_run": (c_int, [c_void_p, c_void_p, c_void_p, c_i64, c_double, c_i64, c_double, ctypes.c_uint64,
                               c_void_p, c_void_p, c_void_p, c_void_p]),
    "pint_async_run_traced": (c_int, [c_void_p, c_void_p, c_void_p, c_i64, c_double, c_i64, c_double,
                                      ctypes.c_uint64, c_void_p, c_void_p, c_void_p, c_void_p, c_i64, c_void_p]),
    "pint_async_domain_create": (c_int, [c_void_p, c_void_p, c_i64, c_i64, c_i64, c_int, c_int, c_i64, c_i64,
                                         ctypes.POINTER(c_void_p)]),
    "pint_async_domain_ipc_handle": (c_int, [c_void_p, c_void_p]),
    "pint_async_domain_connect": (c_int, [c_void_p, c_void_p, c_void_p]),
    "pint_async_domains_connect_local": (c_int, [c_int, c_void_p]),
    "pint_async_domain_reset": (c_int, [c_void_p, c_void_p, c_void_p]),
    "pint_async_domain_launch": (c_int, [c_int, c_void_p, c_double, c_i64, c_double, ctypes.c_uint64, c_void_p]),
    "pint_async_domain_collect": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_i64, c_void_p]),
    "pint_async_domain_destroy": (c_int, [c_void_p]),
    "pint_async_run_domains": (c_int, [c_void_p, c_void_p, c_void_p, c_i64, c_int, c_double, c_i64, c_double,
                                       ctypes.c_uint64, c_void_p, c_void_p, c_void_p, c_void_p, c_i64, c_void_p]),
    "pint_max_reduce": (c_int, [c_void_p, c_void_p, c_i64, c_i64, c_void_p, c_void_p]),
    "pint_equal_flag": (c_int, [c_void_p, c_i32, c_i64, c_void_p, c_void_p, c_void_p, c_void_p]),
    "pint_correct_chain": (c_int, [c_void_p, c_i32, c_i64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                   c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "pint_shared_alloc": (c_int, [c_void_p, c_i64, ctypes.POINTER(c_void_p)]),
    "pint_shared_free": (c_int, [c_void_p, c_void_p]),
    "pint_ipc_export": (c_int, [c_void_p, c_void_p, c_void_p]),
    "pint_ipc_open": (c_int, [c_void_p, c_void_p, ctypes.POINTER(c_void_p)]),
    "pint_ipc_close": (c_int, [c_void_p, c_void_p]),
    "pint_mailbox_push": (c_int, [c_void_p, c_void_p, c_void_p, c_i64, c_void_p, c_i64, c_void_p, c_void_p]),
    "pint_mailbox_read": (c_int, [c_void_p, c_void_p, c_i64, c_i64, c_void_p, c_void_p, c_i64, c_void_p, c_void_p,
                                  c_void_p, c_void_p]),
    "pint_mailbox_wait": (c_int, [c_void_p, c_void_p, c_i64, c_double, c_void_p, c_void_p]),
    "pint_board_post": (c_int, [c_void_p, c_void_p, c_i64, c_void_p, c_void_p]),
    "pint_board_read": (c_int, [c_void_p, c_void_p, c_i32, c_void_p, c_void_p]),
    "pint_tri1d_plan_host": (c_int, [ctypes.POINTER(OpDesc), c_void_p, c_void_p, c_void_p, c_void_p]),
    "pint_tri1d_ccst_host": (c_int, [ctypes.POINTER(OpDesc), c_void_p, c_void_p]),
}

_lib = None
_lock = threading.Lock()


def load_library():
    """Load (once) and type the shared library. Raises NativeLibraryError."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise errors.NativeLibraryError(
                f"{LIB_PATH} is missing; build it with `python -m paper_2110_10762_b200.build`"
                " (there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.pint_abi_version() != 1:
            raise errors.NativeLibraryError("libpint_b200 ABI version mismatch")
        _lib = lib
        return lib


def check(rc: int, ctx, what: str = "") -> None:
    """Raise the reference-taxonomy exception for a nonzero status."""
    if rc == PINT_OK:
        return
    lib = load_library()
    msg = lib.pint_last_error(ctx).decode(errors="replace")
    val = lib.pint_last_error_value(ctx) if ctx else 0.0
    text = f"{what}: {msg}" if what else msg
    if rc == PINT_EDIM:
        raise errors.DimensionError(text)
    if rc == PINT_EARG:
        raise ValueError(text)
    if rc == PINT_ENONFINITE:
        raise ValueError(text)
    if rc == PINT_ENOCONV:
        raise errors.ConvergenceFailure(text, estimate=val)
    if rc == PINT_ESINGULAR:
        raise errors.SingularMatrixError(text, pivot=val)
    if rc == PINT_EUNSUPPORTED:
        raise NotImplementedError(text)
    raise RuntimeError(f"CUDA error in libpint_b200: {text}")


class Context:
    """One pint_ctx per CUDA device (not thread-safe, like the C object)."""

    def __init__(self, device: int):
        lib = load_library()
        h = c_void_p()
        rc = lib.pint_ctx_create(int(device), ctypes.byref(h))
        check(rc, None, f"pint_ctx_create(device={device})")
        self.handle = h
        self.device = int(device)

    def __del__(self):
        try:
            if getattr(self, "handle", None) and _lib is not None:
                _lib.pint_ctx_destroy(self.handle)
        except Exception:
            pass


_contexts: dict[int, Context] = {}


def context(device: int) -> Context:
    with _lock:
        ctx = _contexts.get(device)
    if ctx is None:
        ctx = Context(device)
        with _lock:
            _contexts[device] = ctx
    return ctx
