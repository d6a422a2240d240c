"""CPU ORACLE (test infrastructure only): long-double ground truth for the
1-D implicit rules (oracle/thomas_ld.c, built by oracle/Makefile into
oracle/_build). Coefficients are formed in double exactly as the reference
forms its dense matrices (model.py:172-200); only the solve is carried out in
extended precision, so this is the exact-arithmetic answer to the reference's
own fp64 problem."""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from .heat_oracle import Tridiag1D

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "libthomas_ld.so")
_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            subprocess.check_call(["make", "-s", "-C", HERE])
        lib = ctypes.CDLL(LIB)
        lib.thomas_ld_propagate.restype = ctypes.c_int
        lib.thomas_ld_propagate.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_double,
                                            ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_int64,
                                            ctypes.c_int, ctypes.c_double]
        _lib = lib
    return _lib


class TruthTridiag1D(Tridiag1D):
    """Same construction as heat_oracle.Tridiag1D, long-double solves."""

    def _run(self, states: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(np.array(states, dtype=np.float64, copy=True))
        nb = 1 if x.ndim == 1 else x.shape[0]
        f0 = float(self.f[0])
        f1 = float(self.f[-1]) if self.n > 1 else 0.0
        rc = _load().thomas_ld_propagate(self.n, nb, x.ctypes.data, self.D, self.E, f0, f1, self.steps,
                                         1 if self.rule == "trapezoidal" else 0, self.Dp)
        assert rc == 0
        return x

    def apply(self, u):
        return self._run(np.asarray(u, dtype=float).reshape(-1))

    def apply_batch(self, states):
        return self._run(np.asarray(states, dtype=float))
