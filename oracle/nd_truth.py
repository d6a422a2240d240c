"""CPU ORACLE (test infrastructure only): config-size restatements of the
2-D/3-D fine and coarse maps, fast enough to check the device at the
BASELINE shapes (1024^2, 256^3, 512^3).

* ``StencilND`` — the explicit forward-Euler fine map (I + dt A)^S
  (reference route ``fine_from_onestep(AffinePropagator(I + dt A, dt c, 1), S)``,
  ``model.py:147-154``; A the zero-Dirichlet 3/5/7-point Laplacian,
  ``model.py:209-235`` for 1-D and its Kronecker sums), evaluated by
  ``oracle/stencil_nd.c`` with the per-point expression the device evaluates,
  so fp32/fp64 results are compared bitwise. ``exact=True`` evaluates the same
  map in long double (the rounding floor of the fp64 map).
* ``SpectralND`` — the backward-Euler coarse map (I - dT A)^-1 b, the
  reference's ``_onestep`` + ``lu_solve`` (``model.py:157-184``,
  ``linalg.py:241-266``) solved exactly through the orthonormal sine
  transform that diagonalises A (scipy DST-I, fp64). Its rounding error is a
  few ulps of the condition number (kappa <= 801 at C3), far below the
  per-iteration tolerance; ``tests/test_oracle_nd.py`` pins it against a
  sparse LU of the same system.

The coefficient r = dt/h^2 is formed exactly as the device op forms it
(``dt = span / steps`` in double; ``(float)r`` for fp32).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "libstencil_nd.so")
_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            subprocess.check_call(["make", "-s", "-C", HERE])
        lib = ctypes.CDLL(LIB)
        i64, vp = ctypes.c_int64, ctypes.c_void_p
        for name, rt in (("fe_nd_f64", ctypes.c_double), ("fe_nd_f32", ctypes.c_float),
                         ("fe_nd_ld", ctypes.c_double)):
            f = getattr(lib, name)
            f.restype = ctypes.c_int
            f.argtypes = [ctypes.c_int, i64, i64, i64, vp, i64, rt, i64]
        _lib = lib
    return _lib


def stencil_r(span: float, steps: int, h: float) -> float:
    """r = dt / h^2 with dt = span / steps, in double (as the device op)."""
    dt = float(span) / float(steps)
    return dt / (h * h)


@dataclass
class StencilND:
    """(I + dt A)^S on a C-order grid of ``shape`` (1, 2 or 3 axes)."""

    shape: tuple
    h: float
    span: float
    steps: int
    dtype: type = np.float64
    exact: bool = False

    @property
    def r(self) -> float:
        return stencil_r(self.span, self.steps, self.h)

    def _dims(self):
        s = tuple(int(v) for v in self.shape)
        nd = len(s)
        nz = s[0] if nd == 3 else 1
        ny = s[-2] if nd >= 2 else 1
        return nd, nz, ny, s[-1]

    def apply_batch(self, states: np.ndarray) -> np.ndarray:
        nd, nz, ny, nx = self._dims()
        npts = nz * ny * nx
        lib = _load()
        if self.exact:
            x = np.array(states, dtype=np.float64, copy=True).reshape(-1, npts)
            rc = lib.fe_nd_ld(nd, nz, ny, nx, x.ctypes.data, x.shape[0], self.r, self.steps)
        elif np.dtype(self.dtype) == np.float32:
            x = np.array(states, dtype=np.float32, copy=True).reshape(-1, npts)
            rc = lib.fe_nd_f32(nd, nz, ny, nx, x.ctypes.data, x.shape[0], float(np.float32(self.r)), self.steps)
        else:
            x = np.array(states, dtype=np.float64, copy=True).reshape(-1, npts)
            rc = lib.fe_nd_f64(nd, nz, ny, nx, x.ctypes.data, x.shape[0], self.r, self.steps)
        assert rc == 0
        return x

    def apply(self, u: np.ndarray) -> np.ndarray:
        return self.apply_batch(np.asarray(u).reshape(1, -1))[0]


@dataclass
class SpectralND:
    """(I - dT A)^-1 applied ``steps`` times (backward Euler with step
    dT = span / steps), by the orthonormal DST-I; fp64 arithmetic, result
    cast to ``dtype``."""

    shape: tuple
    h: float
    span: float
    steps: int = 1
    dtype: type = np.float64

    def __post_init__(self):
        dT = float(self.span) / float(self.steps)
        lam = None
        for n in self.shape:
            k = np.arange(1, n + 1, dtype=np.float64)
            l1 = (4.0 / (self.h * self.h)) * np.sin(k * np.pi / (2.0 * (n + 1))) ** 2
            lam = l1 if lam is None else lam[..., None] + l1
        self._inv = 1.0 / (1.0 + dT * np.asarray(lam))

    def apply(self, b: np.ndarray) -> np.ndarray:
        from scipy.fft import dstn, idstn
        x = np.asarray(b, dtype=np.float64).reshape(self.shape)
        for _ in range(self.steps):
            x = idstn(dstn(x, type=1, norm="ortho", workers=-1) * self._inv, type=1, norm="ortho", workers=-1)
        return x.reshape(-1).astype(self.dtype)

    def apply_batch(self, states: np.ndarray) -> np.ndarray:
        return np.stack([self.apply(s) for s in states])
