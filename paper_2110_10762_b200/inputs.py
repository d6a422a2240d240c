"""Seeded synthetic initial states of the BASELINE configurations (SURVEY
§8d): interior grid s_i = i/(n+1) per axis, sine modes with N(0, 1)
amplitudes drawn from numpy's PCG64 (``default_rng(seed)``, the generator the
reference's schedules use, async_engine.py:201). Built on the host in float64
so the GPU path and the CPU checker see the same bits; no dataset is involved.
"""
from __future__ import annotations

import numpy as np


def interior_grid(n: int) -> np.ndarray:
    return np.arange(1, n + 1, dtype=np.float64) / (n + 1)


def sine_u0_1d(n: int, n_modes: int, seed: int = 0) -> np.ndarray:
    """C1/C2: u0 = sin(pi s) + 0.1 * sum_{j=1..n_modes} a_j sin(j pi s)."""
    amp = np.random.default_rng(seed).standard_normal(n_modes)
    s = interior_grid(n)
    modes = np.zeros(n)
    for j, a in enumerate(amp, start=1):
        modes = modes + a * np.sin(j * np.pi * s)
    return np.sin(np.pi * s) + 0.1 * modes


def modes_2d() -> list[tuple[int, int]]:
    """C3: (j, l) in {1..4}^2, row-major."""
    return [(j, l) for j in range(1, 5) for l in range(1, 5)]


def modes_3d() -> list[tuple[int, int, int]]:
    """C4/C5: (j, l, m) in {1..4} x {1, 2} x {1, 2}."""
    return [(j, l, m) for j in range(1, 5) for l in (1, 2) for m in (1, 2)]


def sine_u0_nd(shape, modes, seed: int = 0) -> np.ndarray:
    """C3-C5: u0 = sum_m a_m prod_d sin(k_{m,d} pi s_d) on a C-order grid."""
    shape = tuple(int(n) for n in shape)
    amp = np.random.default_rng(seed).standard_normal(len(modes))
    axes = [interior_grid(n) for n in shape]
    out = np.zeros(shape)
    for a, ks in zip(amp, modes):
        term = np.ones(shape)
        for d, k in enumerate(ks):
            bshape = [1] * len(shape)
            bshape[d] = shape[d]
            term = term * np.sin(k * np.pi * axes[d]).reshape(bshape)
        out = out + a * term
    return out


def sine_u0(shape, n_modes: int | None = None, seed: int = 0) -> np.ndarray:
    """The configuration's initial state for a 1-D/2-D/3-D grid (flattened)."""
    shape = tuple(int(n) for n in shape)
    if len(shape) == 1:
        return sine_u0_1d(shape[0], 8 if n_modes is None else int(n_modes), seed)
    modes = modes_2d() if len(shape) == 2 else modes_3d()
    return sine_u0_nd(shape, modes, seed).reshape(-1)
