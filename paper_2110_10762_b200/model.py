"""Problems and the propagator plugin layer (reference: pintlab/model.py).

The reference builds each propagator as a materialised dense affine map
``u -> M u + b`` (``AffinePropagator``, model.py:111-133) by composing
``steps`` one-step maps (model.py:136-154). Here a propagator is a handle on
an immutable device operator of libpint_b200: it stores only
(shape, h, dt, steps, rule, dtype) plus exact precomputed solver factors, and
``apply`` runs the steps matrix-free on the B200. The registry keeps the
reference's two rules and adds ``forward-euler`` (the explicit fine
propagator of the 2-D/3-D configurations).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _device, _native
from .errors import DegenerateProblemError, DimensionError, SingularSystemError, SingularMatrixError

UNIT_STEP_COST = 1.0  # cost units charged per step (reference model.py:21)
DENSE_LIMIT = 4096    # largest dim for which .a_mat / .matrix are materialised


# ------------------------------------------------------------------ problems

def _as_matrix(m) -> np.ndarray:
    a = np.asarray(m, dtype=float)
    if a.ndim != 2:
        raise DimensionError(f"expected a 2-D matrix, got ndim={a.ndim}")
    if not np.all(np.isfinite(a)):
        raise ValueError("matrix entries must be finite")
    return a


@dataclass
class LinearIVP:
    """u'(t) = A u(t) + c on [0, T] with u(0) = u0 (reference model.py:24-62).

    Dense form, kept for API parity and small problems. The GPU propagators
    accept it when A is a symmetric constant-coefficient tridiagonal matrix
    (a_diag on the diagonal, a_off on both off-diagonals) and c is nonzero only
    at the end nodes — the structure of heat1d_system and scalar_decay_system.
    """

    a_mat: np.ndarray
    forcing: np.ndarray
    u0: np.ndarray
    t_final: float
    label: str = "ivp"

    def __post_init__(self):
        self.a_mat = _as_matrix(self.a_mat)
        if self.a_mat.shape[0] != self.a_mat.shape[1]:
            raise DimensionError(f"system matrix must be square, got {self.a_mat.shape}")
        self.forcing = np.asarray(self.forcing, dtype=float).reshape(-1)
        self.u0 = np.asarray(self.u0, dtype=float).reshape(-1)
        n = self.a_mat.shape[0]
        if self.forcing.shape[0] != n or self.u0.shape[0] != n:
            raise DimensionError("forcing and initial state must match the matrix size")
        self.t_final = float(self.t_final)
        if not self.t_final > 0.0:
            raise ValueError(f"final time must be positive, got {self.t_final}")

    @property
    def dim(self) -> int:
        return self.a_mat.shape[0]

    def to_dict(self) -> dict:
        return {"A": self.a_mat.tolist(), "c": self.forcing.tolist(), "u0": self.u0.tolist(),
                "T": self.t_final, "label": self.label}

    @classmethod
    def from_dict(cls, doc: dict) -> "LinearIVP":
        return cls(doc["A"], doc["c"], doc["u0"], doc["T"], doc.get("label", "ivp"))


@dataclass
class HeatIVP:
    """Matrix-free method-of-lines heat equation on [0, L]^d, n interior nodes
    per axis, h = L/(n+1), Dirichlet boundary values (1-D: left/right; 2-D/3-D:
    zero). ``A = h^-2 * (2d+1)-point Laplacian``; the boundary values enter the
    forcing at the end nodes exactly as in heat1d_system (model.py:209-235).
    """

    shape: tuple
    length: float
    boundary_left: float
    boundary_right: float
    u0: np.ndarray
    t_final: float
    label: str = "heat"

    def __post_init__(self):
        self.shape = tuple(int(n) for n in self.shape)
        if not 1 <= len(self.shape) <= 3:
            raise DimensionError("heat problems are 1-D, 2-D or 3-D")
        if any(n < 1 for n in self.shape):
            raise DegenerateProblemError(f"need at least one interior node per axis, got {self.shape}")
        if not self.length > 0.0:
            raise ValueError(f"rod length must be positive, got {self.length}")
        if len(set(self.shape)) != 1 and len(self.shape) > 1:
            raise DimensionError("2-D/3-D heat grids must have equal spacing (same n per axis)")
        if len(self.shape) > 1 and (self.boundary_left != 0.0 or self.boundary_right != 0.0):
            raise ValueError("2-D/3-D heat problems use zero Dirichlet boundaries")
        self.u0 = np.asarray(self.u0, dtype=float).reshape(-1)
        if self.u0.shape[0] != self.dim:
            raise DimensionError("initial state does not match the grid")
        self.t_final = float(self.t_final)
        if not self.t_final > 0.0:
            raise ValueError(f"final time must be positive, got {self.t_final}")

    @property
    def ndim(self) -> int:
        return len(self.shape)

    @property
    def dim(self) -> int:
        return int(np.prod(self.shape))

    @property
    def h(self) -> float:
        return self.length / (self.shape[0] + 1)

    @property
    def inv_h2(self) -> float:
        h = self.h
        return 1.0 / (h * h)

    def coefficients_1d(self):
        """(a_diag, a_off, c_first, c_last) formed as model.py:226-234 forms them."""
        inv_h2 = self.inv_h2
        n = self.shape[0]
        c = np.zeros(n)
        c[0] += self.boundary_left * inv_h2
        c[-1] += self.boundary_right * inv_h2
        return inv_h2 * -2.0, inv_h2 * 1.0, float(c[0]), float(c[-1])

    @property
    def a_mat(self) -> np.ndarray:
        if self.dim > DENSE_LIMIT:
            raise NotImplementedError(f"dense A of a {self.dim}-point grid is not materialised")
        lap = None
        for d, n in enumerate(self.shape):
            t = np.diag(np.full(n, -2.0)) + np.diag(np.ones(n - 1), 1) + np.diag(np.ones(n - 1), -1)
            for e, m in enumerate(self.shape):
                if e < d:
                    t = np.kron(np.eye(m), t)
                elif e > d:
                    t = np.kron(t, np.eye(m))
            lap = t if lap is None else lap + t
        return self.inv_h2 * lap

    @property
    def forcing(self) -> np.ndarray:
        c = np.zeros(self.dim)
        if self.ndim == 1:
            inv_h2 = self.inv_h2
            c[0] += self.boundary_left * inv_h2
            c[-1] += self.boundary_right * inv_h2
        return c

    def to_dict(self) -> dict:
        return {"heat": {"shape": list(self.shape), "length": self.length,
                         "boundary_left": self.boundary_left, "boundary_right": self.boundary_right},
                "u0": self.u0.tolist(), "T": self.t_final, "label": self.label}

    @classmethod
    def from_dict(cls, doc: dict) -> "HeatIVP":
        h = doc["heat"]
        return cls(tuple(h["shape"]), h["length"], h["boundary_left"], h["boundary_right"],
                   doc["u0"], doc["T"], doc.get("label", "heat"))


def heat1d_system(n_interior: int, length: float, boundary_left: float, boundary_right: float,
                  initial_temp: float, t_final: float) -> HeatIVP:
    """Same signature and operator as the reference (model.py:209-235), built
    matrix-free (the dense A of N = 65,536 would be 32 GiB)."""
    if n_interior < 1:
        raise DegenerateProblemError(f"need at least one interior node, got {n_interior}")
    if not length > 0.0:
        raise ValueError(f"rod length must be positive, got {length}")
    u0 = np.full(n_interior, float(initial_temp))
    return HeatIVP((n_interior,), float(length), float(boundary_left), float(boundary_right), u0,
                   t_final, label=f"heat1d-n{n_interior}")


def heat2d_system(n: int, t_final: float, u0=None, length: float = 1.0) -> HeatIVP:
    """2-D heat on [0, L]^2, n x n interior nodes, zero Dirichlet (BASELINE C3)."""
    u0 = np.zeros(n * n) if u0 is None else u0
    return HeatIVP((n, n), float(length), 0.0, 0.0, u0, t_final, label=f"heat2d-n{n}")


def heat3d_system(n: int, t_final: float, u0=None, length: float = 1.0) -> HeatIVP:
    """3-D heat on [0, L]^3, n^3 interior nodes, zero Dirichlet (BASELINE C4/C5)."""
    u0 = np.zeros(n ** 3) if u0 is None else u0
    return HeatIVP((n, n, n), float(length), 0.0, 0.0, u0, t_final, label=f"heat3d-n{n}")


def scalar_decay_system(rate: float = 1.0, initial: float = 1.0, t_final: float = 1.0) -> LinearIVP:
    """u' = -rate * u (reference model.py:238-243)."""
    if not rate > 0.0:
        raise ValueError(f"decay rate must be positive, got {rate}")
    return LinearIVP([[-rate]], [0.0], [initial], t_final, label="scalar-decay")


@dataclass
class TimeDecomposition:
    """Uniform split of [0, T] into p subintervals (reference model.py:65-108)."""

    p: int
    coarse_dt: float
    fine_dt: float

    def __post_init__(self):
        self.p = int(self.p)
        self.coarse_dt = float(self.coarse_dt)
        self.fine_dt = float(self.fine_dt)
        if self.p < 1:
            raise ValueError(f"need at least one subinterval, got p={self.p}")
        if not self.coarse_dt > 0.0 or not self.fine_dt > 0.0:
            raise ValueError("step widths must be positive")
        steps = self.coarse_dt / self.fine_dt
        if abs(round(steps) - steps) > 1e-9 * max(steps, 1.0) or round(steps) < 1:
            raise ValueError(f"fine step {self.fine_dt} does not divide subinterval {self.coarse_dt}")

    @property
    def fine_steps(self) -> int:
        return int(round(self.coarse_dt / self.fine_dt))

    @property
    def t_final(self) -> float:
        return self.p * self.coarse_dt

    @property
    def boundaries(self) -> np.ndarray:
        return np.arange(self.p + 1) * self.coarse_dt

    def to_dict(self) -> dict:
        return {"p": self.p, "coarse_dt": self.coarse_dt, "fine_dt": self.fine_dt}

    @classmethod
    def from_dict(cls, doc: dict) -> "TimeDecomposition":
        return cls(doc["p"], doc["coarse_dt"], doc["fine_dt"])


# --------------------------------------------------------------- propagators

def _tridiag_structure(ivp: LinearIVP):
    """(a_diag, a_off, c_first, c_last) of a dense LinearIVP with the
    supported structure, else None."""
    a = ivp.a_mat
    n = a.shape[0]
    c = ivp.forcing
    a_d = float(a[0, 0])
    a_o = float(a[0, 1]) if n > 1 else 0.0
    model = np.diag(np.full(n, a_d))
    if n > 1:
        model = model + np.diag(np.full(n - 1, a_o), 1) + np.diag(np.full(n - 1, a_o), -1)
    if not np.array_equal(a, model):
        return None
    inner = c[1:-1] if n > 2 else np.zeros(0)
    if np.any(inner != 0.0):
        return None
    return a_d, a_o, float(c[0]), float(c[-1]) if n > 1 else 0.0


class GPUPropagator:
    """Immutable propagator over one time span, executed on a B200.

    Reference protocol (model.py:111-133, cli.py:273-276): ``apply(state)``
    returns a new state, ``.dim``, ``.cost_units``. Added for the hot path:
    ``apply_batch`` advances many independent slices in one launch.
    """

    def __init__(self, desc: _native.OpDesc, dim: int, dtype: torch.dtype, cost_units: float,
                 device: int, rule: str, span: float, steps: int):
        self._lib = _native.load_library()
        self.device = int(device)
        self._ctx = _native.context(self.device)
        self.desc = desc
        h = ctypes.c_void_p()
        rc = self._lib.pint_op_create(self._ctx.handle, ctypes.byref(desc), ctypes.byref(h))
        if rc == _native.PINT_ESINGULAR:
            pivot = self._lib.pint_last_error_value(self._ctx.handle)
            msg = self._lib.pint_last_error(self._ctx.handle).decode()
            dt = span / steps
            raise SingularSystemError(f"implicit step with dt={dt} is singular ({msg})", dt=dt, pivot=pivot)
        _native.check(rc, self._ctx.handle, "pint_op_create")
        self.handle = h
        self._dim = int(dim)
        self.dtype = dtype
        self.cost_units = float(cost_units)
        self.rule = rule
        self.span = float(span)
        self.steps = int(steps)
        info = _native.OpInfo()
        _native.check(self._lib.pint_op_get_info(h, ctypes.byref(info)), self._ctx.handle)
        self.info = info

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                self._lib.pint_op_destroy(self.handle)
                self.handle = None
        except Exception:
            pass

    @property
    def dim(self) -> int:
        return self._dim

    @property
    def is_tridiagonal(self) -> bool:
        return self.desc.ndim == 1 and self.desc.rule != _native.RULE_FORWARD_EULER

    # ---- raw device entry (pointers), stream-ordered on the current stream
    def apply_ptr(self, in_ptr: int, out_ptr: int, nbatch: int, stride: int, stream: int | None = None) -> None:
        s = _device.stream_ptr(self.device) if stream is None else stream
        rc = self._lib.pint_op_apply_batch(self.handle, ctypes.c_void_p(in_ptr), ctypes.c_void_p(out_ptr),
                                           int(nbatch), int(stride), ctypes.c_void_p(s))
        _native.check(rc, self._ctx.handle, "pint_op_apply_batch")

    def apply_batch(self, states: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """states (nbatch, dim) device tensor -> (nbatch, dim); one launch."""
        if states.dim() != 2 or states.shape[1] != self._dim:
            raise DimensionError(f"states have shape {tuple(states.shape)}, propagator expects (*, {self._dim})")
        if not states.is_cuda or states.dtype != self.dtype:
            states = states.to(device=f"cuda:{self.device}", dtype=self.dtype)
        if states.stride(1) != 1:
            states = states.contiguous()
        if out is None:
            out = torch.empty_like(states)
        nb = states.shape[0]
        if nb:
            self.apply_ptr(states.data_ptr(), out.data_ptr(), nb, states.stride(0))
        return out

    def apply(self, state):
        """Reference contract: a new state of the same kind (numpy in ->
        numpy out; torch tensor in -> CUDA tensor out)."""
        is_torch = isinstance(state, torch.Tensor)
        n = int(state.numel()) if is_torch else int(np.asarray(state).size)
        if n != self._dim:
            raise DimensionError(f"state has dim {n}, propagator expects {self._dim}")
        t, _ = _device.as_device_tensor(state, self.device, self.dtype)
        out = self.apply_batch(t.reshape(1, -1)).reshape(-1)
        if is_torch:
            return out
        return _device.to_host(out).astype(float)

    # ---- dense views for analysis at small sizes (reference .matrix/.offset)
    @property
    def offset(self) -> np.ndarray:
        if self._dim > DENSE_LIMIT:
            raise NotImplementedError("dense offset of a large operator is not materialised")
        z = torch.zeros(1, self._dim, dtype=self.dtype, device=f"cuda:{self.device}")
        return _device.to_host(self.apply_batch(z)[0]).astype(float)

    @property
    def matrix(self) -> np.ndarray:
        if self._dim > DENSE_LIMIT:
            raise NotImplementedError("dense matrix of a large operator is not materialised")
        eye = torch.eye(self._dim, dtype=self.dtype, device=f"cuda:{self.device}")
        cols = self.apply_batch(eye)
        z = self.apply_batch(torch.zeros(1, self._dim, dtype=self.dtype, device=eye.device))
        return _device.to_host((cols - z).T).astype(float)


# 2-D/3-D implicit step: "direct" = sine-transform diagonalisation (exact to
# rounding, as the reference's dense LU); "cg" = conjugate gradients to cg_rtol.
ND_SOLVERS = {"direct": 0, "cg": 1}


def _build(ivp, span: float, steps: int, rule: str, *, dtype=None, device=None,
           cg_rtol: float | None = None, cg_maxit: int = 10_000, solver: str = "direct") -> GPUPropagator:
    if steps < 1:
        raise ValueError(f"step count must be >= 1, got {steps}")
    if not span > 0.0:
        raise ValueError(f"span must be positive, got {span}")
    dev = _device.device_index(device)
    rid = {"backward-euler": _native.RULE_BACKWARD_EULER, "trapezoidal": _native.RULE_TRAPEZOIDAL,
           "forward-euler": _native.RULE_FORWARD_EULER}[rule]
    d = _native.OpDesc()
    d.rule = rid
    d.span = float(span)
    d.steps = int(steps)
    tdt = _device.torch_dtype(dtype) if dtype is not None else torch.float64
    d.dtype = _native.PINT_F64 if tdt == torch.float64 else _native.PINT_F32
    if isinstance(ivp, HeatIVP) and ivp.ndim >= 2 or (isinstance(ivp, HeatIVP) and rule == "forward-euler"):
        if ivp.boundary_left != 0.0 or ivp.boundary_right != 0.0:
            raise NotImplementedError("explicit/CG heat propagators use zero Dirichlet boundaries")
        d.ndim = ivp.ndim
        for i, n in enumerate(ivp.shape):
            d.shape[i] = n
        d.h = ivp.h
        if cg_rtol is None:
            cg_rtol = 1e-12 if tdt == torch.float64 else 1e-6
        d.cg_rtol = float(cg_rtol)
        d.cg_maxit = int(cg_maxit)
        if solver not in ND_SOLVERS:
            raise ValueError(f"solver must be one of {sorted(ND_SOLVERS)}, got {solver!r}")
        d.nd_solver = ND_SOLVERS[solver]
        dim = ivp.dim
    else:
        if rule == "forward-euler":
            raise NotImplementedError("forward-euler is provided for the zero-Dirichlet heat operators")
        if tdt != torch.float64:
            raise NotImplementedError("1-D implicit propagators compute in float64")
        if isinstance(ivp, HeatIVP):
            a_d, a_o, c0, c1 = ivp.coefficients_1d()
            if ivp.dim == 1:
                c1 = 0.0  # c[0] already holds both boundary contributions
        elif isinstance(ivp, LinearIVP):
            st = _tridiag_structure(ivp)
            if st is None:
                raise NotImplementedError(
                    "GPU propagators need a symmetric constant-coefficient tridiagonal A with end-node"
                    " forcing (heat1d_system / scalar_decay_system structure)")
            a_d, a_o, c0, c1 = st
        else:
            raise TypeError(f"unsupported problem type {type(ivp).__name__}")
        d.ndim = 1
        d.shape[0] = ivp.dim
        d.a_diag, d.a_off, d.c_first, d.c_last = a_d, a_o, c0, c1
        dim = ivp.dim
    try:
        return GPUPropagator(d, dim, tdt, steps * UNIT_STEP_COST, dev, rule, span, steps)
    except SingularMatrixError as err:  # pragma: no cover - mapped above
        raise SingularSystemError(str(err), dt=span / steps, pivot=err.pivot) from err


def backward_euler_propagator(ivp, span: float, steps: int, **kw) -> GPUPropagator:
    """Backward Euler over ``span`` in ``steps`` implicit steps (model.py:172-184)."""
    return _build(ivp, span, steps, "backward-euler", **kw)


def trapezoidal_propagator(ivp, span: float, steps: int, **kw) -> GPUPropagator:
    """Trapezoidal rule over ``span`` in ``steps`` implicit steps (model.py:187-200)."""
    return _build(ivp, span, steps, "trapezoidal", **kw)


def forward_euler_propagator(ivp, span: float, steps: int, **kw) -> GPUPropagator:
    """Explicit Euler, the fine propagator of the 2-D/3-D configurations
    (reference route: fine_from_onestep(AffinePropagator(I + dt A, dt c, 1), S))."""
    return _build(ivp, span, steps, "forward-euler", **kw)


PROPAGATOR_RULES = {
    "backward-euler": backward_euler_propagator,
    "trapezoidal": trapezoidal_propagator,
    "forward-euler": forward_euler_propagator,
}


def with_register_layout(prop: GPUPropagator, points_per_thread: int) -> GPUPropagator:
    """The same operator built with another register layout (1-D implicit
    operators: 16 or 32 points per thread). Used to pair a backward-Euler
    coarse operator with a trapezoidal fine operator inside one persistent
    kernel; values agree with ``prop`` to rounding, not bitwise."""
    if prop.info.points_per_thread == points_per_thread:
        return prop
    d = _native.OpDesc()
    ctypes.memmove(ctypes.byref(d), ctypes.byref(prop.desc), ctypes.sizeof(d))
    d.layout_ch = int(points_per_thread)
    return GPUPropagator(d, prop.dim, prop.dtype, prop.cost_units, prop.device, prop.rule, prop.span, prop.steps)
