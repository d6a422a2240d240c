"""Contraction factors of a (coarse, fine) propagator pair (SURVEY §8f row
f4): the reference's certificate layer (analysis.py:36-160) kept by name,
with the operator norms measured matrix-free on the GPU propagators instead
of on dense ``.matrix`` arrays (analysis.py:92-98), so alpha = ||G|| and
alpha~ = ||G|| + ||F - G|| are available at full size (C2: N = 65,536).

Spectral norm: the heat step maps are symmetric (rational functions or
powers of the symmetric A), so ||M||_2 = max |eigenvalue|, found by Lanczos
with full reorthogonalisation on device vectors (the reference's Gram power
iteration, linalg.py:154-238, stalls on the nearly degenerate top modes of
F - G at full size). Infinity norm: exact row sums of |M| from the
GPU-densified operator for dim <= DENSE_LIMIT.
"""
from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import numpy as np
import torch

from .errors import ConvergenceFailure, InvalidThetaError

LANCZOS_TOL = 1e-12
LANCZOS_MAX_ITER = 400
REORTH_BYTES = 2 << 30  # keep every Lanczos vector while they fit in 2 GiB


class NormKind(Enum):
    """Which operator norm drives an analysis (linalg.py:30-38)."""

    INFINITY = "infinity"
    SPECTRAL = "spectral"


@dataclass(frozen=True)
class ContractionReport:
    """Norm data and the derived contraction factors (analysis.py:36-56)."""

    coarse_norm: float
    defect_norm: float
    theta: float
    sync_factor: float
    async_factor: float
    p: int
    norm_kind: NormKind

    def to_dict(self) -> dict:
        return {"coarse_norm": self.coarse_norm, "defect_norm": self.defect_norm, "theta": self.theta,
                "sync_factor": self.sync_factor, "async_factor": self.async_factor, "p": self.p,
                "norm_kind": self.norm_kind.value}


def factors_from_norms(coarse_norm: float, defect_norm: float, p: int, kind: NormKind = NormKind.SPECTRAL,
                       theta: float | None = None) -> ContractionReport:
    """sync = (1 - theta^p) / (1 - theta) * defect (p * defect at theta = 1),
    async = coarse + defect; theta defaults to the coarse norm and may not be
    below it (analysis.py:59-89)."""
    if p < 1:
        raise ValueError(f"need p >= 1, got {p}")
    if coarse_norm < 0.0 or defect_norm < 0.0:
        raise ValueError("norms must be nonnegative")
    th = coarse_norm if theta is None else float(theta)
    if th < coarse_norm:
        raise InvalidThetaError(f"theta={th} is below the coarse norm {coarse_norm}; the geometric-sum bound "
                                "needs theta >= that norm")
    sync = p * defect_norm if th == 1.0 else (1.0 - th ** p) / (1.0 - th) * defect_norm
    return ContractionReport(coarse_norm=float(coarse_norm), defect_norm=float(defect_norm), theta=th,
                             sync_factor=float(sync), async_factor=float(coarse_norm + defect_norm), p=p,
                             norm_kind=kind)


class CheckResult(tuple):
    """(holds, margin) with attribute access; margin > 0 iff holds (analysis.py:101-114)."""

    __slots__ = ()

    def __new__(cls, holds: bool, margin: float):
        return super().__new__(cls, (bool(holds), float(margin)))

    @property
    def holds(self) -> bool:
        return self[0]

    @property
    def margin(self) -> float:
        return self[1]


def sync_convergence_check(report: ContractionReport) -> CheckResult:
    """Coarse map contracts and coarse + defect < 1 + coarse^p * defect;
    the margin is the smaller slack (analysis.py:117-130)."""
    slack_coarse = 1.0 - report.coarse_norm
    slack_combined = 1.0 + report.coarse_norm ** report.p * report.defect_norm - report.async_factor
    return CheckResult(slack_coarse > 0.0 and slack_combined > 0.0, min(slack_coarse, slack_combined))


def async_convergence_check(report: ContractionReport) -> CheckResult:
    """coarse + defect < 1 (analysis.py:133-136)."""
    margin = 1.0 - report.async_factor
    return CheckResult(margin > 0.0, margin)


@dataclass(frozen=True)
class RateComparison:
    """Ordering certificate between the two factors (analysis.py:139-146)."""

    applicable: bool
    sync_factor: float
    async_factor: float
    gap: float | None


def compare_factors(report: ContractionReport) -> RateComparison:
    """sync < async is certified whenever async < 1; needs theta == coarse
    norm (analysis.py:149-165)."""
    if report.theta != report.coarse_norm:
        raise ValueError(f"rate comparison needs theta == coarse_norm; got theta={report.theta}, "
                         f"coarse_norm={report.coarse_norm}")
    if report.async_factor >= 1.0:
        return RateComparison(False, report.sync_factor, report.async_factor, None)
    return RateComparison(True, report.sync_factor, report.async_factor, report.async_factor - report.sync_factor)


# ------------------------------------------------------ matrix-free norms

def _linear_part(prop):
    """x -> M x for an affine GPU propagator x -> M x + b (batched rows)."""
    dev = f"cuda:{prop.device}"
    zero = torch.zeros(1, prop.dim, dtype=prop.dtype, device=dev)
    b = prop.apply_batch(zero)

    def apply(x: torch.Tensor) -> torch.Tensor:
        return prop.apply_batch(x) - b

    return apply


def symmetric_norm(apply, dim: int, dtype, device, *, tol: float = LANCZOS_TOL, max_iter: int = LANCZOS_MAX_ITER,
                   seed: int = 0) -> float:
    """max |eigenvalue| of a symmetric linear operator (= its 2-norm) by
    Lanczos from a seeded Gaussian start; full reorthogonalisation while the
    basis fits in REORTH_BYTES. Converged when the estimate moves by at most
    tol (relative) over two consecutive steps, or the Krylov space closes."""
    g = torch.Generator().manual_seed(seed)
    v = torch.randn(dim, generator=g, dtype=torch.float64).to(device=device, dtype=dtype)
    v = v / torch.linalg.vector_norm(v.double()).to(dtype)
    keep = dim * np.dtype(np.float64 if dtype == torch.float64 else np.float32).itemsize * max_iter <= REORTH_BYTES
    basis = [v] if keep else None
    alphas, betas = [], []
    v_prev = torch.zeros_like(v)
    beta = 0.0
    est_hist = []
    for j in range(min(max_iter, dim)):
        w = apply(v.reshape(1, -1)).reshape(-1)
        a = float(torch.dot(w.double(), v.double()))
        w = w - a * v - beta * v_prev
        if keep:
            for _ in range(2):  # classical Gram-Schmidt twice
                q = torch.stack(basis)
                w = w - (q.T @ (q.double() @ w.double()).to(dtype))
        alphas.append(a)
        beta = float(torch.linalg.vector_norm(w.double()))
        t = np.diag(alphas) + (np.diag(betas, 1) + np.diag(betas, -1) if betas else 0.0)
        theta = np.linalg.eigvalsh(t)
        est = float(np.max(np.abs(theta)))
        est_hist.append(est)
        if beta <= 1e-14 * max(est, 1e-300) or j == dim - 1:  # invariant subspace / full space: exact
            return est
        if len(est_hist) >= 3 and all(abs(est - e) <= tol * max(est, 1e-300) for e in est_hist[-3:-1]):
            return est
        betas.append(beta)
        v_prev, v = v, w / beta
        if keep:
            basis.append(v)
    raise ConvergenceFailure(f"Lanczos norm estimate did not settle within {max_iter} iterations "
                             f"(estimate {est_hist[-1]:.6e})", estimate=est_hist[-1])


def operator_norm(prop, kind: NormKind = NormKind.SPECTRAL, **kw) -> float:
    """Induced norm of a GPU propagator's linear part (linalg.py:154-174)."""
    lin = _linear_part(prop)
    if kind is NormKind.INFINITY:
        from .model import DENSE_LIMIT
        if prop.dim > DENSE_LIMIT:
            raise NotImplementedError("infinity norm needs the dense matrix (dim <= DENSE_LIMIT)")
        return float(np.max(np.sum(np.abs(prop.matrix), axis=1)))
    return symmetric_norm(lin, prop.dim, prop.dtype, f"cuda:{prop.device}", **kw)


def contraction_factors(coarse, fine, p: int, kind: NormKind = NormKind.SPECTRAL, theta: float | None = None,
                        **kw) -> ContractionReport:
    """Measure ||G|| and ||F - G|| of live propagators and derive both
    factors (analysis.py:92-98), matrix-free for the spectral norm."""
    if coarse.dim != fine.dim:
        from .errors import DimensionError
        raise DimensionError("coarse and fine propagators differ in dimension")
    if kind is NormKind.INFINITY:
        from .model import DENSE_LIMIT
        if fine.dim > DENSE_LIMIT:
            raise NotImplementedError("infinity norm needs the dense matrices (dim <= DENSE_LIMIT)")
        gm, fm = coarse.matrix, fine.matrix
        cn = float(np.max(np.sum(np.abs(gm), axis=1)))
        dn = float(np.max(np.sum(np.abs(fm - gm), axis=1)))
        return factors_from_norms(cn, dn, p, kind=kind, theta=theta)
    g_lin, f_lin = _linear_part(coarse), _linear_part(fine)
    dev = f"cuda:{fine.device}"
    cn = symmetric_norm(g_lin, coarse.dim, coarse.dtype, dev, **kw)
    dn = symmetric_norm(lambda x: f_lin(x) - g_lin(x), fine.dim, fine.dtype, dev, **kw)
    return factors_from_norms(cn, dn, p, kind=kind, theta=theta)
