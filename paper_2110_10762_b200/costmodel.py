"""Parareal cost / speedup model, the reference's wall
model (analysis.py:255-392) kept by name, plus the glue that feeds it with
costs measured on the B200 (``measure_costs``).

Model units are whatever the caller uses for ``fine_cost``/``coarse_cost``
(the reference uses solve units; ``measure_costs`` gives seconds).
"""
from __future__ import annotations

from dataclasses import dataclass

from .errors import UndefinedLimitError, UnfittableError


@dataclass(frozen=True)
class CostParams:
    """Inputs of the model (analysis.py:260-283): per-subinterval fine and
    coarse propagation costs, the per-sweep serialisation overhead of the
    synchronous schedule, the sync sweep count k and the async maximum
    per-worker activation count kappa."""

    p: int
    fine_cost: float
    coarse_cost: float
    overhead: float = 0.0
    k: int | None = None
    kappa: int | None = None

    def __post_init__(self):
        if self.p < 1:
            raise ValueError(f"need p >= 1, got {self.p}")
        if min(self.fine_cost, self.coarse_cost, self.overhead) < 0.0:
            raise ValueError("costs must be nonnegative")


@dataclass(frozen=True)
class SpeedupReport:
    """Best-case async/sync ratio and, when k and kappa are known, the
    achieved one (analysis.py:323-329)."""

    bound: float
    achieved: float | None


def sequential_cost(params: CostParams) -> float:
    """p fine propagations (analysis.py:286-288)."""
    return params.p * params.fine_cost


def sync_cost(params: CostParams) -> float:
    """Initialisation (p coarse) + k sweeps of fine + coarse + the cascading
    overhead (p - 1 - (k+1)/2) * overhead (analysis.py:291-309)."""
    if params.k is None:
        raise ValueError("sync cost needs k")
    k, p = params.k, params.p
    if not 0 <= k <= p:
        raise ValueError(f"k must lie in [0, p]; got k={k}, p={p}")
    init = p * params.coarse_cost
    if k == 0:
        return init
    sweep = params.fine_cost + params.coarse_cost + (p - 1 - (k + 1) / 2.0) * params.overhead
    return init + k * sweep


def async_cost(params: CostParams) -> float:
    """Initialisation + kappa fine-plus-coarse evaluations on the busiest
    worker (analysis.py:312-320)."""
    if params.kappa is None:
        raise ValueError("async cost needs kappa")
    if params.kappa < 0:
        raise ValueError(f"kappa must be >= 0, got {params.kappa}")
    return params.p * params.coarse_cost + params.kappa * (params.fine_cost + params.coarse_cost)


def speedup_bound(params: CostParams) -> SpeedupReport:
    """1 + (p-2) overhead / (fine + coarse), the sync/async ratio at k = 1,
    kappa = k; with k and kappa given, also the achieved ratio, which may not
    exceed the bound while kappa >= k (analysis.py:332-356)."""
    if params.p < 2:
        raise ValueError(f"speedup bound needs p >= 2, got p={params.p}")
    per = params.fine_cost + params.coarse_cost
    if per <= 0.0:
        raise UndefinedLimitError("fine + coarse cost must be positive")
    bound = 1.0 + (params.p - 2) * params.overhead / per
    if params.k is None or params.kappa is None:
        return SpeedupReport(bound=bound, achieved=None)
    if params.kappa < params.k:
        raise ValueError(f"kappa={params.kappa} below k={params.k}: an asynchronous run cannot use fewer "
                         "activations than the synchronous sweep count")
    achieved = sync_cost(params) / async_cost(params)
    if achieved > bound * (1.0 + 1e-12):
        raise AssertionError(f"achieved ratio {achieved} exceeds the model bound {bound}")
    return SpeedupReport(bound=bound, achieved=achieved)


def asymptotic_speedups(params: CostParams) -> tuple[float, float, float]:
    """Large-p limits at fixed k of sequential/sync, sequential/async and
    sync/async (analysis.py:359-373)."""
    if params.k is None:
        raise ValueError("asymptotic ratios need k")
    if params.coarse_cost <= 0.0:
        raise UndefinedLimitError("asymptotic ratios diverge or degenerate with zero coarse cost")
    k = params.k
    return (params.fine_cost / (params.coarse_cost + k * params.overhead),
            params.fine_cost / params.coarse_cost,
            1.0 + k * params.overhead / params.coarse_cost)


def fit_overhead(total_cost: float, p: int, k: int, fine_cost: float, coarse_cost: float) -> float:
    """Overhead coefficient that makes sync_cost reproduce ``total_cost``,
    floored at 0 (analysis.py:376-392)."""
    if k < 1:
        raise UnfittableError(f"need k >= 1 to fit the overhead, got k={k}")
    coef = k * (p - 1) - k * (k + 1) / 2.0
    if coef <= 0.0:
        raise UnfittableError(f"overhead coefficient vanishes for p={p}, k={k}; nothing to fit")
    return max((total_cost - p * coarse_cost - k * (fine_cost + coarse_cost)) / coef, 0.0)


# ------------------------------------------------------------------ B200 glue

def measure_costs(coarse, fine, p: int, reps: int = 5) -> dict:
    """Seconds per subinterval on the device, CUDA-event timed after warm-up:
    ``fine_cost`` = one F application of one slice (a worker's unit in the
    model), ``fine_batch`` = F over all p slices in one launch (the B200 sync
    sweep's actual fine phase), ``coarse_cost`` = one G application."""
    import torch

    dev = f"cuda:{fine.device}"
    x = torch.randn(p, fine.dim, dtype=fine.dtype, device=dev)
    y = torch.empty_like(x)

    def timed(fn):
        fn()
        torch.cuda.synchronize(dev)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize(dev)
        return e0.elapsed_time(e1) / reps * 1e-3

    f_one = timed(lambda: fine.apply_batch(x[:1], out=y[:1]))
    f_all = timed(lambda: fine.apply_batch(x, out=y))
    g_one = timed(lambda: coarse.apply_batch(x[:1], out=y[:1]))
    return {"fine_cost": f_one, "fine_batch": f_all, "coarse_cost": g_one}


def model_report(costs: dict, p: int, k: int | None = None, kappa: int | None = None,
                 measured_sync_s: float | None = None) -> dict:
    """Model predictions from measured costs. The B200 sync sweep runs all
    live slices' F concurrently, so its per-sweep fine term is the batch time;
    the reference model's per-worker form uses ``fine_cost``. When the
    measured sync wall time is given, the overhead is fitted to it."""
    out = {"p": p, **{key: float(v) for key, v in costs.items()}}
    base = CostParams(p=p, fine_cost=costs["fine_batch"], coarse_cost=costs["coarse_cost"])
    out["sequential_fine_s"] = sequential_cost(CostParams(p=p, fine_cost=costs["fine_cost"],
                                                          coarse_cost=costs["coarse_cost"]))
    if k is not None:
        ov = 0.0
        if measured_sync_s is not None and 1 <= k < p and k * (p - 1) - k * (k + 1) / 2.0 > 0:
            ov = fit_overhead(measured_sync_s, p, k, base.fine_cost, base.coarse_cost)
        params = CostParams(p=p, fine_cost=base.fine_cost, coarse_cost=base.coarse_cost, overhead=ov, k=k,
                            kappa=kappa)
        out.update({"k": k, "overhead_fit_s": ov, "sync_model_s": sync_cost(params)})
        if measured_sync_s is not None:
            out["sync_measured_s"] = float(measured_sync_s)
        if kappa is not None:
            out.update({"kappa": kappa, "async_model_s": async_cost(params)})
            if p >= 2 and kappa >= k:
                rep = speedup_bound(params)
                out.update({"speedup_bound": rep.bound, "speedup_model": rep.achieved})
        if base.coarse_cost > 0:
            s_sync, s_async, s_cross = asymptotic_speedups(params)
            out.update({"asymptotic_seq_over_sync": s_sync, "asymptotic_seq_over_async": s_async,
                        "asymptotic_sync_over_async": s_cross})
    return out
