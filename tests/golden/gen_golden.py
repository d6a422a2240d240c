"""Generate golden vectors by running the REFERENCE (pintlab) itself.

Run in the build container only (it needs /root/reference, which does not
exist on the GPU box):

    python tests/golden/gen_golden.py

Outputs small ``.npz`` fixtures next to this script. They are committed, so
the CPU oracle tests and the GPU parity tests read them without the
reference. Every fixture records the reference call that produced it.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = os.environ.get("PINT_REF_PATH", "/root/reference/pkg/src")
sys.path.insert(0, REF)
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import pintlab  # noqa: E402
from pintlab.async_engine import AsyncSchedule  # noqa: E402
from pintlab.model import (  # noqa: E402
    AffinePropagator,
    LinearIVP,
    backward_euler_propagator,
    fine_from_onestep,
    heat1d_system,
    scalar_decay_system,
    trapezoidal_propagator,
)

from oracle.heat_oracle import grid, modes_2d, modes_3d, sine_u0_1d, sine_u0_nd  # noqa: E402


def save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print("wrote", path, sum(a.nbytes for a in map(np.asarray, arrays.values())), "bytes")


def c1():
    """BASELINE configs[0]: 1-D heat N=1024, P=16, F=100 BE, G=1 BE, eps=1e-10."""
    n, p, T = 1024, 16, 1.0
    u0 = sine_u0_1d(n, 8, seed=0)
    ivp = LinearIVP(heat1d_system(n, 1.0, 0.0, 0.0, 0.0, T).a_mat, np.zeros(n), u0, T)
    span = T / p
    fine = pintlab.backward_euler_propagator(ivp, span, 100)
    coarse = pintlab.backward_euler_propagator(ivp, span, 1)
    tr = pintlab.run_parareal(coarse, fine, u0, p, 1e-10)
    seq = pintlab.sequential_fine_solve(fine, u0, p)
    save("c1_sync.npz", u0=u0, iterates=np.stack([it.data for it in tr.iterates]),
         deltas=np.array(tr.deltas), k_final=tr.k_final,
         stop_reason=np.array(tr.stop_reason), seq=seq.data,
         meta=np.array(json.dumps(dict(n=n, p=p, T=T, fine_steps=100, coarse_steps=1,
                                       eps=1e-10, seed=0, rule="backward-euler"))))


def fixtures():
    """Reference fixture problems (conftest.py:16-32): heat n in {4,8},
    boundaries 23, initial 30, span 0.2; F = trapezoidal 100, G = BE 1."""
    out = {}
    for n in (4, 8):
        ivp = heat1d_system(n, 1.0, 23.0, 23.0, 30.0, 0.2)
        coarse = backward_euler_propagator(ivp, 0.2, 1)
        fine = trapezoidal_propagator(ivp, 0.2, 100)
        for p in range(2, 9):
            tr = pintlab.run_parareal(coarse, fine, ivp.u0, p, 0.0)
            out[f"n{n}_p{p}_iterates"] = np.stack([it.data for it in tr.iterates])
            out[f"n{n}_p{p}_deltas"] = np.array(tr.deltas)
            tr6 = pintlab.run_parareal(coarse, fine, ivp.u0, p, 1e-6)
            out[f"n{n}_p{p}_eps6_k"] = np.array(tr6.k_final)
            out[f"n{n}_p{p}_eps6_final"] = tr6.iterates[-1].data
        out[f"n{n}_seq8"] = pintlab.sequential_fine_solve(fine, ivp.u0, 8).data
        out[f"n{n}_fine_matrix"] = fine.matrix
        out[f"n{n}_fine_offset"] = fine.offset
        out[f"n{n}_coarse_matrix"] = coarse.matrix
        out[f"n{n}_coarse_offset"] = coarse.offset
    # scalar zero-delay case (test_async_parareal.py:116-139)
    ivp = scalar_decay_system(rate=1.0, t_final=8.0)
    span = ivp.t_final / 8
    coarse = backward_euler_propagator(ivp, span, 1)
    fine = trapezoidal_propagator(ivp, span, 25)
    tr = pintlab.run_parareal(coarse, fine, ivp.u0, 8, 1e-5)
    out["scalar_iterates"] = np.stack([it.data for it in tr.iterates])
    out["scalar_k"] = np.array(tr.k_final)
    save("fixtures.npz", **out)


def one_d_layouts():
    """Single fine/coarse applications for many N (kernel layout edge cases):
    BE and trapezoidal, nonzero Dirichlet boundaries, random state."""
    out = {}
    rng = np.random.default_rng(7)
    for n in (1, 2, 3, 5, 31, 32, 33, 62, 63, 64, 65, 100, 257, 1000, 1025):
        bl, br = 1.5, -0.75
        ivp = heat1d_system(n, 1.0, bl, br, 0.0, 1.0)
        u = rng.standard_normal(n)
        for rule, fn in (("be", backward_euler_propagator), ("cn", trapezoidal_propagator)):
            for span, steps in ((0.01, 7), (0.3, 1)):
                prop = fn(ivp, span, steps)
                out[f"n{n}_{rule}_{steps}"] = prop.apply(u)
        out[f"n{n}_u"] = u
    ivp = scalar_decay_system(rate=0.7, t_final=1.0)
    for rule, fn in (("be", backward_euler_propagator), ("cn", trapezoidal_propagator)):
        out[f"scalar_{rule}"] = fn(ivp, 0.5, 5).apply(np.array([2.0]))
    save("layouts1d.npz", **out)


def kron_laplacian(shape, h):
    mats = []
    for n in shape:
        t = (np.diag(np.full(n, -2.0)) + np.diag(np.ones(n - 1), 1)
             + np.diag(np.ones(n - 1), -1))
        mats.append(t)
    lap = None
    for d, t in enumerate(mats):
        term = t
        for e, n in enumerate(shape):
            if e < d:
                term = np.kron(np.eye(n), term)
            elif e > d:
                term = np.kron(term, np.eye(n))
        lap = term if lap is None else lap + term
    return lap / (h * h)


def reduced_nd():
    """Reduced 2-D/3-D analogs of configs C3/C4 through the reference's dense
    route: F = fine_from_onestep(AffinePropagator(I + dt A, dt c, 1), S),
    G = backward_euler_propagator(ivp, span, 1)."""
    out = {}
    for tag, shape, modes, p, steps, cfl, eps in (
        ("2d", (12, 12), modes_2d(), 8, 50, 0.2, 1e-10),
        ("3d", (6, 6, 6), modes_3d(), 6, 20, 0.15, 1e-9),
    ):
        n = shape[0]
        h = 1.0 / (n + 1)
        dt = cfl * h * h
        span = steps * dt
        a = kron_laplacian(shape, h)
        dim = a.shape[0]
        u0 = sine_u0_nd(shape, modes, seed=0).reshape(-1)
        ivp = LinearIVP(a, np.zeros(dim), u0, p * span)
        one = AffinePropagator(np.eye(dim) + dt * a, dt * np.zeros(dim), 1.0)
        fine = fine_from_onestep(one, steps)
        coarse = backward_euler_propagator(ivp, span, 1)
        tr = pintlab.run_parareal(coarse, fine, u0, p, eps)
        out[f"{tag}_iterates"] = np.stack([it.data for it in tr.iterates])
        out[f"{tag}_deltas"] = np.array(tr.deltas)
        out[f"{tag}_k"] = np.array(tr.k_final)
        out[f"{tag}_stop"] = np.array(tr.stop_reason)
        out[f"{tag}_seq"] = pintlab.sequential_fine_solve(fine, u0, p).data
        out[f"{tag}_meta"] = np.array(json.dumps(dict(shape=shape, p=p, steps=steps,
                                                      cfl=cfl, eps=eps, h=h, dt=dt)))
    save("reduced_nd.npz", **out)


def async_traces():
    """Async event traces of the reference (heat n=4 fixture and scalar)."""
    out = {}
    ivp = heat1d_system(4, 1.0, 23.0, 23.0, 30.0, 0.2)
    coarse = backward_euler_propagator(ivp, 0.2, 1)
    fine = trapezoidal_propagator(ivp, 0.2, 100)
    cases = [
        ("rf_s5_d1_p6", 6, AsyncSchedule(seed=5, delay_bound=1), None),
        ("rf_s9_d2_p6", 6, AsyncSchedule(seed=9, delay_bound=2), None),
        ("adv_s3_d2_p5", 5, AsyncSchedule(seed=3, delay_bound=2, policy="adversarial-stale"), None),
        ("rr_s0_d0_p6_eps", 6, AsyncSchedule(seed=0, delay_bound=0, policy="round-robin"), 1e-6),
        ("rf_s4_d3_p7_eps", 7, AsyncSchedule(seed=4, delay_bound=3), 1e-6),
    ]
    for tag, p, sched, eps in cases:
        tr = pintlab.run_async_parareal(coarse, fine, ivp.u0, p, sched, epsilon=eps)
        out[f"{tag}_components"] = np.array([e.component for e in tr.events])
        out[f"{tag}_reads"] = np.array([[r[2] for r in e.reads] for e in tr.events])
        out[f"{tag}_deltas"] = np.array([e.delta for e in tr.events])
        out[f"{tag}_final"] = tr.state_after(len(tr.events) - 1).data
        out[f"{tag}_counts"] = np.asarray(tr.per_component_counts)
        out[f"{tag}_stop"] = np.array(tr.stop_reason)
        out[f"{tag}_sched"] = np.array(json.dumps(sched.to_dict() | {"p": p, "eps": eps}))
    save("async_traces.npz", **out)


def contraction():
    """pintlab.analysis.contraction_factors (analysis.py:92-98, spectral norm
    by Gram power iteration) on the C1 propagators, a trapezoidal/BE pair
    and a reduced 2-D explicit/implicit pair."""
    from pintlab.analysis import contraction_factors
    from pintlab.linalg import NormKind
    out = {}
    cases = []
    n, p, T = 1024, 16, 1.0
    ivp = LinearIVP(heat1d_system(n, 1.0, 0.0, 0.0, 0.0, T).a_mat, np.zeros(n), np.zeros(n), T)
    cases.append(("c1", ivp, backward_euler_propagator(ivp, T / p, 100), backward_euler_propagator(ivp, T / p, 1),
                  p, dict(shape=[n], fine=["backward-euler", T / p / 100, 100], coarse=["backward-euler", T / p, 1])))
    n, p = 64, 8
    ivp = LinearIVP(heat1d_system(n, 1.0, 0.0, 0.0, 0.0, T).a_mat, np.zeros(n), np.zeros(n), T)
    cases.append(("cn64", ivp, trapezoidal_propagator(ivp, T / p, 50), backward_euler_propagator(ivp, T / p, 1),
                  p, dict(shape=[n], fine=["trapezoidal", T / p / 50, 50], coarse=["backward-euler", T / p, 1])))
    n, p, steps = 12, 8, 40
    h = 1.0 / (n + 1)
    dt = 0.2 * h * h
    a = kron_laplacian((n, n), h)
    ivp2 = LinearIVP(a, np.zeros(n * n), np.zeros(n * n), p * steps * dt)
    one = AffinePropagator(np.eye(n * n) + dt * a, np.zeros(n * n), 1.0)
    cases.append(("fe2d", ivp2, fine_from_onestep(one, steps), backward_euler_propagator(ivp2, steps * dt, 1),
                  p, dict(shape=[n, n], fine=["forward-euler", dt, steps],
                          coarse=["backward-euler", steps * dt, 1])))
    for tag, _, fine, coarse, pp, meta in cases:
        for kind in (NormKind.SPECTRAL, NormKind.INFINITY):
            r = contraction_factors(coarse, fine, pp, kind=kind)
            out[f"{tag}_{kind.value}"] = np.array([r.coarse_norm, r.defect_norm, r.sync_factor, r.async_factor])
        out[f"{tag}_meta"] = np.array(json.dumps(meta | {"p": pp, "length": 1.0}))
    save("contraction.npz", **out)


if __name__ == "__main__":
    contraction()
    c1()
    fixtures()
    one_d_layouts()
    reduced_nd()
    async_traces()
