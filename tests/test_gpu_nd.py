"""GPU parity of the 2-D/3-D explicit stencil (fine) and implicit (coarse:
direct sine-transform solve, and CG) propagators and of synchronous Parareal on the reduced C3/C4 analogs, against
golden vectors from the reference's dense route and the numpy oracle."""
import json

import numpy as np
import pytest

from conftest import golden, rel_l2
from oracle import heat_oracle as H

pytestmark = pytest.mark.gpu


def _setup(gpu, tag, dtype="float64", cg_rtol=None, solver="direct"):
    g = golden("reduced_nd.npz")
    meta = json.loads(str(g[f"{tag}_meta"]))
    shape = tuple(meta["shape"])
    n = shape[0]
    u0 = g[f"{tag}_iterates"][0][0]
    p = meta["p"]
    span = meta["steps"] * meta["dt"]
    mk = gpu.heat2d_system if len(shape) == 2 else gpu.heat3d_system
    ivp = mk(n, t_final=p * span, u0=u0)
    fine = gpu.forward_euler_propagator(ivp, span, meta["steps"], dtype=dtype)
    kw = {"solver": solver} if cg_rtol is None else {"cg_rtol": cg_rtol, "solver": solver}
    coarse = gpu.backward_euler_propagator(ivp, span, 1, dtype=dtype, **kw)
    return g, meta, ivp, fine, coarse, u0


@pytest.mark.parametrize("solver", ("direct", "cg"))
@pytest.mark.parametrize("tag", ("2d", "3d"))
def test_reduced_nd_sync_parareal_matches_reference(gpu, tag, solver):
    g, meta, ivp, fine, coarse, u0 = _setup(gpu, tag, solver=solver)
    tr = gpu.run_parareal(coarse, fine, u0, meta["p"], meta["eps"])
    assert tr.k_final == int(g[f"{tag}_k"])
    assert tr.stop_reason == str(g[f"{tag}_stop"])
    for k, it in enumerate(tr.iterates):
        assert rel_l2(it.data, g[f"{tag}_iterates"][k]) < 1e-11, k
    seq = gpu.sequential_fine_solve(fine, u0, meta["p"])
    assert rel_l2(seq.data, g[f"{tag}_seq"]) < 1e-11


@pytest.mark.parametrize("solver", ("direct", "cg"))
@pytest.mark.parametrize("tag", ("2d", "3d"))
def test_reduced_nd_fp32_within_1e5(gpu, tag, solver):
    g, meta, ivp, fine, coarse, u0 = _setup(gpu, tag, dtype="float32", solver=solver)
    tr = gpu.run_parareal(coarse, fine, u0, meta["p"], 1e-6)
    ref = g[f"{tag}_seq"]
    assert rel_l2(tr.final.data, ref) < 1e-5


@pytest.mark.parametrize("shape,steps,cfl", [((1024, 1024), 40, 0.2), ((96, 96, 96), 30, 0.15),
                                             ((37, 37), 17, 0.2), ((9, 9, 9), 5, 0.1)])
def test_explicit_stencil_matches_oracle(gpu, shape, steps, cfl):
    import torch
    n = shape[0]
    h = 1.0 / (n + 1)
    dt = cfl * h * h
    rng = np.random.default_rng(11)
    u = rng.standard_normal(int(np.prod(shape)))
    if len(set(shape)) != 1:
        pytest.skip("HeatIVP requires equal spacing; covered by the square cases")
    mk = gpu.heat2d_system if len(shape) == 2 else gpu.heat3d_system
    ivp = mk(n, t_final=1.0, u0=u)
    for dtype, tol in (("float64", 1e-13), ("float32", 2e-6)):
        fine = gpu.forward_euler_propagator(ivp, steps * dt, steps, dtype=dtype)
        got = fine.apply(u)
        want = H.ExplicitND(shape, h, dt, steps).apply(u)
        assert rel_l2(got, want) < tol, (dtype, rel_l2(got, want))
        # batch == single, bitwise
        xs = torch.tensor(np.stack([u, 2 * u, -u]), device="cuda", dtype=fine.dtype)
        out = fine.apply_batch(xs)
        assert torch.equal(out[0], fine.apply(xs[0]))


@pytest.mark.parametrize("solver,tol", [("direct", 1e-13), ("cg", 1e-11)])
@pytest.mark.parametrize("shape,steps", [((64, 64), 1), ((20, 20, 20), 1), ((37, 37), 3), ((9, 9, 9), 2),
                                         ((1, 1), 1), ((2, 2, 2), 1), ((130, 130), 1)])
def test_implicit_coarse_matches_sparse_lu(gpu, shape, steps, solver, tol):
    n = shape[0]
    h = 1.0 / (n + 1)
    dT = 50 * h * h
    rng = np.random.default_rng(5)
    u = rng.standard_normal(int(np.prod(shape)))
    mk = gpu.heat2d_system if len(shape) == 2 else gpu.heat3d_system
    ivp = mk(n, t_final=1.0, u0=u)
    G = gpu.backward_euler_propagator(ivp, steps * dT, steps, solver=solver)
    got = G.apply(u)
    want = u
    for _ in range(steps):
        want = H.ImplicitND(shape, h, dT, direct=True).apply(want)
    assert rel_l2(got, want) < tol, rel_l2(got, want)
    G32 = gpu.backward_euler_propagator(ivp, steps * dT, steps, dtype="float32", cg_rtol=1e-6, solver=solver)
    assert rel_l2(G32.apply(u), want) < 1e-5
    # deterministic: same input bits -> same output bits; batch == single
    assert np.array_equal(G.apply(u), got)
    import torch
    xs = torch.tensor(np.stack([u, -2 * u]), device="cuda", dtype=torch.float64)
    out = G.apply_batch(xs)
    assert torch.equal(out[0], G.apply(xs[0]))


@pytest.mark.parametrize("shape,dtype,tol", [((1024, 1024), "float64", 4e-15), ((1024, 1024), "float32", 2e-6),
                                             ((256, 256, 256), "float32", 2e-6), ((128, 128, 128), "float64", 4e-15)])
def test_direct_coarse_residual_at_config_size(gpu, shape, dtype, tol):
    """Size-independent check at the C3/C4 shapes: the normwise backward
    error ||b - A x|| / (||A|| ||x|| + ||b||) of A x = b, A = I - dT Lap_h
    (||A||_2 < 1 + 4 d c), evaluated in fp64 on the device. A backward-stable
    solve keeps it at a small multiple of the working precision."""
    import torch
    n = shape[0]
    h = 1.0 / (n + 1)
    dT = (100 if len(shape) == 2 else 30) * h * h
    u = H.sine_u0_nd(shape, H.modes_2d() if len(shape) == 2 else H.modes_3d(), 0).reshape(-1)
    u = u + 1e-3 * np.random.default_rng(3).standard_normal(u.size)
    mk = gpu.heat2d_system if len(shape) == 2 else gpu.heat3d_system
    ivp = mk(n, t_final=1.0, u0=u)
    G = gpu.backward_euler_propagator(ivp, dT, 1, dtype=dtype)
    b = torch.tensor(u, device="cuda", dtype=G.dtype)
    x = G.apply_batch(b.reshape(1, -1))[0].double().reshape(shape)
    bd = b.double().reshape(shape)
    c = dT / (h * h)
    lap = -2 * len(shape) * x
    for ax in range(len(shape)):
        lap = lap + torch.roll(x, 1, ax) + torch.roll(x, -1, ax)
        # zero Dirichlet: undo the wrap-around
        idx0 = [slice(None)] * len(shape)
        idx0[ax] = 0
        idxl = [slice(None)] * len(shape)
        idxl[ax] = n - 1
        lap[tuple(idx0)] -= x[tuple(idxl)]
        lap[tuple(idxl)] -= x[tuple(idx0)]
    anorm = 1 + 4 * len(shape) * c
    res = (x - c * lap - bd).norm() / (anorm * x.norm() + bd.norm())
    print(f"backward error {shape} {dtype}: {res.item():.3e}")
    assert res.item() < tol, res.item()


def test_cg_reports_nonconvergence(gpu):
    n = 32
    ivp = gpu.heat2d_system(n, t_final=1.0, u0=np.ones(n * n))
    G = gpu.backward_euler_propagator(ivp, 1.0, 1, cg_rtol=1e-14, cg_maxit=3, solver="cg")
    with pytest.raises(gpu.ConvergenceFailure) as err:
        G.apply(np.ones(n * n))
    assert err.value.estimate > 0


def test_unknown_nd_solver_rejected(gpu):
    ivp = gpu.heat2d_system(8, t_final=1.0, u0=np.ones(64))
    with pytest.raises(ValueError):
        gpu.backward_euler_propagator(ivp, 0.1, 1, solver="lu")


@pytest.mark.parametrize("dtype,variants", [("float32", range(0, 12)), ("float64", range(0, 8))])
@pytest.mark.parametrize("shape,steps", [((37, 37, 37), 7), ((19, 19, 19), 13), ((64, 64, 64), 5)])
def test_fe3d_tilings_are_bitwise_identical(gpu, monkeypatch, dtype, variants, shape, steps):
    """Every 3-D tiling (stencil3d.cu variants, fe3d_wave = 0) evaluates the
    same per-point expression, so all give identical bits, on ragged grids
    with partial tiles, z chunks and remainder passes; and the default one
    matches the oracle."""
    import torch
    from oracle import heat_oracle as H
    n = shape[0]
    ivp = gpu.heat3d_system(n, t_final=1.0)
    h = 1.0 / (n + 1)
    x = torch.rand(3, ivp.dim, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(5))
    outs = {}
    for v in variants:
        monkeypatch.setenv("PINT_FE3D_VARIANT", str(v))
        F = gpu.forward_euler_propagator(ivp, steps * 0.15 * h * h, steps, dtype=dtype)
        y = F.apply_batch(x.to(F.dtype))
        outs[v] = y.clone()
    for v in variants:
        assert torch.equal(outs[v], outs[0]), v
    monkeypatch.delenv("PINT_FE3D_VARIANT")
    F = gpu.forward_euler_propagator(ivp, steps * 0.15 * h * h, steps, dtype=dtype)
    y = F.apply_batch(x.to(F.dtype)).double().cpu().numpy()
    ref = H.ExplicitND(shape, h, 0.15 * h * h, steps).apply(x[0].cpu().numpy())
    tol = 1e-5 if dtype == "float32" else 1e-12
    assert np.max(np.abs(y[0] - ref)) <= tol * max(1.0, np.max(np.abs(ref)))


@pytest.mark.parametrize("dtype", ["float32", "float64"])
@pytest.mark.parametrize("shape,steps", [((300, 300), 29), ((41, 57), 9), ((1024, 1024), 12)])
def test_fe2d_variants_are_bitwise_identical(gpu, monkeypatch, dtype, shape, steps):
    """The 2-D wavefront variants (rolled / six-row unrolled steady state)
    give identical bits, and match the oracle."""
    import torch
    n = shape[0]
    if shape[0] != shape[1]:
        pytest.skip("square grids only")
    ivp = gpu.heat2d_system(n, t_final=1.0)
    h = 1.0 / (n + 1)
    x = torch.rand(3, ivp.dim, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(2))
    outs = []
    for v in (0, 1, 2):
        monkeypatch.setenv("PINT_FE2D_VARIANT", str(v))
        F = gpu.forward_euler_propagator(ivp, steps * 0.2 * h * h, steps, dtype=dtype)
        outs.append(F.apply_batch(x.to(F.dtype)).clone())
    assert all(torch.equal(o, outs[0]) for o in outs)
    ref = H.ExplicitND(shape, h, 0.2 * h * h, steps).apply(x[1].cpu().numpy())
    tol = 1e-5 if dtype == "float32" else 1e-12
    assert np.max(np.abs(outs[0][1].double().cpu().numpy() - ref)) <= tol * max(1.0, np.max(np.abs(ref)))


@pytest.mark.parametrize("shape,p,chunk", [((40, 40), 9, 4), ((16, 16, 16), 7, 3), ((33, 33), 5, 1)])
def test_lean_engine_is_bitwise_the_standard_engine(gpu, shape, p, chunk):
    """The in-place engine (2 state copies, for states that fill HBM) gives
    the same iterates, deltas, k and stop reason as the standard engine."""
    from paper_2110_10762_b200 import inputs
    from paper_2110_10762_b200.parareal import LeanSyncEngine
    import paper_2110_10762_b200.parareal as par
    n = shape[0]
    h = 1.0 / (n + 1)
    span = 20 * 0.15 * h * h
    u0 = inputs.sine_u0(shape, seed=2)
    mk = gpu.heat2d_system if len(shape) == 2 else gpu.heat3d_system
    ivp = mk(n, t_final=p * span, u0=u0)
    fine = gpu.forward_euler_propagator(ivp, span, 20)
    coarse = gpu.backward_euler_propagator(ivp, span, 1)
    std = gpu.run_parareal(coarse, fine, u0, p, 0.0, record_iterates=True)
    orig = par.LeanSyncEngine.__init__

    def init(self, c, f, pp, chunk_=chunk):
        orig(self, c, f, pp, chunk=chunk_)
    par.LeanSyncEngine.__init__ = init
    try:
        lean = gpu.run_parareal(coarse, fine, u0, p, 0.0, record_iterates=True, engine="lean")
    finally:
        par.LeanSyncEngine.__init__ = orig
    assert lean.k_final == std.k_final == p and lean.stop_reason == std.stop_reason
    assert lean.deltas == std.deltas
    for a, b in zip(lean.iterates, std.iterates):
        assert np.array_equal(a.data, b.data)
    assert np.array_equal(lean.final.data, gpu.sequential_fine_solve(fine, u0, p).data)
