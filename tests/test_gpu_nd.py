"""GPU parity of the 2-D/3-D explicit stencil (fine) and CG implicit (coarse)
propagators and of synchronous Parareal on the reduced C3/C4 analogs, against
golden vectors from the reference's dense route and the numpy oracle."""
import json

import numpy as np
import pytest

from conftest import golden, rel_l2
from oracle import heat_oracle as H

pytestmark = pytest.mark.gpu


def _setup(gpu, tag, dtype="float64", cg_rtol=None):
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
    kw = {} if cg_rtol is None else {"cg_rtol": cg_rtol}
    coarse = gpu.backward_euler_propagator(ivp, span, 1, dtype=dtype, **kw)
    return g, meta, ivp, fine, coarse, u0


@pytest.mark.parametrize("tag", ("2d", "3d"))
def test_reduced_nd_sync_parareal_matches_reference(gpu, tag):
    g, meta, ivp, fine, coarse, u0 = _setup(gpu, tag)
    tr = gpu.run_parareal(coarse, fine, u0, meta["p"], meta["eps"])
    assert tr.k_final == int(g[f"{tag}_k"])
    assert tr.stop_reason == str(g[f"{tag}_stop"])
    for k, it in enumerate(tr.iterates):
        assert rel_l2(it.data, g[f"{tag}_iterates"][k]) < 1e-11, k
    seq = gpu.sequential_fine_solve(fine, u0, meta["p"])
    assert rel_l2(seq.data, g[f"{tag}_seq"]) < 1e-11


@pytest.mark.parametrize("tag", ("2d", "3d"))
def test_reduced_nd_fp32_within_1e5(gpu, tag):
    g, meta, ivp, fine, coarse, u0 = _setup(gpu, tag, dtype="float32")
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


@pytest.mark.parametrize("shape", [(64, 64), (20, 20, 20)])
def test_cg_coarse_matches_direct_solve(gpu, shape):
    n = shape[0]
    h = 1.0 / (n + 1)
    dT = 50 * h * h
    rng = np.random.default_rng(5)
    u = rng.standard_normal(int(np.prod(shape)))
    mk = gpu.heat2d_system if len(shape) == 2 else gpu.heat3d_system
    ivp = mk(n, t_final=1.0, u0=u)
    G = gpu.backward_euler_propagator(ivp, dT, 1)
    got = G.apply(u)
    want = H.ImplicitND(shape, h, dT, direct=True).apply(u)
    assert rel_l2(got, want) < 1e-11
    G32 = gpu.backward_euler_propagator(ivp, dT, 1, dtype="float32", cg_rtol=1e-6)
    assert rel_l2(G32.apply(u), want) < 1e-5
    # deterministic: same input bits -> same output bits
    assert np.array_equal(G.apply(u), got)


def test_cg_reports_nonconvergence(gpu):
    n = 32
    ivp = gpu.heat2d_system(n, t_final=1.0, u0=np.ones(n * n))
    G = gpu.backward_euler_propagator(ivp, 1.0, 1, cg_rtol=1e-14, cg_maxit=3)
    with pytest.raises(gpu.ConvergenceFailure) as err:
        G.apply(np.ones(n * n))
    assert err.value.estimate > 0
