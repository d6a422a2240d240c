"""CPU checks of the config-size oracle pieces (oracle/nd_truth.py,
oracle/stencil_nd.c, the threaded long-double Thomas) before they are trusted
as the checker of the device at the BASELINE shapes."""
import numpy as np
import pytest

from conftest import golden, rel_l2
from oracle import heat_oracle as H
from oracle.nd_truth import SpectralND, StencilND
from oracle.truth import TruthTridiag1D


@pytest.mark.parametrize("shape,steps,cfl", [((37, 37), 17, 0.2), ((9, 10, 11), 5, 0.15), ((50,), 7, 0.4),
                                             ((1, 1), 3, 0.2), ((2, 2, 2), 2, 0.1)])
def test_stencil_matches_numpy_restatement(shape, steps, cfl):
    n = shape[0]
    h = 1.0 / (n + 1)
    span = steps * cfl * h * h
    u = np.random.default_rng(1).standard_normal(int(np.prod(shape)))
    got = StencilND(shape, h, span, steps).apply(u)
    want = H.ExplicitND(shape, h, span / steps, steps).apply(u)
    assert rel_l2(got, want) < 1e-15
    ld = StencilND(shape, h, span, steps, exact=True).apply(u)
    assert rel_l2(got, ld) < 1e-15
    f32 = StencilND(shape, h, span, steps, dtype=np.float32).apply(u.astype(np.float32))
    assert f32.dtype == np.float32 and rel_l2(f32, want) < 1e-6


def test_stencil_batch_equals_single_and_is_deterministic():
    shape = (33, 34, 35)
    h = 1.0 / 34
    st = StencilND(shape, h, 3 * 0.15 * h * h, 3)
    xs = np.random.default_rng(2).standard_normal((3, int(np.prod(shape))))
    b = st.apply_batch(xs)
    for i in range(3):
        assert np.array_equal(b[i], st.apply(xs[i]))
    assert np.array_equal(b, st.apply_batch(xs))


def test_stencil_reproduces_reference_dense_route():
    """Against the reference's own dense FE route on the reduced 2-D/3-D
    analogs (tests/golden/reduced_nd.npz: sequential fine solutions built by
    pintlab's fine_from_onestep(AffinePropagator(I + dt A, ...)))."""
    import json
    g = golden("reduced_nd.npz")
    for tag in ("2d", "3d"):
        meta = json.loads(str(g[f"{tag}_meta"]))
        shape = tuple(meta["shape"])
        h = 1.0 / (shape[0] + 1)
        F = StencilND(shape, h, meta["steps"] * meta["dt"], meta["steps"])
        seq = H.sequential_fine_solve(F, g[f"{tag}_iterates"][0][0], meta["p"])
        assert rel_l2(seq, g[f"{tag}_seq"]) < 1e-12, tag


@pytest.mark.parametrize("shape,steps", [((20, 20), 1), ((8, 8, 8), 1), ((13, 13), 2), ((1, 1), 1)])
def test_spectral_solve_matches_sparse_lu(shape, steps):
    n = shape[0]
    h = 1.0 / (n + 1)
    dT = 50 * h * h
    u = np.random.default_rng(4).standard_normal(int(np.prod(shape)))
    got = SpectralND(shape, h, steps * dT, steps).apply(u)
    want = u
    for _ in range(steps):
        want = H.ImplicitND(shape, h, dT, direct=True).apply(want)
    assert rel_l2(got, want) < 1e-14


def test_threaded_long_double_thomas_batch_equals_single():
    n = 1000
    a_d, a_o, c = H.heat1d_coeffs(n)
    F = TruthTridiag1D(n, a_d, a_o, c, 1 / 16, 20)
    xs = np.random.default_rng(3).standard_normal((9, n))
    b = F.apply_batch(xs)
    for i in range(9):
        assert np.array_equal(b[i], F.apply(xs[i]))
