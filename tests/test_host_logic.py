"""Host-side logic on CPU (no GPU): problem builders and validation, operator
structure detection, schedules and audits, error mapping, and the exact
solver plan of the 1-D kernels (emulated in numpy from the C++ plan)."""
import numpy as np
import pytest

import paper_2110_10762_b200 as pb
from paper_2110_10762_b200 import _native
from paper_2110_10762_b200.async_engine import ScheduleDriver
from paper_2110_10762_b200.model import _tridiag_structure
from oracle import heat_oracle as H


def test_heat1d_system_matches_reference_structure():
    ivp = pb.heat1d_system(1, 1.0, 23.0, 23.0, 30.0, 0.2)
    assert ivp.a_mat.shape == (1, 1) and ivp.a_mat[0, 0] == -8.0
    assert ivp.forcing[0] == 4.0 * (23.0 + 23.0)
    assert np.array_equal(ivp.u0, [30.0])
    a_d, a_o, c0, c1 = ivp.coefficients_1d()
    assert a_d == -8.0 and c0 == 184.0
    ivp = pb.heat1d_system(6, 1.0, 23.0, 23.0, 23.0, 0.2)
    assert np.allclose(ivp.a_mat @ ivp.u0 + ivp.forcing, 0.0, atol=1e-10)
    with pytest.raises(pb.DegenerateProblemError):
        pb.heat1d_system(0, 1.0, 0.0, 0.0, 0.0, 1.0)


def test_linear_ivp_validation_and_structure_detection():
    with pytest.raises(pb.DimensionError):
        pb.LinearIVP(np.ones((2, 3)), np.zeros(2), np.zeros(2), 1.0)
    with pytest.raises(pb.DimensionError):
        pb.LinearIVP(np.eye(2), np.zeros(3), np.zeros(2), 1.0)
    with pytest.raises(ValueError):
        pb.LinearIVP(np.eye(2), np.zeros(2), np.zeros(2), 0.0)
    heat = pb.heat1d_system(5, 1.0, 1.0, 2.0, 0.0, 1.0)
    dense = pb.LinearIVP(heat.a_mat, heat.forcing, heat.u0, 1.0)
    assert _tridiag_structure(dense) == heat.coefficients_1d()
    assert _tridiag_structure(pb.scalar_decay_system(0.5)) == (-0.5, 0.0, 0.0, 0.0)
    rng = np.random.default_rng(0)
    assert _tridiag_structure(pb.LinearIVP(rng.normal(size=(3, 3)), np.zeros(3), np.zeros(3), 1.0)) is None
    back = pb.LinearIVP.from_dict(dense.to_dict())
    assert np.array_equal(back.a_mat, dense.a_mat)
    h2 = pb.heat2d_system(4, 1.0, u0=np.arange(16.0))
    assert pb.HeatIVP.from_dict(h2.to_dict()).shape == (4, 4)
    assert h2.a_mat.shape == (16, 16) and np.allclose(h2.a_mat, h2.a_mat.T)


def test_time_decomposition():
    td = pb.TimeDecomposition(p=4, coarse_dt=0.2, fine_dt=0.05)
    assert td.fine_steps == 4 and td.t_final == pytest.approx(0.8)
    assert pb.TimeDecomposition.from_dict(td.to_dict()) == td
    with pytest.raises(ValueError):
        pb.TimeDecomposition(p=4, coarse_dt=0.2, fine_dt=0.07)


def test_registry_is_a_superset_of_the_reference():
    assert {"backward-euler", "trapezoidal"} <= set(pb.PROPAGATOR_RULES)
    assert set(pb.PROPAGATOR_RULES) == {"backward-euler", "trapezoidal", "forward-euler"}


@pytest.mark.parametrize("policy", pb.POLICIES)
@pytest.mark.parametrize("bound", [0, 1, 3])
def test_schedule_driver_is_the_oracle_schedule(policy, bound):
    s = pb.AsyncSchedule(seed=13, delay_bound=bound, policy=policy)
    a = ScheduleDriver(s, 6)
    b = H.ScheduleDriver(13, bound, policy, 6)
    for k in range(300):
        assert a.next_component(k) == b.next_component(k)
        assert a.sample_staleness() == b.sample_staleness()


def test_schedule_validation_and_round_trip():
    sched = pb.AsyncSchedule(seed=5, delay_bound=2, policy=pb.POLICY_ROUND_ROBIN)
    assert sched.window(4) == 12
    assert pb.AsyncSchedule.from_dict(sched.to_dict()) == sched
    for bad in ({"delay_bound": -1}, {"delay_bound": 0, "policy": "eager"}, {"delay_bound": 0, "max_events": 0}):
        with pytest.raises(ValueError):
            pb.AsyncSchedule(seed=1, **bad)


def _trace(events, p, sched):
    return pb.AsyncTrace(events=events, snapshots=[], initial=None, per_component_counts=np.zeros(p + 1, int),
                         stop_event=len(events) - 1, stop_reason="x", schedule=sched, n_updatable=p,
                         persistent_slots={2: 1})


def test_validate_schedule_flags_violations():
    s = pb.AsyncSchedule(seed=0, delay_bound=0)
    ok = [pb.UpdateRecord(0, 1, ((0, 1, 0), (0, 2, 0)), "", 0.0),
          pb.UpdateRecord(1, 2, ((1, 1, 1), (1, 2, 0)), "", 0.0)]
    assert pb.validate_schedule(_trace(ok, 2, s)).ok
    # component 2 never fires in a window of 2 -> fairness; stale read -> staleness
    bad = [pb.UpdateRecord(0, 1, ((0, 1, 0), (0, 2, 0)), "", 0.0),
           pb.UpdateRecord(1, 1, ((0, 1, 0), (0, 2, 5)), "", 0.0)]
    rep = pb.validate_schedule(_trace(bad, 2, s))
    assert rep.fairness_violations and rep.provenance_violations and not rep.ok


def test_async_stop_check_edges():
    assert pb.async_stop_check([1e-7, 2e-7], epsilon=1e-6, drained=True)
    assert not pb.async_stop_check([1e-6, 2e-7], epsilon=1e-6, drained=True)
    assert not pb.async_stop_check([1e-9], epsilon=1e-6, drained=False)
    with pytest.raises(ValueError):
        pb.async_stop_check([0.0], epsilon=0.0, drained=True)


def test_status_codes_map_to_the_reference_exceptions():
    cases = {_native.PINT_EDIM: pb.DimensionError, _native.PINT_EARG: ValueError,
             _native.PINT_ENONFINITE: ValueError, _native.PINT_ENOCONV: pb.ConvergenceFailure,
             _native.PINT_EUNSUPPORTED: NotImplementedError, _native.PINT_ECUDA: RuntimeError}
    for rc, exc in cases.items():
        with pytest.raises(exc):
            _native.check(rc, None, "probe")


# ----------------------------------------------------- exact solver plan (CPU)
@pytest.mark.parametrize("n", [1, 2, 5, 31, 32, 33, 63, 64, 100, 1000, 2047, 4096, 65536])
@pytest.mark.parametrize("r", [0.5, 656.6, 6.7e7])
def test_partitioned_plan_solves_the_step_system(n, r):
    """One emulated kernel step (numpy, plan exported by the C++ host code)
    solves (I - dt A) x = d for the heat operator to fp64 accuracy."""
    import tri1d_emulator as EM
    h = 1.0 / (n + 1)
    inv_h2 = 1.0 / (h * h)
    dt = r / inv_h2
    P = EM.export_plan(n, -2.0 * inv_h2, inv_h2, 0.0, 0.0, dt, 1)
    d = np.random.default_rng(n).standard_normal(n)
    x = EM.step(d, P)
    D, E = P["D"], P["E"]
    res = D * x
    res[1:] += E * x[:-1]
    res[:-1] += E * x[1:]
    scale = abs(D) * np.abs(x).max() + np.abs(d).max()
    assert np.max(np.abs(res - d)) / scale < 1e-14


def test_plan_reports_singular_steps():
    from paper_2110_10762_b200 import _native as nat
    import ctypes
    d = nat.OpDesc()
    d.ndim, d.rule, d.dtype = 1, 0, nat.PINT_F64
    d.shape[0] = 1
    d.span, d.steps, d.a_diag = 1.0, 1, 1.0  # u' = u, dt = 1: 1 - dt*a = 0
    dims = (ctypes.c_int32 * 6)()
    assert nat.load_library().pint_tri1d_plan_host(ctypes.byref(d), dims, None, None, None) == nat.PINT_ESINGULAR


def test_package_inputs_match_the_oracle_bitwise():
    """bench.py and the CLI build their seeded inputs with the package
    (paper_2110_10762_b200/inputs.py), never with oracle/; both must give the
    same bits as the oracle's generators."""
    import numpy as np

    from oracle import heat_oracle as H
    from paper_2110_10762_b200 import inputs as I
    for n, m, seed in [(1024, 8, 0), (65536, 32, 0), (7, 3, 4)]:
        assert np.array_equal(I.sine_u0_1d(n, m, seed), H.sine_u0_1d(n, m, seed))
    assert I.modes_2d() == H.modes_2d() and I.modes_3d() == H.modes_3d()
    for shape in [(24, 24), (9, 10, 11)]:
        modes = I.modes_2d() if len(shape) == 2 else I.modes_3d()
        assert np.array_equal(I.sine_u0_nd(shape, modes, 2), H.sine_u0_nd(shape, modes, 2))
        assert np.array_equal(I.sine_u0(shape, seed=2), H.sine_u0_nd(shape, modes, 2).reshape(-1))


def test_async_mapping_validation():
    """reference async_engine.py:98-120."""
    from paper_2110_10762_b200.async_engine import AsyncMapping
    ok = AsyncMapping(2, 2, None, {1: ((0, 1), (0, 2)), 2: ((1, 1), (1, 2))}, {2: 1})
    assert ok.n_updatable == 2
    with pytest.raises(ValueError):
        AsyncMapping(0, 1, None, {})
    with pytest.raises(ValueError):
        AsyncMapping(2, 1, None, {1: ((0, 1),)})
    with pytest.raises(pb.DimensionError):
        AsyncMapping(1, 1, None, {1: ((5, 1),)})
    with pytest.raises(pb.DimensionError):
        AsyncMapping(1, 1, None, {1: ((0, 2),)})
    with pytest.raises(ValueError):
        AsyncMapping(1, 3, None, {1: ((0, 1), (0, 2), (0, 3))}, {2: 1, 3: 2})
    with pytest.raises(ValueError):
        AsyncMapping(2, 2, None, {1: ((0, 1), (0, 2)), 2: ((1, 1), (0, 2))}, {2: 1})


def test_simulate_async_needs_the_parareal_mapping():
    from paper_2110_10762_b200.async_engine import AsyncMapping
    m = AsyncMapping(1, 1, lambda i, r: r[(0, 1)], {1: ((0, 1),)})
    with pytest.raises(NotImplementedError):
        pb.simulate_async(m, np.zeros((2, 3)), pb.AsyncSchedule(seed=0, delay_bound=0))


def test_fast_path_factors_and_dispatch():
    """The backward-Euler fast path (constant-coefficient twisted chunk solve,
    csrc/tri1d.cu): closed-form factors satisfy their defining identities and
    the dispatch falls back to the exact-pivot path where the scheme does not
    apply (ragged N, boundary forcing, dt far beyond the slowest mode)."""
    import ctypes

    from paper_2110_10762_b200 import _native as nat
    lib = nat.load_library()

    def query(n, r, c_first=0.0):
        h = 1.0 / (n + 1)
        d = nat.OpDesc()
        d.ndim, d.rule, d.dtype = 1, 0, nat.PINT_F64
        d.shape[0] = n
        d.span, d.steps = r * h * h, 1
        d.a_diag, d.a_off, d.c_first, d.c_last = -2.0 / (h * h), 1.0 / (h * h), c_first, 0.0
        usable = ctypes.c_int32(-1)
        fac = np.zeros(11 + 3 * 16)
        rc = lib.pint_tri1d_ccst_host(ctypes.byref(d), ctypes.byref(usable), fac.ctypes.data_as(ctypes.c_void_p))
        assert rc == 0
        return usable.value, fac

    ok, f = query(65536, 67110.9)
    assert ok == 1
    mu, kap, kapm, al, be, ga, sAB, sB, nlam, CmAB, CmN = f[:11]
    lam = -nlam
    D, E = 1.0 + 2 * 67110.9, -67110.9
    c = 1.0 / kap
    assert abs(c * c - D * c + E * E) / (c * c) < 1e-12      # c solves c^2 - D c + E^2 = 0
    assert abs(lam - (-E / c)) < 1e-15 and abs(mu - lam * lam) < 1e-15
    assert abs(kapm - 1.0 / (c * (1.0 - mu))) / kapm < 1e-10
    assert abs(sAB - (1.0 - mu) / (1.0 + lam ** 32)) / sAB < 1e-10
    assert abs(CmAB - lam ** 16 / (1.0 + lam ** 32)) < 1e-12 and 0.49 < CmAB < 0.5
    g, rs, ro = f[11:27], f[27:43], f[43:59]
    assert np.allclose(rs[:15] * ro[:15], 1.0, rtol=1e-15)
    assert np.allclose(ro[:15], lam ** np.arange(15, 0, -1), rtol=1e-13)
    assert np.allclose(g[:15], -E * lam ** (2.0 * np.arange(15) - 15), rtol=1e-12)
    # dispatch
    assert query(65535, 67110.9)[0] == 0          # N not a multiple of the chunk
    assert query(1000, 656.6)[0] == 0             # partially filled last thread
    assert query(1024, 656.6)[0] == 1
    assert query(1024, 656.6, c_first=1.0)[0] == 0  # boundary forcing
    assert query(1024, 1e10)[0] == 0              # dt >> slowest mode: exact-pivot path
    assert query(65536, 1e10)[0] == 1


@pytest.mark.parametrize("a_d,a_o", [(-4.0, -1.5), (6.0, 1.0), (6.0, -2.4), (-2.0e4, 0.9e4)])
def test_fast_path_step_with_either_sign_of_the_coefficients(a_d, a_o):
    """The C ABI takes any symmetric constant-coefficient operator: positive
    off-diagonal step-matrix entries (lambda < 0) and negative diagonals run
    the same fast path; one emulated step solves (I - dt A) x = d."""
    import tri1d_emulator as EM
    n = 2048
    P = EM.export_plan(n, a_d, a_o, 0.0, 0.0, 1.0, 1)
    assert P["ccst"]
    d = np.random.default_rng(5).standard_normal(n)
    x = EM.step(d, P)
    D, E = P["D"], P["E"]
    res = D * x
    res[1:] += E * x[:-1]
    res[:-1] += E * x[1:]
    scale = abs(D) * np.abs(x).max() + np.abs(d).max()
    assert np.max(np.abs(res - d)) / scale < 1e-14
