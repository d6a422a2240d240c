"""Error semantics through the C ABI on the GPU, mirroring the reference's own
error tests: test_model.py:132-138 (singular implicit step), :166-174
(degenerate heat problem, apply dimension check), linalg.py:74-75 (non-finite
block entries), test_parareal.py:107-118 (argument checks),
test_async_engine.py:213 (HorizonExhausted), test_async_parareal.py:106-113
(stop-check edges)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_singular_implicit_step_is_reported(gpu):
    # backward Euler on u' = u with dt = 1 makes (I - dt A) exactly singular
    ivp = gpu.LinearIVP(np.array([[1.0]]), np.zeros(1), np.ones(1), 2.0)
    with pytest.raises(gpu.SingularSystemError) as err:
        gpu.backward_euler_propagator(ivp, 1.0, 1)
    assert err.value.dt == 1.0
    # the trapezoidal rule is singular at dt = 2 for the same problem
    with pytest.raises(gpu.SingularSystemError) as err:
        gpu.trapezoidal_propagator(ivp, 2.0, 1)
    assert err.value.dt == 2.0
    # nearby dt is fine and matches the closed form 1 / (1 - dt)
    out = gpu.backward_euler_propagator(ivp, 0.5, 1).apply(np.array([3.0]))
    assert out[0] == pytest.approx(6.0, rel=1e-15)


def test_degenerate_problem_and_apply_dim_check(gpu):
    with pytest.raises(gpu.DegenerateProblemError):
        gpu.heat1d_system(0, 1.0, 0.0, 0.0, 0.0, 1.0)
    ivp = gpu.heat1d_system(2, 1.0, 0.0, 0.0, 0.0, 1.0)
    prop = gpu.backward_euler_propagator(ivp, 0.5, 1)
    with pytest.raises(gpu.DimensionError):
        prop.apply(np.ones(3))
    ivp2 = gpu.heat2d_system(16, 1.0)
    fe = gpu.forward_euler_propagator(ivp2, 0.01, 10)
    with pytest.raises(gpu.DimensionError):
        fe.apply(np.ones(16 * 16 + 1))


def test_non_finite_initial_state_is_rejected(gpu):
    ivp = gpu.heat1d_system(64, 1.0, 0.0, 0.0, 0.0, 1.0)
    fine = gpu.backward_euler_propagator(ivp, 1 / 8, 10)
    coarse = gpu.backward_euler_propagator(ivp, 1 / 8, 1)
    u0 = np.ones(64)
    u0[7] = np.nan
    with pytest.raises(ValueError):
        gpu.run_parareal(coarse, fine, u0, 8, 1e-10)
    u0[7] = np.inf
    with pytest.raises(ValueError):
        gpu.run_parareal(coarse, fine, u0, 8, 1e-10)


def test_overflowing_iterate_is_reported_non_finite(gpu):
    """An unstable explicit F overflows to inf inside the sweep: the device
    non-finite flag surfaces as the reference's ValueError (linalg.py:74-75)
    instead of a silent inf/nan iterate."""
    ivp = gpu.heat2d_system(32, 1.0)
    h2 = (1.0 / 33) ** 2
    # dt = 50 h^2 is far beyond the FE stability limit h^2/4: growth ~ 400^steps
    fine = gpu.forward_euler_propagator(ivp, 200 * 50 * h2, 200, dtype="float32")
    coarse = gpu.backward_euler_propagator(ivp, 200 * 50 * h2, 1, dtype="float32")
    rng = np.random.default_rng(0)
    u0 = rng.standard_normal(32 * 32)
    with pytest.raises(ValueError, match="finite"):
        gpu.run_parareal(coarse, fine, u0, 4, 1e-6)


def test_driver_argument_checks(gpu):
    ivp = gpu.heat1d_system(16, 1.0, 0.0, 0.0, 0.0, 1.0)
    fine = gpu.backward_euler_propagator(ivp, 0.25, 10)
    coarse = gpu.backward_euler_propagator(ivp, 0.25, 1)
    other = gpu.backward_euler_propagator(gpu.heat1d_system(17, 1.0, 0.0, 0.0, 0.0, 1.0), 0.25, 1)
    u0 = np.ones(16)
    with pytest.raises(ValueError):
        gpu.run_parareal(coarse, fine, u0, 0, 1e-10)
    with pytest.raises(ValueError):
        gpu.run_parareal(coarse, fine, u0, 4, -1.0)
    with pytest.raises(ValueError):
        gpu.run_parareal(coarse, fine, u0, 4, 1e-10, k_max=0)
    with pytest.raises(gpu.DimensionError):
        gpu.run_parareal(coarse, fine, np.ones(15), 4, 1e-10)
    with pytest.raises(gpu.DimensionError):
        gpu.run_parareal(other, fine, u0, 4, 1e-10)
    with pytest.raises(ValueError):
        gpu.sequential_fine_solve(fine, u0, 0)
    with pytest.raises(ValueError):
        gpu.coarse_init(coarse, u0, 0)


def test_async_horizon_exhausted_and_stop_check_edges(gpu):
    ivp = gpu.heat1d_system(256, 1.0, 0.0, 0.0, 0.0, 1.0)
    fine = gpu.backward_euler_propagator(ivp, 1 / 16, 50)
    coarse = gpu.backward_euler_propagator(ivp, 1 / 16, 1)
    u0 = np.sin(np.pi * np.arange(1, 257) / 257)
    # the simulator with a horizon far too short for exact quiescence
    sched = gpu.AsyncSchedule(seed=1, delay_bound=1, max_events=20)
    with pytest.raises(gpu.HorizonExhausted) as err:
        gpu.run_async_parareal(coarse, fine, u0, 16, sched)
    assert len(err.value.trace.events) == 20
    # the device runtime with an activation budget far too small
    with pytest.raises(gpu.HorizonExhausted):
        gpu.run_async_parareal_device(coarse, fine, u0, 16, None, max_events=20)
    assert gpu.async_stop_check([1e-7, 2e-7], epsilon=1e-6, drained=True)
    assert not gpu.async_stop_check([1e-6, 2e-7], epsilon=1e-6, drained=True)
    assert not gpu.async_stop_check([1e-9], epsilon=1e-6, drained=False)
    for eps in (0.0, -1.0):
        with pytest.raises(ValueError):
            gpu.async_stop_check([0.0], epsilon=eps, drained=True)
    with pytest.raises(ValueError):
        gpu.async_parareal_mapping(coarse, fine, 0)


def test_parareal_mapping_shape_and_simulate_async(gpu):
    """reference test_async_parareal.py:34-45: the two-slot mapping, and the
    generic event loop entry (simulate_async) running it equals
    run_async_parareal bitwise."""
    ivp = gpu.heat1d_system(8, 1.0, 23.0, 23.0, 30.0, 0.2)
    coarse = gpu.backward_euler_propagator(ivp, 0.2, 1)
    fine = gpu.trapezoidal_propagator(ivp, 0.2, 100)
    mapping = gpu.async_parareal_mapping(coarse, fine, 4)
    assert mapping.n_updatable == 4 and mapping.arity == 2
    assert mapping.persistent_slots == {gpu.REMEMBERED_SLOT: gpu.FRESH_SLOT}
    for i in range(1, 5):
        assert mapping.read_set[i] == ((i - 1, gpu.FRESH_SLOT), (i - 1, gpu.REMEMBERED_SLOT))
    sched = gpu.AsyncSchedule(seed=2, delay_bound=1)
    want = gpu.run_async_parareal(coarse, fine, ivp.u0, 4, sched)
    init = gpu.coarse_init(coarse, ivp.u0, 4)
    got = gpu.simulate_async(mapping, init, sched)
    assert got.stop_reason == want.stop_reason
    assert len(got.events) == len(want.events)
    assert np.array_equal(got.final.data, want.final.data)
    # eval_fn is the update kernel on its two readings
    v = mapping.eval_fn(2, {(1, gpu.FRESH_SLOT): init.data[1], (1, gpu.REMEMBERED_SLOT): init.data[1]})
    assert np.array_equal(v, fine.apply(init.data[1]))
    with pytest.raises(gpu.DimensionError):
        gpu.simulate_async(mapping, init.data[:4], sched)
