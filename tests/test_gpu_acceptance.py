"""The reference's acceptance criteria that lie on the hot path
(pintlab tests/test_acceptance.py: crit 1, 2, 3, 8, 9), run through the GPU
drivers and propagators. Same setups, seeds, schedules and tolerances."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HEAT_SPAN = 0.2


def heat_setup(gpu, n):
    ivp = gpu.heat1d_system(n, 1.0, 23.0, 23.0, 30.0, HEAT_SPAN)
    return ivp, gpu.backward_euler_propagator(ivp, HEAT_SPAN, 1), gpu.trapezoidal_propagator(ivp, HEAT_SPAN, 100)


def scalar_setup(gpu):
    ivp = gpu.scalar_decay_system(rate=1.0, t_final=8.0)
    span = ivp.t_final / 8
    return ivp, gpu.backward_euler_propagator(ivp, span, 1), gpu.trapezoidal_propagator(ivp, span, 25)


def suite_layout(seed):
    """test_acceptance.py:80-86: (n, delay_bound, p) for seeds 1..20."""
    return (4 if seed % 2 == 1 else 8), (seed - 1) % 3 + 1, 2 + (seed - 1) % 7


def max_block_norm(x, kind):
    """linalg.py:136-146: largest per-block norm (2-norm / max-abs)."""
    x = np.asarray(x)
    return float(np.max(np.abs(x))) if kind == "infinity" else float(np.max(np.linalg.norm(x, axis=1)))


def test_crit01_sync_finite_termination(gpu):
    for n in (4, 8):
        ivp, coarse, fine = heat_setup(gpu, n)
        assert fine.cost_units / coarse.cost_units == 100.0
        for p in range(2, 9):
            seq = gpu.sequential_fine_solve(fine, ivp.u0, p).data
            tr = gpu.run_parareal(coarse, fine, ivp.u0, p, 0.0)
            gap = np.max(np.abs(tr.iterates[-1].data - seq) / np.abs(seq))
            assert tr.k_final == p and gap <= 1e-12, (n, p, tr.k_final, gap)


def test_crit02_async_exact_quiescence(gpu):
    for seed in range(1, 21):
        n, d, p = suite_layout(seed)
        ivp, coarse, fine = heat_setup(gpu, n)
        seq = gpu.sequential_fine_solve(fine, ivp.u0, p).data
        sched = gpu.AsyncSchedule(seed=seed, delay_bound=d, policy=gpu.POLICY_RANDOM_FAIR)
        tr = gpu.run_async_parareal(coarse, fine, ivp.u0, p, sched)
        final = tr.state_after(len(tr.events) - 1).data
        assert np.max(np.abs(final - seq) / np.abs(seq)) <= 1e-12, seed
        # a finite match index (analysis.py:223-240)
        assert any(np.allclose(tr.state_after(i).data, seq, rtol=1e-12, atol=0.0)
                   for i in range(-1, len(tr.events))), seed


def test_crit03_sync_error_contraction_bound(gpu):
    cases = []
    for n in (4, 8):
        ivp, coarse, fine = heat_setup(gpu, n)
        cases.append((f"heat-{n}", coarse, fine, ivp.u0, 8))
    ivp, coarse, fine = scalar_setup(gpu)
    cases.append(("scalar-decay", coarse, fine, ivp.u0, 8))
    slack = 1.0 + 1e-10
    for label, coarse, fine, u0, p in cases:
        spectral = gpu.contraction_factors(coarse, fine, p, kind=gpu.NormKind.SPECTRAL)
        assert spectral.coarse_norm < 1.0, label
        seq = gpu.sequential_fine_solve(fine, u0, p).data
        tr = gpu.run_parareal(coarse, fine, u0, p, 0.0)
        pairings = [("spectral", spectral, "spectral"),
                    ("infinity", gpu.contraction_factors(coarse, fine, p, kind=gpu.NormKind.INFINITY), "infinity"),
                    ("mixed", spectral, "infinity")]
        for tag, rep, err_kind in pairings:
            errors = [max_block_norm(it.data - seq, err_kind) for it in tr.iterates]
            for k, e_k in enumerate(errors):
                assert e_k <= rep.sync_factor ** k * errors[0] * slack, (label, tag, k)


def test_crit08_zero_delay_bitwise_reduction(gpu):
    ivp, coarse, fine = scalar_setup(gpu)
    p, eps = 8, 1e-5
    sync = gpu.run_parareal(coarse, fine, ivp.u0, p, eps)
    sched = gpu.AsyncSchedule(seed=0, delay_bound=0, policy=gpu.POLICY_ROUND_ROBIN)
    tr = gpu.run_async_parareal(coarse, fine, ivp.u0, p, sched, epsilon=eps)
    _, kappa = gpu.update_counts(tr)
    assert sync.stop_reason == "threshold" and kappa == sync.k_final
    for cycle in range(sync.k_final):
        assert np.array_equal(tr.state_after(cycle * p + p - 1).data, sync.iterates[cycle + 1].data)


def test_crit09_async_activation_counts(gpu):
    eps = 1e-6
    for seed in range(1, 21):
        n, d, p = suite_layout(seed)
        ivp, coarse, fine = heat_setup(gpu, n)
        sync = gpu.run_parareal(coarse, fine, ivp.u0, p, eps)
        sched = gpu.AsyncSchedule(seed=seed, delay_bound=d, policy=gpu.POLICY_RANDOM_FAIR)
        tr = gpu.run_async_parareal(coarse, fine, ivp.u0, p, sched, epsilon=eps)
        _, kappa = gpu.update_counts(tr)
        assert kappa >= sync.k_final, (seed, kappa, sync.k_final)
        # and the device runtime (real concurrency) on the same problem
        res = gpu.run_async_parareal_device(coarse, fine, ivp.u0, p, eps, seed=seed)
        assert res.kappa >= sync.k_final, (seed, res.kappa, sync.k_final)
