"""The reference's driver-semantics tests (pintlab tests/test_parareal.py:
coarse_init, parareal_update branches, stop order, k_max, epsilon = 0,
frozen prefix) restated on the GPU propagators (scalar decay and heat1d
instead of the reference's literal 1x1 affine maps, which the structured GPU
operators do not represent)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_coarse_init_geometric_sequence(gpu):
    # backward Euler, one step: lambda_i = (1 / (1 + rate dt))^i  (test_parareal.py:29-33)
    ivp = gpu.scalar_decay_system(rate=0.25, t_final=3.0)
    coarse = gpu.backward_euler_propagator(ivp, 1.0, 1)
    lam = gpu.coarse_init(coarse, [1.0], 3).data.ravel()
    assert np.allclose(lam, [1.0, 0.8, 0.64, 0.512], rtol=0, atol=1e-15)


def test_update_kernel_branches(gpu):
    # (G(fresh) + F(old)) - G(old); bitwise-equal readings collapse to F(old) (test_parareal.py:51-59)
    ivp = gpu.scalar_decay_system(rate=0.25, t_final=2.0)
    coarse = gpu.backward_euler_propagator(ivp, 1.0, 1)
    fine = gpu.trapezoidal_propagator(ivp, 1.0, 25)
    fresh, old = np.array([0.77880]), np.array([0.8])
    got = gpu.parareal_update(coarse, fine, fresh, old)
    want = (coarse.apply(fresh) + fine.apply(old)) - coarse.apply(old)
    assert got[0] == want[0]
    same = gpu.parareal_update(coarse, fine, old.copy(), old)
    assert np.array_equal(same, fine.apply(old))


def test_equal_propagators_stop_at_first_sweep(gpu):
    # test_parareal.py:62-69
    ivp = gpu.scalar_decay_system(rate=1.0, t_final=4.0)
    coarse = gpu.backward_euler_propagator(ivp, 1.0, 5)
    tr = gpu.run_parareal(coarse, coarse, ivp.u0, 4, epsilon=1e-12)
    assert tr.k_final == 1 and tr.stop_reason == "threshold"
    assert tr.deltas == [0.0]
    assert np.array_equal(tr.iterates[1].data, tr.iterates[0].data)


def test_epsilon_zero_disables_threshold(gpu):
    # strict comparison: delta == 0 < 0 is false -> k = p, "exact" (test_parareal.py:72-78)
    ivp = gpu.scalar_decay_system(rate=1.0, t_final=3.0)
    coarse = gpu.backward_euler_propagator(ivp, 1.0, 2)
    tr = gpu.run_parareal(coarse, coarse, ivp.u0, 3, epsilon=0.0)
    assert tr.k_final == 3 and tr.stop_reason == "exact"


def test_k_max_stop_and_argument_errors(gpu):
    # test_parareal.py:107-118
    ivp = gpu.scalar_decay_system(rate=1.0, t_final=6.0)
    coarse = gpu.backward_euler_propagator(ivp, 1.0, 1)
    fine = gpu.trapezoidal_propagator(ivp, 1.0, 25)
    tr = gpu.run_parareal(coarse, fine, ivp.u0, 6, epsilon=1e-14, k_max=2)
    assert tr.k_final == 2 and tr.stop_reason == "k_max" and len(tr.iterates) == 3
    with pytest.raises(ValueError):
        gpu.run_parareal(coarse, fine, ivp.u0, 6, epsilon=-1.0)
    with pytest.raises(ValueError):
        gpu.run_parareal(coarse, fine, ivp.u0, 6, epsilon=1e-9, k_max=0)


@pytest.mark.parametrize("n,p", [(4, 6), (64, 9), (1024, 16)])
def test_prefix_is_frozen_and_exact_bitwise(gpu, n, p):
    # test_parareal.py:91-104, on the heat fixture and larger grids
    ivp = gpu.heat1d_system(n, 1.0, 23.0, 23.0, 30.0, 0.2)
    coarse = gpu.backward_euler_propagator(ivp, 0.2 / p, 1)
    fine = gpu.trapezoidal_propagator(ivp, 0.2 / p, 100)
    tr = gpu.run_parareal(coarse, fine, ivp.u0, p, epsilon=0.0, record_iterates=True)
    seq = gpu.sequential_fine_solve(fine, ivp.u0, p).data
    for k in range(1, len(tr.iterates)):
        for i in range(k):
            assert np.array_equal(tr.iterates[k].data[i], tr.iterates[k - 1].data[i])
        for i in range(k + 1):
            assert np.array_equal(tr.iterates[k].data[i], seq[i])


def test_parareal_iterate_is_the_unfrozen_sweep(gpu):
    # parareal_iterate (parareal.py:66-76): every slice updated, no freeze;
    # after p iterations from the coarse guess it is the sequential fine solve
    ivp = gpu.heat1d_system(8, 1.0, 23.0, 23.0, 30.0, 0.2)
    p = 5
    coarse = gpu.backward_euler_propagator(ivp, 0.2 / p, 1)
    fine = gpu.trapezoidal_propagator(ivp, 0.2 / p, 100)
    lam = gpu.coarse_init(coarse, ivp.u0, p)
    for _ in range(p):
        lam = gpu.parareal_iterate(coarse, fine, lam)
    seq = gpu.sequential_fine_solve(fine, ivp.u0, p).data
    assert np.array_equal(lam.data, seq)


def test_parareal_iterate_host_buffers_equal_one_run_parareal_sweep(gpu):
    """The public host-in/host-out call (the bench's e2e) is bitwise one sweep
    of run_parareal from the same iterate: at the C2 layout (chunked,
    pipelined, graph-replayed sweep) and at a 3-D generic-chain layout."""
    import torch
    from paper_2110_10762_b200.inputs import sine_u0_1d
    n, p = 65536, 64
    ivp = gpu.heat1d_system(n, 1.0, 0.0, 0.0, 0.0, 1.0)
    fine = gpu.backward_euler_propagator(ivp, 1.0 / p, 50)
    coarse = gpu.backward_euler_propagator(ivp, 1.0 / p, 1)
    u0 = sine_u0_1d(n, 32, 0)
    tr = gpu.run_parareal(coarse, fine, u0, p, 0.0, k_max=1, record_iterates=True)
    host = torch.from_numpy(tr.iterates[0].data.copy()).pin_memory()
    out = torch.empty_like(host).pin_memory()
    for _ in range(2):  # second call replays the captured graph
        new = gpu.parareal_iterate(coarse, fine, gpu.BlockVector(host, check_finite=False), out=out)
        assert new.tensor.device.type == "cpu"
        assert torch.equal(new.tensor, tr.iterates[1].tensor.cpu())
    # 3-D: the generic chain (pint_correct_chain)
    m, q = 24, 5
    h = 1.0 / (m + 1)
    ivp3 = gpu.heat3d_system(m, t_final=1.0)
    f3 = gpu.forward_euler_propagator(ivp3, 7 * 0.15 * h * h, 7, dtype="float32")
    g3 = gpu.backward_euler_propagator(ivp3, 7 * 0.15 * h * h, 1, dtype="float32")
    u3 = np.random.default_rng(2).standard_normal(m ** 3)
    t3 = gpu.run_parareal(g3, f3, u3, q, 0.0, k_max=2, record_iterates=True)
    for k in (0, 1):
        h3 = torch.from_numpy(t3.iterates[k].data.copy())
        new = gpu.parareal_iterate(g3, f3, gpu.BlockVector(h3, check_finite=False))
        # slices frozen in run_parareal (i < k) are recomputed F-only from unchanged
        # inputs by the unfrozen sweep: the same bits
        assert torch.equal(new.tensor, t3.iterates[k + 1].tensor.cpu())
