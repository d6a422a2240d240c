"""Asynchronous Parareal on the GPU: the reference's deterministic event
semantics (same seeds -> same activations, reads and values), exactness
cascade, and the zero-delay reduction to the synchronous sweep."""
import json

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu

CASES = ("rf_s5_d1_p6", "rf_s9_d2_p6", "adv_s3_d2_p5", "rr_s0_d0_p6_eps", "rf_s4_d3_p7_eps")


def heat_pair(gpu, n):
    ivp = gpu.heat1d_system(n, 1.0, 23.0, 23.0, 30.0, 0.2)
    return ivp, gpu.backward_euler_propagator(ivp, 0.2, 1), gpu.trapezoidal_propagator(ivp, 0.2, 100)


@pytest.mark.parametrize("tag", CASES)
def test_async_trace_matches_reference(gpu, tag):
    g = golden("async_traces.npz")
    sched = json.loads(str(g[f"{tag}_sched"]))
    ivp, coarse, fine = heat_pair(gpu, 4)
    s = gpu.AsyncSchedule(seed=sched["seed"], delay_bound=sched["delay_bound"], policy=sched["policy"])
    tr = gpu.run_async_parareal(coarse, fine, ivp.u0, sched["p"], s, epsilon=sched["eps"])
    comps = np.array([e.component for e in tr.events])
    reads = np.array([[r[2] for r in e.reads] for e in tr.events])
    assert np.array_equal(comps, g[f"{tag}_components"])
    assert np.array_equal(reads, g[f"{tag}_reads"])
    assert tr.stop_reason == str(g[f"{tag}_stop"])
    assert np.array_equal(tr.per_component_counts, g[f"{tag}_counts"])
    final = tr.state_after(len(tr.events) - 1).data
    assert np.max(np.abs(final - g[f"{tag}_final"]) / np.abs(g[f"{tag}_final"])) < 1e-12


def test_event_replay_and_remembered_slot(gpu):
    ivp, coarse, fine = heat_pair(gpu, 4)
    tr = gpu.run_async_parareal(coarse, fine, ivp.u0, 5, gpu.AsyncSchedule(seed=12, delay_bound=2))
    prev_fresh = {}
    for idx, ev in enumerate(tr.events):
        reads = {slot: (src, v) for src, slot, v in ev.reads}
        if ev.component in prev_fresh:
            assert reads[gpu.REMEMBERED_SLOT] == prev_fresh[ev.component]
        else:
            assert reads[gpu.REMEMBERED_SLOT][1] == 0
        prev_fresh[ev.component] = reads[gpu.FRESH_SLOT]
        vals = {slot: tr.version_value(src, v) for src, slot, v in ev.reads}
        want = gpu.parareal_update(coarse, fine, vals[gpu.FRESH_SLOT], vals[gpu.REMEMBERED_SLOT])
        assert np.array_equal(want, tr.snapshots[idx][ev.component]), idx
    assert gpu.validate_schedule(tr).ok


def test_quiescence_is_the_sequential_fine_solution_bitwise(gpu):
    ivp, coarse, fine = heat_pair(gpu, 4)
    p = 6
    seq = gpu.sequential_fine_solve(fine, ivp.u0, p).data
    for seed, d in [(5, 1), (9, 2), (14, 3)]:
        tr = gpu.run_async_parareal(coarse, fine, ivp.u0, p, gpu.AsyncSchedule(seed=seed, delay_bound=d))
        assert tr.stop_reason == "quiescence"
        assert np.array_equal(tr.state_after(len(tr.events) - 1).data, seq)


def test_zero_delay_round_robin_is_the_sync_sweep_bitwise(gpu):
    ivp = gpu.scalar_decay_system(rate=1.0, t_final=8.0)
    p = 8
    coarse = gpu.backward_euler_propagator(ivp, 1.0, 1)
    fine = gpu.trapezoidal_propagator(ivp, 1.0, 25)
    sync = gpu.run_parareal(coarse, fine, ivp.u0, p, 1e-5)
    assert sync.stop_reason == "threshold" and sync.k_final == 7
    sched = gpu.AsyncSchedule(seed=0, delay_bound=0, policy=gpu.POLICY_ROUND_ROBIN)
    tr = gpu.run_async_parareal(coarse, fine, ivp.u0, p, sched, epsilon=1e-5)
    assert tr.stop_reason == "stop-predicate"
    _, kappa = gpu.update_counts(tr)
    assert kappa == sync.k_final
    for cycle in range(sync.k_final):
        assert np.array_equal(tr.state_after(cycle * p + p - 1).data, sync.iterates[cycle + 1].data), cycle


def test_c1_async_reaches_the_sync_solution(gpu):
    """Async-Parareal must reach the same converged solution within the
    stopping tolerance (north star)."""
    from oracle import heat_oracle as H
    n, p = 1024, 16
    u0 = H.sine_u0_1d(n, 8, 0)
    ivp = gpu.heat1d_system(n, 1.0, 0.0, 0.0, 0.0, 1.0)
    fine = gpu.backward_euler_propagator(ivp, 1 / p, 100)
    coarse = gpu.backward_euler_propagator(ivp, 1 / p, 1)
    seq = gpu.sequential_fine_solve(fine, u0, p).data
    tr = gpu.run_async_parareal(coarse, fine, u0, p, gpu.AsyncSchedule(seed=3, delay_bound=2), epsilon=1e-10,
                                record_snapshots=False)
    final = tr.state_after(len(tr.events) - 1).data
    assert np.max(np.abs(final - seq)) < 1e-8
    _, kappa = gpu.update_counts(tr)
    sync = gpu.run_parareal(coarse, fine, u0, p, 1e-10)
    assert kappa >= sync.k_final


# ------------------------------------------------ device runtime (real async)
@pytest.mark.parametrize("delay", [0.0, 0.2])
def test_device_async_quiescence_is_the_sequential_solution(gpu, delay):
    """Real concurrency: exact quiescence lands on the sequential fine solution
    bitwise (finite termination)."""
    from oracle import heat_oracle as H
    n, p = 1024, 16
    u0 = H.sine_u0_1d(n, 8, 0)
    ivp = gpu.heat1d_system(n, 1.0, 0.0, 0.0, 0.0, 1.0)
    fine = gpu.backward_euler_propagator(ivp, 1 / p, 100)
    coarse = gpu.backward_euler_propagator(ivp, 1 / p, 1)
    seq = gpu.sequential_fine_solve(fine, u0, p).data
    res = gpu.run_async_parareal_device(coarse, fine, u0, p, None, delay_frac=delay, seed=7)
    assert res.stop_reason == "converged"
    assert np.array_equal(res.final.data, seq)
    assert res.kappa >= 1 and res.activations >= p


@pytest.mark.parametrize("n,p,domains,rule", [(65537, 24, 1, "be"), (100_000, 20, 2, "be"), (40_001, 16, 2, "cn")])
def test_device_async_ragged_large_grid_quiescence(gpu, n, p, domains, rule):
    """Ragged C2-scale grids (10- and 14-CTA clusters, padded warps, tail
    chunks; trapezoidal F with forcing on the 16-point layout): the
    persistent runtime still quiesces on the sequential fine solution
    bitwise."""
    from paper_2110_10762_b200.inputs import sine_u0_1d
    u0 = sine_u0_1d(n, 16, 5)
    ivp = gpu.heat1d_system(n, 1.0, 0.0, 0.0, 0.0, 1.0) if rule == "be" else gpu.heat1d_system(n, 1.0, 0.4, 0.1, 0.0, 1.0)
    fn = gpu.backward_euler_propagator if rule == "be" else gpu.trapezoidal_propagator
    fine = fn(ivp, 1 / p, 10)
    coarse = gpu.backward_euler_propagator(ivp, 1 / p, 1)
    seq = gpu.sequential_fine_solve(fine, u0, p).data
    res = gpu.run_async_parareal_device(coarse, fine, u0, p, None, delay_frac=0.1, seed=n, domains=domains)
    assert res.stop_reason == "converged"
    assert np.array_equal(res.final.data, seq)


def test_device_async_epsilon_stop_reaches_sync_solution(gpu):
    from oracle import heat_oracle as H
    n, p = 1024, 16
    u0 = H.sine_u0_1d(n, 8, 0)
    ivp = gpu.heat1d_system(n, 1.0, 0.0, 0.0, 0.0, 1.0)
    fine = gpu.backward_euler_propagator(ivp, 1 / p, 100)
    coarse = gpu.backward_euler_propagator(ivp, 1 / p, 1)
    seq = gpu.sequential_fine_solve(fine, u0, p).data
    res = gpu.run_async_parareal_device(coarse, fine, u0, p, 1e-10)
    assert res.stop_reason == "converged"
    assert np.max(np.abs(res.final.data - seq)) < 1e-8


def test_device_async_fixture_with_boundary_forcing(gpu):
    ivp, coarse, fine = heat_pair(gpu, 8)
    for p in (3, 7):
        seq = gpu.sequential_fine_solve(fine, ivp.u0, p).data
        res = gpu.run_async_parareal_device(coarse, fine, ivp.u0, p, None, seed=p)
        assert np.array_equal(res.final.data, seq)


@pytest.mark.parametrize("delay,n,p", [(0.0, 1024, 16), (0.3, 1024, 16), (0.0, 65536, 24)])
def test_device_async_trace_audit(gpu, delay, n, p):
    """Race audit of real concurrent runs: every published
    activation read a version that had been published (causality), its
    remembered reading is the previous fresh reading of the same slice
    (provenance), per-slice publish counts match the counters, several
    activations were in flight at once, and the trace exports as the
    reference's AsyncTrace/JSONL."""
    from oracle import heat_oracle as H
    u0 = H.sine_u0_1d(n, 8, 0)
    ivp = gpu.heat1d_system(n, 1.0, 0.0, 0.0, 0.0, 1.0)
    fine = gpu.backward_euler_propagator(ivp, 1 / p, 100)
    coarse = gpu.backward_euler_propagator(ivp, 1 / p, 1)
    res = gpu.run_async_parareal_device(coarse, fine, u0, p, None, delay_frac=delay, seed=3, record_trace=True)
    assert res.stop_reason == "converged"
    rec = res.trace_records
    assert len(rec) == res.activations
    audit = gpu.audit_device_trace(rec, p, res.per_component_counts)
    assert audit["ok"], audit
    assert audit["peak_in_flight"] >= 2, audit
    assert audit["clusters_used"] >= 2, audit
    # exact quiescence: each slice's last publish was F-only on the newest predecessor
    last = {}
    for r in rec:
        last[int(r[0])] = r
    assert all(int(last[i][3]) == 1 for i in range(1, p + 1))
    tr = res.to_async_trace()
    assert len(tr.events) == res.activations
    assert tr.to_jsonl().count("\n") == res.activations
    _, kappa = gpu.update_counts(tr)
    assert kappa == res.kappa


# ------------------------------------- multi-domain runtime (multi-GPU protocol)
def _c1_pair(gpu, n, p):
    from oracle import heat_oracle as H
    u0 = H.sine_u0_1d(n, 8, 0)
    ivp = gpu.heat1d_system(n, 1.0, 0.0, 0.0, 0.0, 1.0)
    return u0, gpu.backward_euler_propagator(ivp, 1 / p, 100), gpu.backward_euler_propagator(ivp, 1 / p, 1)


@pytest.mark.parametrize("domains,delay,n,p", [(2, 0.0, 1024, 16), (3, 0.2, 1024, 16), (4, 0.0, 1024, 17),
                                               (8, 0.1, 1024, 16), (4, 0.0, 65536, 24)])
def test_device_async_domains_quiescence(gpu, domains, delay, n, p):
    """Slices split into `domains` contiguous domains with their own rings,
    ghost mailboxes (the predecessor domain pushes its last slice into them)
    and status boards, hosted by one launch: the multi-GPU protocol on one
    device. Exact quiescence must land on the sequential fine solution
    bitwise, the trace must pass the race audit, and every domain boundary
    must have carried pushed versions."""
    from paper_2110_10762_b200.distributed import async_partition
    u0, fine, coarse = _c1_pair(gpu, n, p)
    seq = gpu.sequential_fine_solve(fine, u0, p).data
    res = gpu.run_async_parareal_device(coarse, fine, u0, p, None, delay_frac=delay, seed=11, record_trace=True,
                                        domains=domains)
    assert res.stop_reason == "converged"
    assert np.array_equal(res.final.data, seq)
    rec = res.trace_records
    assert len(rec) == res.activations
    audit = gpu.audit_device_trace(rec, p, res.per_component_counts)
    assert audit["ok"], audit
    owners = rec[:, 7] // 65536
    parts = async_partition(p, domains)
    assert set(owners.tolist()) == set(range(domains))
    for o, i in zip(owners, rec[:, 0]):
        assert parts[o][0] <= i <= parts[o][1]
    for lo, _ in parts[1:]:
        first = rec[rec[:, 0] == lo]
        assert first[:, 1].max() >= 1  # read versions of the ghost pushed by the previous domain
    last = {}
    for r in rec:
        last[int(r[0])] = r
    assert all(int(last[i][3]) == 1 for i in range(1, p + 1))


def test_device_async_domains_epsilon_stop(gpu):
    n, p = 1024, 16
    u0, fine, coarse = _c1_pair(gpu, n, p)
    seq = gpu.sequential_fine_solve(fine, u0, p).data
    for domains in (2, 4):
        res = gpu.run_async_parareal_device(coarse, fine, u0, p, 1e-10, domains=domains, seed=domains)
        assert res.stop_reason == "converged"
        assert np.max(np.abs(res.final.data - seq)) < 1e-8
        sync = gpu.run_parareal(coarse, fine, u0, p, 1e-10)
        assert res.kappa >= sync.k_final


def test_device_async_domains_arguments(gpu):
    n, p = 1024, 4
    u0, fine, coarse = _c1_pair(gpu, n, p)
    with pytest.raises(ValueError):
        gpu.run_async_parareal_device(coarse, fine, u0, p, None, domains=5)
    with pytest.raises(ValueError):  # the status word holds 21-bit counters
        gpu.run_async_parareal_device(coarse, fine, u0, p, None, domains=2, max_events=1 << 22)


# ------------------------------------------- 2-D/3-D: stream-orchestrated runtime
def _nd_pair(gpu, shape, p, steps, cfl, dtype="float64"):
    from paper_2110_10762_b200 import inputs
    n = shape[0]
    h = 1.0 / (n + 1)
    span = steps * cfl * h * h
    u0 = inputs.sine_u0(shape, seed=1)
    mk = gpu.heat2d_system if len(shape) == 2 else gpu.heat3d_system
    ivp = mk(n, t_final=p * span, u0=u0)
    fine = gpu.forward_euler_propagator(ivp, span, steps, dtype=dtype)
    coarse = gpu.backward_euler_propagator(ivp, span, 1, dtype=dtype)
    return u0, fine, coarse


@pytest.mark.parametrize("shape,p,lanes,domains,delay", [((48, 48), 8, 3, 1, 0.0), ((48, 48), 9, 4, 3, 0.3),
                                                         ((20, 20, 20), 6, 2, 2, 0.0)])
def test_stream_async_quiescence_is_the_sequential_solution(gpu, shape, p, lanes, domains, delay):
    """2-D/3-D async Parareal on CUDA streams: exact quiescence lands on the
    sequential fine solution bitwise (finite termination), the trace passes
    the race audit, and domain boundaries carried pushed versions."""
    from paper_2110_10762_b200.distributed import async_partition
    u0, fine, coarse = _nd_pair(gpu, shape, p, 40, 0.2 if len(shape) == 2 else 0.15)
    seq = gpu.sequential_fine_solve(fine, u0, p).data
    res = gpu.run_async_parareal_device(coarse, fine, u0, p, None, lanes=lanes, domains=domains,
                                        delay_frac=delay, seed=3)
    assert res.stop_reason == "converged"
    assert np.array_equal(res.final.data, seq)
    audit = gpu.audit_device_trace(res.trace_records, p, res.per_component_counts)
    assert audit["ok"], audit
    rec = res.trace_records
    for lo, _ in async_partition(p, domains)[1:]:
        assert rec[rec[:, 0] == lo][:, 1].max() >= 1


def test_stream_async_epsilon_stop(gpu):
    u0, fine, coarse = _nd_pair(gpu, (64, 64), 8, 100, 0.2)
    seq = gpu.sequential_fine_solve(fine, u0, p=8).data
    res = gpu.run_async_parareal_device(coarse, fine, u0, 8, 1e-10, lanes=4, domains=2)
    assert res.stop_reason == "converged"
    assert np.max(np.abs(res.final.data - seq)) < 1e-8
    sync = gpu.run_parareal(coarse, fine, u0, 8, 1e-10)
    assert res.kappa >= sync.k_final
