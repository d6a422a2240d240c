"""Cost model against the reference's own known answers
(pkg/tests/test_analysis.py:226-272, test_acceptance.py:280-297). Host logic
only: runs without a GPU."""
import pytest

import paper_2110_10762_b200 as pb

REF = dict(p=16, fine_cost=14.0, coarse_cost=0.14, overhead=1.53)


def test_reference_cost_numbers():
    params = pb.CostParams(k=10, kappa=10, **REF)
    assert pb.sequential_cost(params) == pytest.approx(224.0, rel=1e-12)
    assert pb.sync_cost(params) == pytest.approx(288.99, abs=1e-9)
    assert pb.async_cost(params) == pytest.approx(143.64, abs=1e-9)
    assert pb.async_cost(pb.CostParams(k=10, kappa=24, **REF)) == pytest.approx(341.60, abs=1e-9)


def test_speedup_bound_numbers():
    rep = pb.speedup_bound(pb.CostParams(k=10, kappa=10, **REF))
    assert rep.bound == pytest.approx(1.0 + 14 * 1.53 / 14.14, rel=1e-12)
    assert rep.bound == pytest.approx(2.515, abs=1e-3)
    assert rep.achieved == pytest.approx(288.99 / 143.64, rel=1e-12)
    assert pb.speedup_bound(pb.CostParams(**REF)).achieved is None
    with pytest.raises(ValueError):
        pb.speedup_bound(pb.CostParams(k=10, kappa=5, **REF))
    with pytest.raises(ValueError):
        pb.speedup_bound(pb.CostParams(p=1, fine_cost=1.0, coarse_cost=1.0))
    with pytest.raises(pb.UndefinedLimitError):
        pb.speedup_bound(pb.CostParams(p=4, fine_cost=0.0, coarse_cost=0.0))


def test_asymptotic_limits():
    s, a, c = pb.asymptotic_speedups(pb.CostParams(k=10, **REF))
    assert s == pytest.approx(14.0 / (0.14 + 15.3), rel=1e-12)
    assert a == pytest.approx(100.0, rel=1e-12)
    assert c == pytest.approx(1.0 + 15.3 / 0.14, rel=1e-12)
    with pytest.raises(pb.UndefinedLimitError):
        pb.asymptotic_speedups(pb.CostParams(p=4, fine_cost=1.0, coarse_cost=0.0, k=2))


def test_fit_overhead_round_trip_and_edges():
    total = pb.sync_cost(pb.CostParams(k=10, **REF))
    assert pb.fit_overhead(total, 16, 10, 14.0, 0.14) == pytest.approx(1.53, rel=1e-12)
    with pytest.raises(pb.UnfittableError):
        pb.fit_overhead(100.0, 16, 0, 14.0, 0.14)
    with pytest.raises(pb.UnfittableError):
        pb.fit_overhead(100.0, 3, 3, 14.0, 0.14)
    assert pb.fit_overhead(0.0, 16, 10, 14.0, 0.14) == 0.0


def test_cost_model_edges():
    assert pb.sync_cost(pb.CostParams(p=4, fine_cost=2.0, coarse_cost=0.5, overhead=1.0, k=0)) == pytest.approx(2.0)
    with pytest.raises(ValueError):
        pb.sync_cost(pb.CostParams(p=4, fine_cost=2.0, coarse_cost=0.5, k=5))
    with pytest.raises(ValueError):
        pb.sync_cost(pb.CostParams(p=4, fine_cost=2.0, coarse_cost=0.5))
    with pytest.raises(ValueError):
        pb.async_cost(pb.CostParams(p=4, fine_cost=2.0, coarse_cost=0.5, kappa=-1))
    with pytest.raises(ValueError):
        pb.CostParams(p=0, fine_cost=1.0, coarse_cost=1.0)
    with pytest.raises(ValueError):
        pb.CostParams(p=2, fine_cost=-1.0, coarse_cost=1.0)


def test_model_report_from_measured_costs():
    costs = {"fine_cost": 2.0e-3, "fine_batch": 4.0e-3, "coarse_cost": 1.0e-4}
    total = pb.sync_cost(pb.CostParams(p=64, fine_cost=4.0e-3, coarse_cost=1.0e-4, overhead=2.0e-6, k=15))
    rep = pb.model_report(costs, 64, k=15, kappa=20, measured_sync_s=total)
    assert rep["overhead_fit_s"] == pytest.approx(2.0e-6, rel=1e-9)
    assert rep["sync_model_s"] == pytest.approx(total, rel=1e-12)
    assert rep["sequential_fine_s"] == pytest.approx(64 * 2.0e-3)
    assert rep["async_model_s"] == pytest.approx(64 * 1e-4 + 20 * 4.1e-3)
    assert rep["speedup_bound"] >= rep["speedup_model"]
