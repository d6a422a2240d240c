"""Contraction factors. Host logic against the reference's
own worked numbers (pkg/tests/test_analysis.py:38-103); the modal oracle
against golden values from the reference's dense contraction_factors
(tests/golden/contraction.npz); the GPU's matrix-free Lanczos norms against
both, including the full C2 size."""
import json

import numpy as np
import pytest

import paper_2110_10762_b200 as pb
from conftest import golden
from oracle import heat_oracle as H


def test_worked_scalar_factors():
    r = pb.factors_from_norms(0.8, 0.0212, p=4)
    assert r.theta == 0.8
    assert r.sync_factor == pytest.approx((1 - 0.8 ** 4) / 0.2 * 0.0212, rel=1e-12)
    assert r.sync_factor == pytest.approx(0.0625824, rel=1e-9)
    assert r.async_factor == pytest.approx(0.8212, rel=1e-12)
    sync = pb.sync_convergence_check(r)
    assert sync.holds
    assert sync.margin == pytest.approx(min(0.2, 1.0 + 0.8 ** 4 * 0.0212 - 0.8212), rel=1e-12)
    asyn = pb.async_convergence_check(r)
    assert asyn.holds and asyn.margin == pytest.approx(0.17880, rel=1e-9)
    cmp = pb.compare_factors(r)
    assert cmp.applicable and cmp.gap == pytest.approx(0.7586176, rel=1e-9)
    holds, margin = pb.CheckResult(True, 0.25)
    assert holds and margin == 0.25
    assert r.to_dict()["norm_kind"] == "spectral"


def test_theta_edges():
    assert pb.factors_from_norms(0.8, 0.0212, p=4, theta=1.0).sync_factor == pytest.approx(4 * 0.0212, rel=1e-12)
    assert pb.factors_from_norms(1.0, 0.1, p=3).sync_factor == pytest.approx(0.3)
    with pytest.raises(pb.InvalidThetaError):
        pb.factors_from_norms(0.8, 0.0212, p=4, theta=0.5)
    with pytest.raises(ValueError):
        pb.factors_from_norms(-0.1, 0.0212, p=4)
    with pytest.raises(ValueError):
        pb.factors_from_norms(0.8, 0.0212, p=0)
    with pytest.raises(ValueError):
        pb.compare_factors(pb.factors_from_norms(0.8, 0.0212, p=4, theta=0.9))
    cmp = pb.compare_factors(pb.factors_from_norms(0.9, 0.3, p=4))
    assert not cmp.applicable and cmp.gap is None
    r = pb.factors_from_norms(1.1, 0.05, p=4)
    assert not pb.sync_convergence_check(r).holds and not pb.async_convergence_check(r).holds


@pytest.mark.parametrize("tag", ["c1", "cn64", "fe2d"])
def test_modal_oracle_matches_reference_dense_norms(tag):
    g = golden("contraction.npz")
    meta = json.loads(str(g[f"{tag}_meta"]))
    cn, dn = H.modal_norms(tuple(meta["shape"]), meta["length"], tuple(meta["fine"]), tuple(meta["coarse"]))
    ref = g[f"{tag}_spectral"]
    assert cn == pytest.approx(ref[0], rel=1e-9)
    assert dn == pytest.approx(ref[1], rel=1e-9)
    r = pb.factors_from_norms(cn, dn, meta["p"])
    assert r.sync_factor == pytest.approx(ref[2], rel=1e-9)
    assert r.async_factor == pytest.approx(ref[3], rel=1e-9)


def _props(gpu, meta, dtype="float64"):
    shape = tuple(meta["shape"])
    n = shape[0]
    (fr, fdt, fs), (cr, cdt, cs) = meta["fine"], meta["coarse"]
    if len(shape) == 1:
        ivp = gpu.heat1d_system(n, meta["length"], 0.0, 0.0, 0.0, 1.0)
    else:
        ivp = (gpu.heat2d_system if len(shape) == 2 else gpu.heat3d_system)(n, t_final=1.0)
    fine = gpu.PROPAGATOR_RULES[fr](ivp, fdt * fs, fs, dtype=dtype)
    coarse = gpu.PROPAGATOR_RULES[cr](ivp, cdt * cs, cs, dtype=dtype)
    return coarse, fine


@pytest.mark.gpu
@pytest.mark.parametrize("tag", ["c1", "cn64", "fe2d"])
def test_gpu_contraction_factors_match_reference(gpu, tag):
    g = golden("contraction.npz")
    meta = json.loads(str(g[f"{tag}_meta"]))
    coarse, fine = _props(gpu, meta)
    r = gpu.contraction_factors(coarse, fine, meta["p"])
    ref = g[f"{tag}_spectral"]
    np.testing.assert_allclose([r.coarse_norm, r.defect_norm, r.sync_factor, r.async_factor], ref, rtol=1e-9)
    ri = gpu.contraction_factors(coarse, fine, meta["p"], kind=gpu.NormKind.INFINITY)
    np.testing.assert_allclose([ri.coarse_norm, ri.defect_norm, ri.sync_factor, ri.async_factor],
                               g[f"{tag}_infinity"], rtol=1e-9)


@pytest.mark.gpu
@pytest.mark.parametrize("shape,fine,coarse,p", [
    ((65536,), ("backward-euler", 1 / 64 / 1000, 1000), ("backward-euler", 1 / 64, 1), 64),   # C2
    ((256, 256), ("forward-euler", 0.2 / 257 ** 2, 500), ("backward-euler", 100 / 257 ** 2, 1), 32),
])
def test_gpu_contraction_factors_full_size_vs_modal(gpu, shape, fine, coarse, p):
    meta = {"shape": list(shape), "length": 1.0, "fine": list(fine), "coarse": list(coarse)}
    G, F = _props(gpu, meta)
    r = gpu.contraction_factors(G, F, p)
    cn, dn = H.modal_norms(shape, 1.0, fine, coarse)
    assert r.coarse_norm == pytest.approx(cn, rel=1e-9)
    assert r.defect_norm == pytest.approx(dn, rel=1e-8)
