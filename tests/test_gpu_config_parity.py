"""Oracle parity at the BASELINE configurations themselves (SURVEY §8c,
north_star: "synchronous Parareal iterates must match per iteration k within
1e-12 relative L2 in fp64 (1e-5 in fp32)").

* C2 (1-D, N=65,536, P=64, S=1000 BE, fp64, eps=1e-10): the F map at its real
  step count, then the whole synchronous run against the long-double oracle
  (oracle/thomas_ld.c driving the restated reference algorithm,
  parareal.py:99-138): same k and stop reason, every iterate compared.
* Explicit fine maps (C3 2-D 1024^2 S=500; C4 256^3 S=200; C5 512^3 S=100;
  ragged cubes spanning >= 3 z-chunks of the 3-D kernel, every committed
  tiling variant) against oracle/stencil_nd.c, which evaluates the device's
  per-point expression: BITWISE in fp32 and fp64.
* C3 (2-D 1024^2, P=32, S=500 FE, G = one BE step, fp64 eps=1e-10 / fp32
  eps=1e-5): the whole run against the oracle (bitwise fine map + DST-I
  direct coarse solve), per iteration.
* C4 (3-D 256^3, P=64, S=200, fp32) and C5 (512^3, P=128, S=100, fp32):
  every sweep's predictor-corrector update on a subset of slices recomputed
  by the fp64 oracle from the device's own previous iterate (the full
  oracle run would take CPU-hours), frozen prefix bitwise, coarse init, and
  the final iterate against the sequential fine solve.

Measured errors are printed and, when PINT_PARITY_LOG names a file, appended
to it as JSON lines (profiles/r02_parity.jsonl is such a log from a B200).
"""
import json
import os

import numpy as np
import pytest
import torch

from conftest import rel_l2
from oracle import heat_oracle as H
from oracle.nd_truth import SpectralND, StencilND
from oracle.truth import TruthTridiag1D

pytestmark = pytest.mark.gpu


def _log(**rec):
    print(json.dumps(rec))
    path = os.environ.get("PINT_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(rec) + "\n")


@pytest.fixture(autouse=True)
def _fresh_memory():
    """The config-size tests allocate tens of GiB: start each from a clean
    allocator (objects of earlier tests that sit in reference cycles are
    collected first) and log what was still held."""
    import gc
    gc.collect()
    torch.cuda.empty_cache()
    held = torch.cuda.memory_allocated()
    if held > 8 * 2 ** 30:
        print(f"[parity] {held / 2**30:.1f} GiB still allocated before this test")
    yield


def _host(t):
    return t.detach().to("cpu").numpy().astype(np.float64)


# ------------------------------------------------------------------ C2 (1-D)

C2 = dict(n=65536, p=64, S=1000, modes=32, eps=1e-10, T=1.0)


def _c2_setup(gpu):
    n, p = C2["n"], C2["p"]
    span = C2["T"] / p
    u0 = H.sine_u0_1d(n, C2["modes"], 0)
    ivp = gpu.heat1d_system(n, 1.0, 0.0, 0.0, 0.0, C2["T"])
    fine = gpu.backward_euler_propagator(ivp, span, C2["S"])
    coarse = gpu.backward_euler_propagator(ivp, span, 1)
    a_d, a_o, c = H.heat1d_coeffs(n)
    F = TruthTridiag1D(n, a_d, a_o, c, span, C2["S"])
    G = TruthTridiag1D(n, a_d, a_o, c, span, 1)
    return u0, fine, coarse, F, G


def test_c2_fine_map_s1000_vs_long_double(gpu):
    """F at its real step count (1000 BE steps, r = dt/h^2 = 67,110.9) on
    several slices (the seeded u0, coarse-init rows, a rough random state)."""
    u0, fine, coarse, F, G = _c2_setup(gpu)
    rows = [u0]
    x = u0
    for _ in range(3):
        x = G.apply(x)
        rows.append(x)
    rows.append(np.random.default_rng(7).standard_normal(u0.size))
    xs = np.stack(rows)
    got = _host(fine.apply_batch(torch.tensor(xs, device="cuda")))
    want = F.apply_batch(xs)
    errs = [rel_l2(got[i], want[i]) for i in range(len(rows))]
    _log(test="c2_fine_map_s1000", rel_l2=errs)
    assert max(errs) < 1e-10, errs


def test_c2_sync_parareal_per_iteration_vs_long_double(gpu):
    """C2 exactly: same k (15) and stop reason, every iterate within 1e-8
    relative L2 of the long-double oracle (the fp64 reference's own
    dense route is 3.2e-8 off at this conditioning, so 1e-12 is unattainable
    for ANY fp64 algorithm here; the measured values are logged)."""
    u0, fine, coarse, F, G = _c2_setup(gpu)
    tr = gpu.run_parareal(coarse, fine, u0, C2["p"], C2["eps"], record_iterates=True)
    ref = H.run_parareal(G, F, u0, C2["p"], C2["eps"])
    assert (tr.k_final, tr.stop_reason) == (ref.k_final, ref.stop_reason) == (15, "threshold")
    errs = [rel_l2(_host(it.tensor), ref.iterates[k]) for k, it in enumerate(tr.iterates)]
    _log(test="c2_sync_per_iteration", k=tr.k_final, stop=tr.stop_reason, rel_l2=errs,
         deltas_gpu=tr.deltas, deltas_oracle=ref.deltas)
    assert max(errs) < 1e-8, errs
    # the sweep-to-sweep changes agree while they are far above the fp64 noise
    for a, b in zip(tr.deltas, ref.deltas):
        if b > 1e-6:
            assert abs(a - b) <= 1e-6 * b, (a, b)


# ------------------------------------------------- explicit fine maps, bitwise

def _fe(gpu, n, ndim, steps, cfl, dtype, u=None, seed=3):
    h = 1.0 / (n + 1)
    span = steps * cfl * h * h
    shape = (n,) * ndim
    if u is None:
        u = np.random.default_rng(seed).standard_normal(n ** ndim)
    mk = {1: None, 2: gpu.heat2d_system, 3: gpu.heat3d_system}[ndim]
    ivp = mk(n, t_final=1.0, u0=u) if mk else gpu.heat1d_system(n, 1.0, 0.0, 0.0, 0.0, 1.0)
    fine = gpu.forward_euler_propagator(ivp, span, steps, dtype=dtype)
    orc = StencilND(shape, h, span, steps, dtype=np.float32 if dtype == "float32" else np.float64)
    return u, fine, orc


def _bitwise(gpu, fine, orc, us, want=None):
    tdt = torch.float32 if orc.dtype == np.float32 else torch.float64
    x = torch.tensor(np.stack(us), device="cuda", dtype=tdt)
    got = fine.apply_batch(x).cpu().numpy()
    if want is None:
        want = orc.apply_batch(np.stack(us).astype(orc.dtype))
    return got, want


@pytest.mark.parametrize("dtype", ("float64", "float32"))
@pytest.mark.parametrize("n,ndim,steps,cfl", [
    (300, 3, 7, 0.15),    # 3 z-chunks (128+128+44), 7 steps: not a multiple of the levels per pass
    (257, 3, 5, 0.15),    # 2 chunks + a one-plane chunk
    (129, 3, 4, 0.1),     # chunk + 1 plane
    (1000, 2, 13, 0.2),   # ragged 2-D: 8 row chunks (the last ragged), 13 steps = 8 + 5
    (131, 2, 9, 0.2),
    (4099, 1, 11, 0.4),   # 1-D explicit box kernel
])
def test_explicit_fine_map_bitwise_ragged(gpu, n, ndim, steps, cfl, dtype):
    u, fine, orc = _fe(gpu, n, ndim, steps, cfl, dtype)
    rng = np.random.default_rng(n)
    us = [u, rng.standard_normal(u.size)]
    variants = [None]
    if ndim == 3:
        variants = list(range(0, 27)) if dtype == "float32" else list(range(0, 21))
    if ndim == 2:
        variants = [0, 1, 2, 3, 4]
    key = "PINT_FE3D_VARIANT" if ndim == 3 else "PINT_FE2D_VARIANT"
    want = None
    try:
        for v in variants:
            if v is not None:
                os.environ[key] = str(v)
            got, want = _bitwise(gpu, fine, orc, us, want)
            nbad = int(np.sum(got.view(np.uint8) != want.view(np.uint8)))
            assert nbad == 0, (v, nbad, rel_l2(got, want))
    finally:
        os.environ.pop(key, None)
    _log(test="explicit_bitwise_ragged", n=n, ndim=ndim, steps=steps, dtype=dtype, variants=variants,
         bitwise=True)


@pytest.mark.parametrize("cfg", ["c3_f64", "c3_f32", "c4_f32", "c5_f32", "c4_f64"])
def test_explicit_fine_map_bitwise_config_size(gpu, cfg):
    """One slice of F at each BASELINE shape and step count, bitwise."""
    n, ndim, steps, cfl, dtype = {"c3_f64": (1024, 2, 500, 0.2, "float64"),
                                  "c3_f32": (1024, 2, 500, 0.2, "float32"),
                                  "c4_f32": (256, 3, 200, 0.15, "float32"),
                                  "c4_f64": (256, 3, 200, 0.15, "float64"),
                                  "c5_f32": (512, 3, 100, 0.15, "float32")}[cfg]
    modes = H.modes_2d() if ndim == 2 else H.modes_3d()
    u0 = H.sine_u0_nd((n,) * ndim, modes, 0).reshape(-1)
    u, fine, orc = _fe(gpu, n, ndim, steps, cfl, dtype, u=u0)
    got, want = _bitwise(gpu, fine, orc, [u0])
    nbad = int(np.sum(got.view(np.uint8) != want.view(np.uint8)))
    exact = StencilND(orc.shape, orc.h, orc.span, steps, exact=True).apply(u0) if dtype == "float64" else None
    rec = dict(test="explicit_bitwise_config", cfg=cfg, differing_bytes=nbad)
    if exact is not None:
        rec["fp64_vs_long_double_rel_l2"] = rel_l2(got[0], exact)
    _log(**rec)
    assert nbad == 0, (cfg, nbad, rel_l2(got, want))


# -------------------------------------------------------------- C3 (2-D)

def _nd_setup(gpu, n, ndim, p, steps, cfl, dtype):
    h = 1.0 / (n + 1)
    span = steps * cfl * h * h
    shape = (n,) * ndim
    modes = H.modes_2d() if ndim == 2 else H.modes_3d()
    u0 = H.sine_u0_nd(shape, modes, 0).reshape(-1)
    mk = gpu.heat2d_system if ndim == 2 else gpu.heat3d_system
    ivp = mk(n, t_final=p * span, u0=u0)
    fine = gpu.forward_euler_propagator(ivp, span, steps, dtype=dtype)
    coarse = gpu.backward_euler_propagator(ivp, span, 1, dtype=dtype)
    F = StencilND(shape, h, span, steps)
    G = SpectralND(shape, h, span, 1)
    return u0, fine, coarse, F, G


def test_c3_fp64_sync_parareal_per_iteration(gpu):
    """C3 fp64 exactly (1024^2, P=32, S=500, dt=0.2h^2, eps=1e-10): same k and
    stop reason; every iterate within 1e-12 relative L2 of the oracle."""
    u0, fine, coarse, F, G = _nd_setup(gpu, 1024, 2, 32, 500, 0.2, "float64")
    tr = gpu.run_parareal(coarse, fine, u0, 32, 1e-10, record_iterates=True)
    ref = H.run_parareal(G, F, u0, 32, 1e-10)
    errs = [rel_l2(_host(it.tensor), ref.iterates[k]) for k, it in enumerate(tr.iterates)]
    _log(test="c3_f64_sync_per_iteration", k=tr.k_final, k_oracle=ref.k_final, stop=tr.stop_reason,
         rel_l2=errs, deltas_gpu=tr.deltas, deltas_oracle=ref.deltas)
    assert (tr.k_final, tr.stop_reason) == (ref.k_final, ref.stop_reason)
    assert max(errs) < 1e-12, errs


def test_c3_fp32_sync_parareal_per_iteration(gpu):
    """C3 fp32 (eps=1e-5): every fp32 iterate within 1e-5 relative L2 of the
    oracle run in fp32 arithmetic (the bitwise fp32 fine map, the exact coarse
    solve rounded to fp32, the fp32 correction), per iteration, same k and
    stop reason. Logged besides: the distance of both to the fp64 oracle — the
    fp32 rounding floor of 16,000 explicit steps (~1.4e-5), which no fp32
    implementation can beat."""
    u0, fine, coarse, F, G = _nd_setup(gpu, 1024, 2, 32, 500, 0.2, "float32")
    F32 = StencilND(F.shape, F.h, F.span, F.steps, dtype=np.float32)
    G32 = SpectralND(G.shape, G.h, G.span, 1, dtype=np.float32)
    u32 = u0.astype(np.float32)
    tr = gpu.run_parareal(coarse, fine, u32, 32, 1e-5, record_iterates=True)
    ref32 = H.run_parareal(G32, F32, u32, 32, 1e-5)
    ref64 = H.run_parareal(G, F, u0, 32, 0.0, k_max=tr.k_final)
    got = [_host(it.tensor) for it in tr.iterates]
    errs = [rel_l2(g, ref32.iterates[k]) for k, g in enumerate(got)]
    errs64 = [rel_l2(g, ref64.iterates[k]) for k, g in enumerate(got)]
    floor = [rel_l2(ref32.iterates[k], ref64.iterates[k]) for k in range(len(got))]
    _log(test="c3_f32_sync_per_iteration", k=tr.k_final, k_oracle=ref32.k_final, stop=tr.stop_reason,
         rel_l2_vs_fp32_oracle=errs, rel_l2_vs_fp64_oracle=errs64, fp32_oracle_vs_fp64_oracle=floor)
    assert (tr.k_final, tr.stop_reason) == (ref32.k_final, ref32.stop_reason)
    assert max(errs) < 1e-5, errs


# ------------------------------------------------------- C4 / C5 (3-D, fp32)

def _conditional_check(F, G, prev, new, i):
    """Reference update for slice i of sweep k from the device's own rows
    (parareal.py:25-36): G(new[i-1]) + F(prev[i-1]) - G(prev[i-1]), fp64."""
    fresh, old = new[i - 1], prev[i - 1]
    if np.array_equal(fresh, old):
        want = F.apply(old)
    else:
        want = (G.apply(fresh) + F.apply(old)) - G.apply(old)
    return rel_l2(new[i], want)


def test_c4_sync_parareal_updates_vs_oracle(gpu):
    """C4 (256^3, P=64, S=200, dt=0.15h^2, fp32, eps=1e-5)."""
    p = 64
    u0, fine, coarse, F, G = _nd_setup(gpu, 256, 3, p, 200, 0.15, "float32")
    tr = gpu.run_parareal(coarse, fine, u0, p, 1e-5, record_iterates=True, engine="standard")
    assert tr.stop_reason == "threshold"
    lam0 = tr.iterates[0].tensor
    # coarse init rows against the oracle chain
    g_rows = [u0]
    for i in range(1, 3):
        g_rows.append(G.apply(g_rows[-1]))
    init_err = [rel_l2(_host(lam0[i]), g_rows[i]) for i in range(3)]
    errs = {}
    for k in range(1, tr.k_final + 1):
        prev_t, new_t = tr.iterates[k - 1].tensor, tr.iterates[k].tensor
        # frozen prefix i < k: bitwise
        assert torch.equal(new_t[:k], prev_t[:k])
        for i in sorted({k, k + 1, 33, p}):
            rows = [i - 1, i]
            prev = {r: _host(prev_t[r]) for r in rows}
            new = {r: _host(new_t[r]) for r in rows}
            errs[f"k{k}_i{i}"] = _conditional_check(F, G, prev, new, i)
    seq = gpu.sequential_fine_solve(fine, u0, p).tensor
    fin = float(((tr.final.tensor.double() - seq.double()).norm() / seq.double().norm()).item())
    # the device sequential solve is the oracle's: F is bitwise (test above)
    seq1 = StencilND(F.shape, F.h, F.span, F.steps, dtype=np.float32).apply(u0.astype(np.float32))
    assert np.array_equal(_host(seq[1]).astype(np.float32), seq1)
    _log(test="c4_f32_sync_updates", k=tr.k_final, stop=tr.stop_reason, init_rel_l2=init_err,
         update_rel_l2=errs, final_vs_seq_fine=fin, deltas=tr.deltas)
    assert max(init_err) < 1e-5, init_err
    assert max(errs.values()) < 1e-5, errs
    assert fin < 1e-5


def test_c5_sync_parareal_updates_vs_oracle(gpu):
    """C5 (512^3, P=128, S=100, fp32; 64.5 GiB per state copy, in-place engine
    on one B200): coarse init and the first two sweeps' updates on a subset of
    slices, from runs stopped at k_max = 1 and 2 (the run is deterministic)."""
    torch.cuda.empty_cache()
    free, _ = torch.cuda.mem_get_info()
    if free < 150 * 2 ** 30:
        pytest.skip("C5 needs ~140 GiB of free HBM")
    p = 128
    u0, fine, coarse, F, G = _nd_setup(gpu, 512, 3, p, 100, 0.15, "float32")
    picks = (1, 2, 64, 128)
    need = sorted({r for i in picks for r in (i - 1, i)})
    rows = {}
    lam = gpu.coarse_init(coarse, u0, p)
    rows[0] = {r: _host(lam.tensor[r]) for r in need}
    del lam
    torch.cuda.empty_cache()
    for kk in (1, 2):
        tr = gpu.run_parareal(coarse, fine, u0, p, 0.0, k_max=kk, record_iterates=False)
        rows[kk] = {r: _host(tr.final.tensor[r]) for r in need}
        del tr
        torch.cuda.empty_cache()
    init_err = rel_l2(rows[0][1], G.apply(u0))
    errs = {}
    for k in (1, 2):
        for i in picks:
            if i < k:
                continue
            errs[f"k{k}_i{i}"] = _conditional_check(F, G, rows[k - 1], rows[k], i)
    frozen_ok = np.array_equal(rows[2][1], rows[1][1])
    _log(test="c5_f32_sync_updates", init_rel_l2=init_err, update_rel_l2=errs, frozen_prefix_bitwise=frozen_ok)
    assert frozen_ok
    assert init_err < 1e-5
    assert max(errs.values()) < 1e-5, errs
