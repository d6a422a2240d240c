"""Throughput of the 2-D/3-D propagators and sync Parareal at the BASELINE
C3/C4 shapes (secondary measurements; the bench line is C2).

    python scripts/bench_configs.py [c3|c4|all] [--tol]

Per config: F batch over all slices (explicit stencil, grid-point updates/s
and HBM fraction at 2*sizeof(T) bytes/update), one coarse CG solve (time,
iterations), and optionally sync Parareal to tolerance."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2110_10762_b200 as pb  # noqa: E402
from paper_2110_10762_b200 import inputs as H  # noqa: E402  (seeded synthetic inputs)

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0

CONFIGS = {
    "c3_f64": dict(shape=(1024, 1024), p=32, steps=500, cfl=0.2, dtype="float64", eps=1e-10, rtol=1e-12),
    "c3_f32": dict(shape=(1024, 1024), p=32, steps=500, cfl=0.2, dtype="float32", eps=1e-5, rtol=1e-6),
    "c4_f32": dict(shape=(256, 256, 256), p=64, steps=200, cfl=0.15, dtype="float32", eps=1e-5, rtol=1e-6),
    # C5 is a multi-GPU configuration (P = 128, 64.5 GiB per state copy); on one
    # GPU only the fine batch of a 16-slice share is timed (no time to tolerance)
    "c5_f32": dict(shape=(512, 512, 512), p=16, steps=100, cfl=0.15, dtype="float32", eps=1e-6, rtol=1e-6,
                   fine_only=True),
}


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def run(name, cfg, tol):
    shape, p, steps = cfg["shape"], cfg["p"], cfg["steps"]
    n = shape[0]
    h = 1.0 / (n + 1)
    dt = cfg["cfl"] * h * h
    span = steps * dt
    modes = H.modes_2d() if len(shape) == 2 else H.modes_3d()
    u0 = H.sine_u0_nd(shape, modes, 0).reshape(-1)
    mk = pb.heat2d_system if len(shape) == 2 else pb.heat3d_system
    ivp = mk(n, t_final=p * span, u0=u0)
    fine = pb.forward_euler_propagator(ivp, span, steps, dtype=cfg["dtype"])
    coarse = pb.backward_euler_propagator(ivp, span, 1, dtype=cfg["dtype"], cg_rtol=cfg["rtol"])
    dim = ivp.dim
    tdt = torch.float64 if cfg["dtype"] == "float64" else torch.float32
    esz = 8 if tdt == torch.float64 else 4
    x = torch.tensor(np.tile(u0, (p, 1)), dtype=tdt, device="cuda")
    y = torch.empty_like(x)
    ms_f = timed(lambda: fine.apply_batch(x, out=y))
    upd = p * steps * dim
    out = {"config": name, "shape": shape, "slices": p, "fine_steps": steps, "dtype": cfg["dtype"],
           "fine_batch_ms": ms_f, "fine_GPt_s": upd / ms_f / 1e6,
           "fine_hbm_frac_alg": upd * 2 * esz / (ms_f * 1e-3) / 1e9 / PEAK}
    g_in = x[0:1].clone()
    g_out = torch.empty_like(g_in)
    ms_g = timed(lambda: coarse.apply_ptr(g_in.data_ptr(), g_out.data_ptr(), 1, dim), reps=2)
    cg = pb.backward_euler_propagator(ivp, span, 1, dtype=cfg["dtype"], cg_rtol=cfg["rtol"], solver="cg")
    ms_cg = timed(lambda: cg.apply_ptr(g_in.data_ptr(), g_out.data_ptr(), 1, dim), reps=2)
    out.update({"coarse_solve_ms": ms_g, "coarse_over_fine_slice": ms_g / (ms_f / p), "cg_solve_ms": ms_cg})
    if tol and not cfg.get("fine_only"):
        pb.run_parareal(coarse, fine, u0, p, cfg["eps"], k_max=1, record_iterates=False)  # warm-up (allocations)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        tr = pb.run_parareal(coarse, fine, u0, p, cfg["eps"], record_iterates=False)
        torch.cuda.synchronize()
        out.update({"time_to_tol_s": time.perf_counter() - t0, "k": tr.k_final, "stop": tr.stop_reason,
                    "epsilon": cfg["eps"]})
    print(json.dumps(out), flush=True)
    return out


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    tol = "--tol" in sys.argv
    for name, cfg in CONFIGS.items():
        if which == "all" or name.startswith(which):
            run(name, cfg, tol)
