"""Benchmark of the Parareal hot path on B200 (BASELINE.json metric
"fine-propagator grid-point updates/s (% HBM roofline); Parareal
time-to-tolerance").

Workload (BASELINE configs[1], one GPU): 1-D heat u_t = u_xx, N = 65,536
interior points, P = 64 slices, F = 1000 backward-Euler steps per slice,
G = 1 step, fp64, seeded 32-mode sine u0. One bench step is one synchronous
Parareal sweep with every slice live (k = 1): the batched fine propagation of
all 64 slices (64 x 1000 x 65,536 = 4.19e9 grid-point updates) followed by the
fused coarse chain + predictor-corrector + convergence norm, and the
8-byte delta read that drives the stop test.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 (torchrun, one rank per GPU, NCCL): weak scaling — every rank owns 64
consecutive slices of a P = 64 N chain; the coarse chain crosses ranks through
one NCCL send/recv of the 512 KiB boundary state per sweep.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_POINTS = 65536
P_LOCAL = 64
FINE_STEPS = 1000
COARSE_STEPS = 1
T_FINAL = 1.0
N_MODES = 32
METRIC = "fine-propagator grid-point updates/s"
UNIT = "GPt-updates/s"
BYTES_PER_UPDATE = 16  # one fp64 read + one fp64 write per grid-point update
FP64_INSTR_PER_UPDATE = 163 / 32  # tri1d_batch_kernel: executed DFMA+DADD+DMUL per thread-step (SASS, windowed level-2 path) / points per thread


def workload_config(n_gpus: int) -> dict:
    return {"workload": "C2: 1-D heat, N=65536, P=64 slices/GPU, F=1000 BE steps/slice, G=1 BE step, fp64; "
                        "one bench step = one sync Parareal sweep (k=1, all slices live)",
            "n_points": N_POINTS, "slices": P_LOCAL * n_gpus, "slices_per_gpu": P_LOCAL,
            "fine_steps": FINE_STEPS, "coarse_steps": COARSE_STEPS, "u0": f"seeded {N_MODES}-mode sine (seed 0)",
            "l2": "L2 flushed (256 MiB write) before every timed step",
            "parallelism": f"time-slices sharded over {n_gpus} GPU(s)"}


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clocks and throttle reasons during the timed region (NVML)."""

    def __init__(self, device: int = 0, period: float = 0.002):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.ok = False
        self.period = period

    def _run(self):
        nv = self.nv
        names = {
            getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8): "hw_slowdown",
            getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40): "hw_thermal_slowdown",
            getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20): "sw_thermal_slowdown",
            getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4): "sw_power_cap",
            getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80): "hw_power_brake_slowdown",
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in names.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self) -> dict:
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------- CPU baseline
def _cpu_worker(args):
    n, steps, reps, seed = args
    from oracle import heat_oracle as H
    a_d, a_o, c = H.heat1d_coeffs(n)
    F = H.Tridiag1D(n, a_d, a_o, c, T_FINAL / P_LOCAL * steps / FINE_STEPS, steps)
    u = H.sine_u0_1d(n, N_MODES, seed)
    t0 = time.perf_counter()
    for _ in range(reps):
        u = F.apply(u)
    return time.perf_counter() - t0, n * steps * reps


def cpu_baseline(target_s: float = 15.0) -> dict:
    """The oracle restatement of the reference's fine propagator (numpy +
    LAPACK gttrs, one tridiagonal solve per step, same coefficients) on the
    host's cores, one slice per worker process, BLAS threads = 1, sized to
    ~target_s of wall time."""
    import multiprocessing as mp
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    cores = os.cpu_count() or 1
    t, upd = _cpu_worker((N_POINTS, 50, 1, 0))
    rate1 = upd / t
    slice_s = N_POINTS * FINE_STEPS / rate1          # one full fine slice on one core
    reps = int(max(1, round(target_s / slice_s)))
    ctx = mp.get_context("fork")
    t0 = time.perf_counter()
    with ctx.Pool(cores) as pool:
        res = pool.map(_cpu_worker, [(N_POINTS, FINE_STEPS, reps, s) for s in range(cores)])
    wall = time.perf_counter() - t0
    total = sum(r[1] for r in res)
    return {"value": total / wall / 1e9, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{cores * reps} slice applications of F (1000 BE steps, N={N_POINTS}; "
                      f"oracle/heat_oracle.py Tridiag1D = LAPACK gttrs per step), {reps} per process on "
                      f"{cores} processes, {wall:.1f}s wall",
            "cpu": _cpu_model()}


def _cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ------------------------------------------------------------------- peaks
def measured_peaks() -> dict:
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


def _ncu_field(key: str, scale: float = 1.0):
    path = os.path.join(ROOT, "profiles", "ncu_fine_kernel.json")
    if os.path.exists(path):
        with open(path) as f:
            v = json.load(f).get(key)
        return None if v is None else v * scale
    return None


def ncu_traffic() -> float | None:
    """DRAM bytes per launch of the fine kernel from the committed ncu capture."""
    path = os.path.join(ROOT, "profiles", "ncu_fine_kernel.json")
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f).get("dram_bytes_per_launch")
    return None


# -------------------------------------------------------------- reference arm
def _cpu_pool(cores: int):
    import multiprocessing as mp
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    return mp.get_context("fork").Pool(cores)


def run_reference(args, rank: int, world: int) -> None:
    """The reference's fine propagation restated on the host (oracle port:
    LAPACK gttrs per backward-Euler step, the reference's coefficients), all
    host cores, one slice per process. Every step is one bounded sample of
    the C2 workload: `cores` slice applications of F (1000 steps, N = 65,536)
    run concurrently; W untimed warm-up samples, then exactly K timed ones."""
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    pool = _cpu_pool(cores)
    try:
        def sample(seed0):
            t0 = time.perf_counter()
            res = pool.map(_cpu_worker, [(N_POINTS, FINE_STEPS, 1, seed0 + s) for s in range(cores)])
            return time.perf_counter() - t0, sum(r[1] for r in res)

        for w in range(args.warmup):
            sample(1000 * (w + 1))
        secs, upd = [], 0
        for k in range(args.steps):
            t, u = sample(k)
            secs.append(t)
            upd += u
    finally:
        pool.close()
        pool.join()
    value = upd / sum(secs) / 1e9
    desc = (f"each step: {cores} concurrent slice applications of F (1000 BE steps, N={N_POINTS}; "
            f"oracle/heat_oracle.py Tridiag1D = LAPACK gttrs per step), one per process")
    cb = {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": desc, "cpu": _cpu_model()}
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": float(np.mean(secs)) * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(world), "cpu_baseline": cb,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------- our arm
def run_ours(args, rank: int, world: int) -> None:
    import torch

    import paper_2110_10762_b200 as pb
    from paper_2110_10762_b200 import distributed as dist_rt
    from paper_2110_10762_b200.inputs import sine_u0_1d
    from paper_2110_10762_b200.parareal import SyncEngine

    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
    dev = torch.cuda.current_device()
    P_glob = P_LOCAL * world
    span = T_FINAL / P_glob
    ivp = pb.heat1d_system(N_POINTS, 1.0, 0.0, 0.0, 0.0, T_FINAL)
    fine = pb.backward_euler_propagator(ivp, span, FINE_STEPS)
    coarse = pb.backward_euler_propagator(ivp, span, COARSE_STEPS)
    u0 = sine_u0_1d(N_POINTS, N_MODES, 0)  # seeded synthetic input

    if world > 1:
        eng = dist_rt.ShardedSyncEngine(coarse, fine, P_LOCAL, rank, world)
    else:
        eng = SyncEngine(coarse, fine, P_LOCAL)
    eng.init(u0)
    stream = torch.cuda.current_stream()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    peaks = measured_peaks()
    updates_per_step = P_LOCAL * FINE_STEPS * N_POINTS  # per rank

    # the timed sweep always starts from the same (coarse-initialised)
    # iterate and G(old) cache, restored outside the timed region
    base = eng.lam_a.clone()
    base_g = eng.eng.gcache.clone() if world > 1 else eng.gcache.clone()
    gcache = eng.eng.gcache if world > 1 else eng.gcache
    nxt = eng.lam_b

    def one_step(timed_fine: list | None):
        eng.lam_a.copy_(base)
        gcache.copy_(base_g)
        eng.prev = eng.lam_a
        flush.fill_(1.0)
        if world > 1:
            dist_rt.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        ef = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        eng.sweep(1, nxt, fine_done_event=ef)
        delta = eng.read_delta()
        e1.record(stream)
        torch.cuda.synchronize()
        if timed_fine is not None:
            timed_fine.append(e0.elapsed_time(ef))
        return e0.elapsed_time(e1), delta

    for _ in range(args.warmup):
        one_step(None)
    step_ms, fine_ms = [], []
    with ClockSampler(dev) as clocks:
        for _ in range(args.steps):
            ms, delta = one_step(fine_ms)
            step_ms.append(ms)
    ms_step_local = float(np.mean(step_ms))
    ms_fine = float(np.mean(fine_ms))
    ms_step = dist_rt.max_over_ranks(ms_step_local) if world > 1 else ms_step_local
    value = updates_per_step * world / (ms_step * 1e-3) / 1e9

    # end-to-end through the reference's public API with host buffers: one
    # full sweep pb.parareal_iterate (parareal.py:66-76) from a pinned host
    # iterate to a pinned host result, every step (H2D of the iterate, the
    # sweep, D2H of the new iterate inside the timed region)
    host_in = torch.from_numpy(base.cpu().numpy()).pin_memory()
    host_out = torch.empty_like(host_in).pin_memory()
    lam_host = pb.BlockVector(host_in, check_finite=False)
    e2e_ms = []
    for it in range(args.warmup + args.steps):
        flush.fill_(1.0)
        if world > 1:
            dist_rt.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if world == 1:
            res = pb.parareal_iterate(coarse, fine, lam_host, out=host_out)
        else:
            eng.lam_a.copy_(host_in, non_blocking=True)
            eng.prev = eng.lam_a
            eng.sweep(1, nxt)
            eng.read_delta()
            host_out.copy_(nxt, non_blocking=True)
        torch.cuda.synchronize()
        if it >= args.warmup:
            e2e_ms.append((time.perf_counter() - t0) * 1e3)
    if world == 1:
        assert res.tensor.data_ptr() == host_out.data_ptr()
        # the public call is one sweep of the engine: same bits as the device step
        eng.lam_a.copy_(base)
        gcache.copy_(base_g)
        eng.prev = eng.lam_a
        eng.sweep(1, nxt)
        same = bool(torch.equal(nxt.cpu(), host_out))
        eng.prev = eng.lam_a
    ms_e2e = float(np.mean(e2e_ms))
    if world > 1:
        ms_e2e = dist_rt.max_over_ranks(ms_e2e)
    e2e_value = updates_per_step * world / (ms_e2e * 1e-3) / 1e9
    nbytes = host_in.numel() * host_in.element_size()

    achieved = updates_per_step * BYTES_PER_UPDATE / (ms_fine * 1e-3) / 1e9
    traffic = ncu_traffic()
    info = fine.info
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": workload_config(world),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": achieved / peaks["hbm_gbs"], "traffic": traffic,
                     "kernel": "tri1d_batch_kernel (F over all slices)",
                     "algorithmic_bytes_per_launch": updates_per_step * BYTES_PER_UPDATE,
                     "fine_kernel_ms": ms_fine, "peak_source": peaks["source"],
                     "note": "algorithmic bytes = 16 B per grid-point update (SURVEY 8d); the slice state "
                             "stays in registers for all 1000 steps, so frac > 1 is expected and `traffic` "
                             "(ncu DRAM bytes/launch) is ~2 state copies"},
        "compute": {"bound": "fp64 pipe + latency (state is register-resident; HBM is not the limit)",
                    "fp64_pipe_frac_ncu": _ncu_field("fp64_pipe_pct_of_peak", 0.01),
                    # live: this run's F rate x the kernel's FP64 instructions per update
                    # (SASS: 144 DFMA + 34 DMUL + 6 DADD per 32-point thread-step)
                    "fp64_instr_per_update": FP64_INSTR_PER_UPDATE,
                    "fp64_frac_live": updates_per_step / (ms_fine * 1e-3) * FP64_INSTR_PER_UPDATE / 17.95e12,
                    "fp64_peak_instr_s_measured": 17.95e12,
                    "source": "profiles/ncu_fine_kernel.json, profiles/r02_ncu_summary.md, scripts/microbench.cu"},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
                "ms_per_step": ms_e2e,
                "call": "paper_2110_10762_b200.parareal_iterate(coarse, fine, BlockVector(pinned host iterate), "
                        "out=pinned host) — the reference's parareal_iterate, parareal.py:66-76",
                "equals_device_sweep_bitwise": same if world == 1 else None},
        "gpu_launches": None,
        "clocks": clocks.summary(),
        "layout": {"threads_per_slice": info.threads_per_slice, "points_per_thread": info.points_per_thread,
                   "ctas_per_slice": info.batch_cluster},
        "delta_first_sweep": delta,
    }
    line["gpu_launches"] = args.steps * (eng.launches_per_sweep(1) if world == 1 else eng.launches_per_sweep())
    if world > 1 and args.time_to_tol:
        line["multi_gpu"] = multi_gpu_time_to_tolerance(rank, world)
    if rank == 0:
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline()
        if args.time_to_tol and world == 1:
            line["time_to_tolerance"] = time_to_tolerance(coarse, fine, u0, P_LOCAL)
        if args.configs and world == 1:
            line["configs"] = nd_configs(not args.no_cpu_baseline)
            if not args.no_cpu_baseline:
                line["cpu_time_to_tolerance"] = cpu_time_to_tolerance()
        print(json.dumps(line), flush=True)


def time_to_tolerance(coarse, fine, u0, p: int, eps: float = 1e-10) -> dict:
    """Sync Parareal to eps (wall clock after device sync), the
    device async runtime to the same eps, both checked against the
    sequential fine solve on the GPU, plus the reference cost model fed with
    the measured C_F / C_G."""
    import torch

    import paper_2110_10762_b200 as pb
    pb.run_parareal(coarse, fine, u0, p, eps, k_max=2, record_iterates=False)  # warm-up (allocations)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tr = pb.run_parareal(coarse, fine, u0, p, eps, record_iterates=False)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    seq = pb.sequential_fine_solve(fine, u0, p).tensor

    def err(x):
        d = (x - seq).abs().max().item()
        return {"max_abs_vs_seq_fine": d, "rel_l2_vs_seq_fine": ((x - seq).norm() / seq.norm()).item()}

    out = {"seconds": wall, "k": tr.k_final, "stop_reason": tr.stop_reason, "epsilon": eps,
           "last_delta": tr.deltas[-1], **err(tr.final.tensor)}
    kappa = None
    try:
        try:  # warm-up: first launch of the persistent kernel (module load, attributes), not timed
            pb.run_async_parareal_device(coarse, fine, u0, p, eps, max_events=2 * p)
        except pb.HorizonExhausted:
            pass
        torch.cuda.synchronize()
        res = pb.run_async_parareal_device(coarse, fine, u0, p, eps, record_trace=True)
        kappa = res.kappa
        out["async_device"] = {"seconds": res.wall_s, "kappa": res.kappa, "activations": res.activations,
                               "stop_reason": res.stop_reason, "concurrent_clusters": res.concurrent_clusters,
                               **err(res.final.tensor),
                               "audit": pb.audit_device_trace(res.trace_records, p, res.per_component_counts)}
    except Exception as exc:  # reported, never silently replaced
        out["async_device"] = {"error": f"{type(exc).__name__}: {exc}"}
    costs = pb.measure_costs(coarse, fine, p)
    out["cost_model"] = pb.model_report(costs, p, k=tr.k_final, kappa=kappa, measured_sync_s=wall)
    rep = pb.contraction_factors(coarse, fine, p)  # matrix-free spectral norms at full size
    out["contraction"] = rep.to_dict() | {"sync_check": list(pb.sync_convergence_check(rep)),
                                           "async_check": list(pb.async_convergence_check(rep))}
    return out


# ------------------------------------------------- 2-D / 3-D configurations
ND_CONFIGS = {
    "c3_f64": dict(shape=(1024, 1024), p=32, steps=500, cfl=0.2, dtype="float64", eps=1e-10),
    "c3_f32": dict(shape=(1024, 1024), p=32, steps=500, cfl=0.2, dtype="float32", eps=1e-5),
    "c4_f32": dict(shape=(256, 256, 256), p=64, steps=200, cfl=0.15, dtype="float32", eps=1e-5, async_mp=True),
    # C5 runs at 2/4/8 GPUs in BASELINE (P = 128, 64.5 GiB per state copy); on
    # one GPU its per-GPU share (16 slices at 8 GPUs) is timed for F
    "c5_f32_share": dict(shape=(512, 512, 512), p=16, steps=100, cfl=0.15, dtype="float32", fine_only=True),
}


def _sine_u0_device(shape, seed=0):
    """inputs.sine_u0_nd built on the GPU with numpy's sines and the same
    elementwise operation order (same bits, no 1 GB host temporaries)."""
    import torch

    from paper_2110_10762_b200.inputs import interior_grid, modes_2d, modes_3d
    modes = modes_2d() if len(shape) == 2 else modes_3d()
    amp = np.random.default_rng(seed).standard_normal(len(modes))
    axes = [interior_grid(n) for n in shape]
    out = torch.zeros(shape, dtype=torch.float64, device="cuda")
    for a, ks in zip(amp, modes):
        term = torch.ones(shape, dtype=torch.float64, device="cuda")
        for d, k in enumerate(ks):
            bshape = [1] * len(shape)
            bshape[d] = shape[d]
            term = term * torch.from_numpy(np.sin(k * np.pi * axes[d])).to("cuda").reshape(bshape)
        out = out + float(a) * term
    return out.reshape(-1)


def _world1():
    """A one-rank process group for the multi-process runtime (N = 1)."""
    import socket

    import torch.distributed as dist
    if dist.is_initialized():
        return False
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1)
    return True


def _cpu_port_fine(shape, steps, cfl, dtype, target_s=2.0) -> dict:
    """The oracle restatement of the explicit fine map (oracle/stencil_nd.c,
    OpenMP over the host cores) timed on one slice of the configuration."""
    from oracle.nd_truth import StencilND
    n = shape[0]
    h = 1.0 / (n + 1)
    st = StencilND(shape, h, steps * cfl * h * h, steps, dtype=np.float32 if dtype == "float32" else np.float64)
    u = np.random.default_rng(0).standard_normal(int(np.prod(shape)))
    t0 = time.perf_counter()
    st.apply(u)
    t1 = time.perf_counter() - t0
    reps = max(1, min(8, int(target_s / max(t1, 1e-3))))
    t0 = time.perf_counter()
    for _ in range(reps):
        st.apply(u)
    t = (time.perf_counter() - t0) / reps
    upd = int(np.prod(shape)) * steps
    return {"value": upd / t / 1e9, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
            "sample": f"{reps + 1} slice applications of F ({steps} FE steps, {'x'.join(map(str, shape))}, {dtype}; "
                      f"oracle/stencil_nd.c, OpenMP over {os.cpu_count()} threads)"}


def _nd_config(name: str, cfg: dict, with_cpu: bool) -> dict:
    import torch

    import paper_2110_10762_b200 as pb
    shape, p, steps = cfg["shape"], cfg["p"], cfg["steps"]
    n = shape[0]
    h = 1.0 / (n + 1)
    span = steps * cfg["cfl"] * h * h
    u0 = _sine_u0_device(shape)
    mk = pb.heat2d_system if len(shape) == 2 else pb.heat3d_system
    ivp = mk(n, t_final=p * span, u0=None)
    fine = pb.forward_euler_propagator(ivp, span, steps, dtype=cfg["dtype"])
    coarse = pb.backward_euler_propagator(ivp, span, 1, dtype=cfg["dtype"])
    dim = ivp.dim
    esz = 8 if cfg["dtype"] == "float64" else 4
    x = u0.to(fine.dtype).reshape(1, -1).repeat(p, 1)
    y = torch.empty_like(x)
    out = {"workload": f"{'x'.join(map(str, shape))}, P={p}, F={steps} FE steps (dt={cfg['cfl']}h^2), "
                       f"G=1 BE step (direct sine-transform solve), {cfg['dtype']}",
           "l2": f"state {x.numel() * esz / 2**20:.0f} MiB per F batch (larger than the 126 MB L2)"}
    fine.apply_batch(x, out=y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 3
    with ClockSampler(torch.cuda.current_device()) as clk:
        e0.record()
        for _ in range(reps):
            fine.apply_batch(x, out=y)
        e1.record()
        torch.cuda.synchronize()
    ms_f = e0.elapsed_time(e1) / reps
    upd = p * steps * dim
    peak = measured_peaks()["hbm_gbs"]
    out.update({"fine_batch_ms": ms_f, "fine_GPt_s": upd / ms_f / 1e6,
                "fine_roofline": {"bound": "hbm", "achieved": upd * 2 * esz / (ms_f * 1e-3) / 1e9, "peak": peak,
                                  "unit": "GB/s", "frac": upd * 2 * esz / (ms_f * 1e-3) / 1e9 / peak,
                                  "note": f"algorithmic bytes 2*{esz} B per update; S levels per HBM pass"},
                "clocks": clk.summary()})
    g_in, g_out = x[0:1].clone(), torch.empty_like(x[0:1])
    coarse.apply_ptr(g_in.data_ptr(), g_out.data_ptr(), 1, dim)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(3):
        coarse.apply_ptr(g_in.data_ptr(), g_out.data_ptr(), 1, dim)
    e1.record()
    torch.cuda.synchronize()
    out["coarse_solve_ms"] = e0.elapsed_time(e1) / 3
    del x, y
    if not cfg.get("fine_only"):
        u0h = u0.to(fine.dtype)
        pb.run_parareal(coarse, fine, u0h, p, cfg["eps"], k_max=1, record_iterates=False)  # warm-up
        torch.cuda.synchronize()
        with ClockSampler(torch.cuda.current_device()) as clk:
            t0 = time.perf_counter()
            tr = pb.run_parareal(coarse, fine, u0h, p, cfg["eps"], record_iterates=False)
            torch.cuda.synchronize()
            wall = time.perf_counter() - t0
        seq = pb.sequential_fine_solve(fine, u0h, p).tensor
        fin = tr.final.tensor
        out["sync_time_to_tolerance"] = {
            "seconds": wall, "k": tr.k_final, "stop_reason": tr.stop_reason, "epsilon": cfg["eps"],
            "rel_l2_vs_seq_fine": float(((fin.double() - seq.double()).norm() / seq.double().norm()).item()),
            "clocks": clk.summary()}
        del tr, fin
        if cfg.get("async_mp"):
            from paper_2110_10762_b200.async_mp import run_async_parareal_mp
            made = _world1()
            try:
                run_async_parareal_mp(coarse, fine, u0h, p, cfg["eps"], lanes=2, max_events=64)  # warm-up
            except pb.HorizonExhausted:
                pass
            try:
                res = run_async_parareal_mp(coarse, fine, u0h, p, cfg["eps"], lanes=2, gather=True)
                out["async_time_to_tolerance_1gpu"] = {
                    "seconds": res.wall_s, "kappa": res.kappa, "activations": res.activations,
                    "stop_reason": res.stop_reason, "runtime": "async_mp (one rank, 2 lanes)",
                    "rel_l2_vs_seq_fine": float(((res.final.double() - seq.double()).norm()
                                                 / seq.double().norm()).item())}
            except Exception as exc:  # reported, never silently replaced
                out["async_time_to_tolerance_1gpu"] = {"error": f"{type(exc).__name__}: {exc}"}
            finally:
                if made:
                    import torch.distributed as dist
                    dist.destroy_process_group()
        del seq
    torch.cuda.empty_cache()
    if with_cpu:
        out["cpu_port_fine"] = _cpu_port_fine(shape, steps, cfg["cfl"], cfg["dtype"])
    return out


def nd_configs(with_cpu: bool) -> dict:
    out = {}
    for name, cfg in ND_CONFIGS.items():
        try:
            out[name] = _nd_config(name, cfg, with_cpu)
        except Exception as exc:  # reported, never silently replaced
            out[name] = {"error": f"{type(exc).__name__}: {exc}"}
    return out


def cpu_time_to_tolerance() -> dict:
    """The oracle restatement of the reference's synchronous run
    (parareal.py:99-138) on the host: C1 (LAPACK step maps, the reference's
    own scale) and C3 fp64 (oracle/stencil_nd.c fine map over all cores,
    exact sine-transform coarse solve)."""
    from oracle import heat_oracle as H
    from oracle.nd_truth import SpectralND, StencilND
    out = {"cores": os.cpu_count(), "kind": "port"}
    n, p = 1024, 16
    a_d, a_o, c = H.heat1d_coeffs(n)
    F = H.Tridiag1D(n, a_d, a_o, c, 1.0 / p, 100)
    G = H.Tridiag1D(n, a_d, a_o, c, 1.0 / p, 1)
    u0 = H.sine_u0_1d(n, 8, 0)
    t0 = time.perf_counter()
    tr = H.run_parareal(G, F, u0, p, 1e-10)
    out["c1"] = {"seconds": time.perf_counter() - t0, "k": tr.k_final, "stop_reason": tr.stop_reason}
    n, p, steps = 1024, 32, 500
    h = 1.0 / (n + 1)
    span = steps * 0.2 * h * h
    u0 = H.sine_u0_nd((n, n), H.modes_2d(), 0).reshape(-1)
    t0 = time.perf_counter()
    tr = H.run_parareal(SpectralND((n, n), h, span), StencilND((n, n), h, span, steps), u0, p, 1e-10)
    out["c3_f64"] = {"seconds": time.perf_counter() - t0, "k": tr.k_final, "stop_reason": tr.stop_reason}
    return out


def multi_gpu_time_to_tolerance(rank: int, world: int) -> dict:
    """At N ranks: the 1-D device async runtime across GPUs (C2 slices split
    over the ranks, P2P mailbox pushes, on-device stop) and the multi-process
    runtime of whole-GPU activations at C4 (P = 64 split over the ranks)."""
    import torch

    import paper_2110_10762_b200 as pb
    from paper_2110_10762_b200 import distributed as dist_rt
    from paper_2110_10762_b200.async_mp import run_async_parareal_mp
    from paper_2110_10762_b200.inputs import sine_u0_1d
    out = {}
    try:
        ivp = pb.heat1d_system(N_POINTS, 1.0, 0.0, 0.0, 0.0, T_FINAL)
        fine = pb.backward_euler_propagator(ivp, T_FINAL / P_LOCAL, FINE_STEPS)
        coarse = pb.backward_euler_propagator(ivp, T_FINAL / P_LOCAL, 1)
        u0 = sine_u0_1d(N_POINTS, N_MODES, 0)
        r = dist_rt.run_async_parareal_distributed(coarse, fine, u0, P_LOCAL, 1e-10, gather=False, max_events=20_000)
        out["c2_async_1d"] = {"seconds": r["wall_s"], "kappa": r["kappa"], "activations": r["activations"],
                              "stop_reason": r["stop_reason"], "slices": P_LOCAL, "n_gpus": world}
    except Exception as exc:
        out["c2_async_1d"] = {"error": f"{type(exc).__name__}: {exc}"}
    try:
        cfg = ND_CONFIGS["c4_f32"]
        shape, p, steps = cfg["shape"], cfg["p"], cfg["steps"]
        h = 1.0 / (shape[0] + 1)
        span = steps * cfg["cfl"] * h * h
        ivp = pb.heat3d_system(shape[0], t_final=p * span, u0=None)
        fine = pb.forward_euler_propagator(ivp, span, steps, dtype="float32")
        coarse = pb.backward_euler_propagator(ivp, span, 1, dtype="float32")
        u0 = _sine_u0_device(shape).to(torch.float32)
        r = run_async_parareal_mp(coarse, fine, u0, p, cfg["eps"], lanes=2, max_events=20_000, timeout_s=120.0)
        out["c4_async_nd"] = {"seconds": r.wall_s, "kappa": r.kappa, "activations": r.activations,
                              "stop_reason": r.stop_reason, "slices": p, "n_gpus": world}
    except Exception as exc:
        out["c4_async_nd"] = {"error": f"{type(exc).__name__}: {exc}"}
    return out


def dry_run(rank: int, world: int) -> None:
    """The rank layout of an N-GPU run without GPU work (gloo): which slices
    every rank owns in the weak-scaling sync bench and in the async runs."""
    import torch.distributed as dist

    from paper_2110_10762_b200.distributed import async_partition
    if world > 1:
        dist.init_process_group("gloo")
    info = {"rank": rank, "local_rank": int(os.environ.get("LOCAL_RANK", 0)), "pid": os.getpid()}
    ranks = [None] * world
    if world > 1:
        dist.all_gather_object(ranks, info)
        dist.destroy_process_group()
    else:
        ranks = [info]
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "ranks": ranks,
                          "sync_c2_slices": [[r * P_LOCAL + 1, (r + 1) * P_LOCAL] for r in range(world)],
                          "async_c2_partition": async_partition(P_LOCAL, world),
                          "async_c4_partition": async_partition(ND_CONFIGS["c4_f32"]["p"], world)}), flush=True)


def _launch_ranks(n: int, check_devices: bool = True) -> int:
    """Re-run this command under torchrun, one rank per GPU (127.0.0.1)."""
    import socket
    import subprocess

    import torch
    have = torch.cuda.device_count()
    if check_devices and have < n:
        sys.stderr.write(f"bench.py: --gpus {n} requested but only {have} CUDA device(s) are visible\n")
        return 2
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--time-to-tol", action="store_true", default=True,
                    help="sync + device-async time to tolerance, cost model, contraction factors (default on)")
    ap.add_argument("--no-time-to-tol", dest="time_to_tol", action="store_false")
    ap.add_argument("--configs", action="store_true", default=True,
                    help="C3/C4/C5 lines (2-D/3-D fine throughput, time to tolerance, CPU port) (default on)")
    ap.add_argument("--no-configs", dest="configs", action="store_false")
    ap.add_argument("--dry-run", action="store_true",
                    help="launch the N ranks (gloo, no GPU work) and print the rank layout")
    args = ap.parse_args()
    if args.gpus < 1:
        raise SystemExit("--gpus must be >= 1")
    world_env = os.environ.get("WORLD_SIZE")
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        # host-only arm: rank 0 measures, the other ranks exit without work
        run_reference(args, rank, int(world_env) if world_env else args.gpus)
        return
    if world_env is None and args.gpus > 1:
        sys.exit(_launch_ranks(args.gpus, check_devices=not args.dry_run))
    world = int(world_env) if world_env else 1
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.dry_run:
        dry_run(rank, world)
        return
    if world > 1:
        from paper_2110_10762_b200 import distributed as dist_rt
        dist_rt.init_process_group()
    run_ours(args, rank, world)
    if world > 1:
        from paper_2110_10762_b200 import distributed as dist_rt
        dist_rt.destroy()


if __name__ == "__main__":
    main()
