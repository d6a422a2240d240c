"""Asynchronous Parareal (reference: pintlab/async_parareal.py:1-84).

Worker i owns interface state i. On activation it reads its predecessor
twice: slot 1 (FRESH) takes the freshest version the schedule lets it see,
slot 2 (REMEMBERED) replays the version it consumed through slot 1 at its
previous activation (default version 0 = the coarse initial value). When the
two readings coincide bitwise the update collapses to F(remembered), which
drives finite termination.

``run_async_parareal`` keeps the reference's deterministic event semantics
(same seeds -> same activation order, staleness draws, reads and values) with
the state, the version-stamped retention buffers and every evaluation
(F, G, the equality test, the correction and the delta) on the GPU.
"""
from __future__ import annotations

import ctypes
import hashlib
from collections import deque

import numpy as np
import torch

from . import _device, _native
from .async_engine import (
    STOP_PREDICATE,
    STOP_QUIESCENCE,
    POLICY_ROUND_ROBIN,
    AsyncMapping,
    AsyncSchedule,
    AsyncTrace,
    EngineView,
    ScheduleDriver,
    UpdateRecord,
)
from .errors import HorizonExhausted
from .linalg import BlockVector
from .parareal import _coarse_init_into, _u0_tensor, correct_into, parareal_update

FRESH_SLOT = 1
REMEMBERED_SLOT = 2
PERSISTENT_SLOTS = {REMEMBERED_SLOT: FRESH_SLOT}
SNAPSHOT_LIMIT_BYTES = 1 << 30


def async_parareal_mapping(coarse, fine, p: int) -> AsyncMapping:
    """Two-slot mapping whose synchronous sweep is classic Parareal
    (async_parareal.py:24-49): component i reads (i-1, FRESH) and
    (i-1, REMEMBERED); REMEMBERED replays FRESH's previous reading. The
    evaluation is ``parareal_update`` on the GPU."""
    if p < 1:
        raise ValueError(f"need p >= 1 subintervals, got {p}")

    def eval_fn(i: int, read_values: dict):
        return parareal_update(coarse, fine, read_values[(i - 1, FRESH_SLOT)], read_values[(i - 1, REMEMBERED_SLOT)])

    read_set = {i: ((i - 1, FRESH_SLOT), (i - 1, REMEMBERED_SLOT)) for i in range(1, p + 1)}
    return AsyncMapping(n_updatable=p, arity=2, eval_fn=eval_fn, read_set=read_set,
                        persistent_slots=dict(PERSISTENT_SLOTS), propagators=(coarse, fine))


def simulate_async(mapping: AsyncMapping, init, schedule: AsyncSchedule, stop=None,
                   record_snapshots: bool = True) -> AsyncTrace:
    """Event loop of async_engine.py:238-365 for the Parareal mapping: runs
    ``simulate_parareal_async`` (GPU state, retention buffers and evaluations).
    ``init`` is a BlockVector / array / tensor with p + 1 rows."""
    from .errors import DimensionError
    if mapping.propagators is None:
        raise NotImplementedError("simulate_async runs the Parareal mapping (async_parareal_mapping); "
                                  "other fixed-point mappings are outside this build's hot path")
    coarse, fine = mapping.propagators
    p = mapping.n_updatable
    t = init.tensor if isinstance(init, BlockVector) else init
    t, _ = _device.as_device_tensor(t, coarse.device, coarse.dtype)
    t = t.reshape(t.shape[0], -1) if t.dim() > 1 else t.reshape(1, -1)
    if t.shape[0] != p + 1:
        raise DimensionError(f"init has {t.shape[0]} blocks, expected {p + 1}")
    if t.shape[1] != coarse.dim:
        raise DimensionError(f"init blocks have dim {t.shape[1]}, expected {coarse.dim}")
    return simulate_parareal_async(coarse, fine, t.contiguous().clone(), schedule, stop=stop,
                                   record_snapshots=record_snapshots)


def async_stop_check(worker_deltas, epsilon: float, drained: bool) -> bool:
    """Every worker's last change strictly below epsilon and no newer version
    still unseen by its consumer (async_parareal.py:52-58)."""
    if epsilon <= 0.0:
        raise ValueError(f"epsilon must be positive, got {epsilon}")
    deltas = np.asarray(worker_deltas, dtype=float)
    return bool(drained and float(np.max(deltas)) < epsilon)


class _Evaluator:
    """parareal_update on device buffers with a device-side F-only flag."""

    def __init__(self, coarse, fine):
        self.coarse, self.fine = coarse, fine
        dev = f"cuda:{fine.device}"
        n = fine.dim
        self.gf = torch.empty(1, n, dtype=fine.dtype, device=dev)
        self.go = torch.empty_like(self.gf)
        self.fo = torch.empty_like(self.gf)
        self.eq = torch.zeros(1, dtype=torch.uint8, device=dev)
        self.delta = torch.zeros(1, dtype=torch.float64, device=dev)
        self.flag = torch.zeros(1, dtype=torch.int32, device=dev)
        self.lib = _native.load_library()
        self.dt = _native.PINT_F64 if fine.dtype == torch.float64 else _native.PINT_F32

    def __call__(self, fresh: torch.Tensor, rem: torch.Tensor, same_version: bool, prev: torch.Tensor,
                 out: torch.Tensor) -> None:
        n = self.fine.dim
        self.fine.apply_ptr(rem.data_ptr(), self.fo.data_ptr(), 1, n)
        if same_version:
            self.eq.fill_(1)
        else:
            s = ctypes.c_void_p(_device.stream_ptr(self.fine.device))
            rc = self.lib.pint_equal_flag(self.fine._ctx.handle, self.dt, n, ctypes.c_void_p(fresh.data_ptr()),
                                          ctypes.c_void_p(rem.data_ptr()), ctypes.c_void_p(self.eq.data_ptr()), s)
            _native.check(rc, self.fine._ctx.handle, "pint_equal_flag")
            self.coarse.apply_ptr(fresh.data_ptr(), self.gf.data_ptr(), 1, n)
            self.coarse.apply_ptr(rem.data_ptr(), self.go.data_ptr(), 1, n)
        correct_into(self.fine, self.gf, self.fo, self.go, prev.reshape(1, -1), out.reshape(1, -1), self.eq,
                     self.delta, self.flag, 1)


def simulate_parareal_async(coarse, fine, init: torch.Tensor, schedule: AsyncSchedule, stop=None,
                            record_snapshots: bool = True, record_digests: bool | None = None) -> AsyncTrace:
    """Event loop of async_engine.py:238-365 specialised to the two-slot
    Parareal mapping (async_parareal.py:24-49), evaluated on the GPU."""
    p = init.shape[0] - 1
    n = init.shape[1]
    bound = schedule.delay_bound
    window = schedule.window(p)
    driver = ScheduleDriver(schedule, p)
    esz = init.element_size()
    if record_snapshots and (p + 1) * n * esz * min(schedule.max_events, 4096) > SNAPSHOT_LIMIT_BYTES:
        record_snapshots = False
    if record_digests is None:
        record_digests = n <= 4096
    state = init.clone()
    versions = [0] * (p + 1)
    buffers = [deque([(0, init[i].clone())], maxlen=bound + 1) for i in range(p + 1)]
    remembered: dict = {}
    consumed: dict = {}
    last = np.full(p + 1, np.inf)
    last[0] = 0.0
    counts = np.zeros(p + 1, dtype=int)
    events, snapshots = [], []
    zero_streak = 0
    quiescent_streak = (bound + 3) * window
    stop_reason = None
    ev = _Evaluator(coarse, fine)
    for k in range(schedule.max_events):
        comp = driver.next_component(k)
        src = comp - 1
        staleness = driver.sample_staleness()
        vf = max(versions[src] - staleness, 0)
        buf = buffers[src]
        idx = len(buf) - 1 - (buf[-1][0] - vf)
        if idx < 0:
            raise KeyError(f"version {vf} already evicted from the retention buffer")
        fresh = buf[idx][1]
        vr, rem = remembered.get(comp, (0, init[src]))
        consumed[comp] = vf
        new = torch.empty_like(state[comp])
        ev(fresh, rem, vr == vf, state[comp], new)
        delta = float(ev.delta.item())
        if bool(ev.flag.item()):
            raise ValueError("block entries must be finite")
        state[comp].copy_(new)
        versions[comp] += 1
        buffers[comp].append((versions[comp], new))
        counts[comp] += 1
        last[comp] = delta
        remembered[comp] = (vf, fresh)
        digest = hashlib.sha256(_device.to_host(new).tobytes()).hexdigest()[:16] if record_digests else ""
        events.append(UpdateRecord(k_global=k, component=comp,
                                   reads=((src, FRESH_SLOT, vf), (src, REMEMBERED_SLOT, vr)),
                                   digest=digest, delta=delta))
        if record_snapshots:
            snapshots.append(BlockVector(state.clone(), check_finite=False))
        zero_streak = zero_streak + 1 if delta == 0.0 else 0
        if zero_streak >= quiescent_streak:
            stop_reason = STOP_QUIESCENCE
            break
        if stop is not None:
            drained = all(consumed.get(i) == versions[i - 1] for i in range(1, p + 1))
            if stop(EngineView(k, BlockVector(state, check_finite=False), last.copy(), drained)):
                stop_reason = STOP_PREDICATE
                break
    trace = AsyncTrace(events=events, snapshots=snapshots, initial=BlockVector(init.clone(), check_finite=False),
                       per_component_counts=counts, stop_event=len(events) - 1, stop_reason=stop_reason or "",
                       schedule=schedule, n_updatable=p, persistent_slots=dict(PERSISTENT_SLOTS),
                       final=BlockVector(state.clone(), check_finite=False))
    if stop_reason is None:
        raise HorizonExhausted(f"no stop condition met within {schedule.max_events} events", trace)
    return trace


def run_async_parareal(coarse, fine, u0, p: int, schedule: AsyncSchedule, epsilon: float | None = None,
                       record_snapshots: bool = True) -> AsyncTrace:
    """Asynchronous iteration from the coarse initialization
    (async_parareal.py:61-84). With epsilon, stops once all per-worker last
    changes are strictly below it and the read edges are drained; with
    epsilon None it runs to exact quiescence."""
    if p < 1:
        raise ValueError(f"need p >= 1 subintervals, got {p}")
    init = torch.empty(p + 1, coarse.dim, dtype=coarse.dtype, device=f"cuda:{coarse.device}")
    init[0] = _u0_tensor(coarse, u0)
    _coarse_init_into(coarse, init, p, None)
    stop = None
    if epsilon is not None:
        eps = float(epsilon)

        def stop(view: EngineView) -> bool:
            return async_stop_check(view.last_deltas[1:], eps, view.drained)

    return simulate_parareal_async(coarse, fine, init, schedule, stop=stop, record_snapshots=record_snapshots)


TRACE_FIELDS = ("slice", "fresh_version", "remembered_version", "f_only", "delta_bits", "t_start_ns",
                "t_publish_ns", "cluster")


class DeviceAsyncResult:
    """Outcome of ``run_async_parareal_device``. With ``record_trace=True``
    ``trace_records`` holds one int64 row per published activation, in
    publish order (columns ``TRACE_FIELDS``)."""

    def __init__(self, final, counts, info, wall_s, trace_records=None, p=None, seed=0):
        self.final = final
        self.per_component_counts = counts
        self.activations = int(info[0])
        self.stop_reason = {1: "converged", 2: "max_events"}.get(int(info[1]), "unknown")
        self.retries = int(info[3])
        self.concurrent_clusters = int(info[4])
        self.wall_s = wall_s
        self.trace_records = trace_records
        self.p = p
        self.seed = seed

    @property
    def kappa(self) -> int:
        """Busiest worker's activation count (the paper's kappa(k~))."""
        return int(np.max(self.per_component_counts[1:])) if len(self.per_component_counts) > 1 else 0

    def to_async_trace(self) -> AsyncTrace:
        """The device run as the reference's trace type (async_engine.py:122-190):
        event k = k-th publish; component i read (i-1, FRESH, v) and
        (i-1, REMEMBERED, v_rem). Values are not snapshotted (digest "")."""
        if self.trace_records is None:
            raise ValueError("run with record_trace=True to get a trace")
        return device_records_to_trace(self.trace_records, self.p, self.per_component_counts, self.final,
                                       self.stop_reason, self.seed)


def device_records_to_trace(records: np.ndarray, p: int, counts, final, stop_reason: str, seed: int = 0):
    events = []
    for k, r in enumerate(np.asarray(records, dtype=np.int64)):
        i, vf, vr, fonly, dbits = int(r[0]), int(r[1]), int(r[2]), int(r[3]), int(r[4])
        delta = float(np.array([dbits], dtype=np.int64).view(np.float64)[0])
        events.append(UpdateRecord(k_global=k, component=i,
                                   reads=((i - 1, FRESH_SLOT, vf), (i - 1, REMEMBERED_SLOT, vr)),
                                   digest="", delta=delta, frozen=False))
    # the device ticket queue claims slices in round-robin order; staleness is whatever the hardware produced
    sched = AsyncSchedule(seed=int(seed), delay_bound=max(1, len(events)), policy=POLICY_ROUND_ROBIN,
                          max_events=max(1, len(events)))
    return AsyncTrace(events=events, snapshots=[], initial=None, per_component_counts=np.asarray(counts),
                      stop_event=len(events) - 1, stop_reason=stop_reason, schedule=sched, n_updatable=p,
                      persistent_slots=dict(PERSISTENT_SLOTS), final=final)


def audit_device_trace(records: np.ndarray, p: int, counts=None) -> dict:
    """Race audit of a device async run: replays the publish
    order through ``validate_schedule`` with an unbounded delay (so only a
    read of a not-yet-published version counts as a staleness violation —
    causality) and checks remembered-slot provenance; reports the observed
    staleness (versions behind the newest at publish time), the per-slice
    publish counts against ``counts``, and the peak number of activations in
    flight at once (from the globaltimer stamps)."""
    from .async_engine import validate_schedule

    rec = np.asarray(records, dtype=np.int64).reshape(-1, len(TRACE_FIELDS))
    n = len(rec)
    trace = device_records_to_trace(rec, p, counts if counts is not None else np.zeros(p + 1), None, "")
    val = validate_schedule(trace, delay_bound=n + 1, window=n + 1)
    versions = np.zeros(p + 1, dtype=np.int64)
    stale = []
    for r in rec:
        i, vf = int(r[0]), int(r[1])
        stale.append(int(versions[i - 1] - vf) if i > 1 else 0)
        versions[i] += 1
    pub = np.bincount(rec[:, 0], minlength=p + 1) if n else np.zeros(p + 1, dtype=np.int64)
    # peak concurrency: sweep over [t_start, t_publish] intervals
    ev = sorted([(int(t0), 1) for t0 in rec[:, 5]] + [(int(t1), -1) for t1 in rec[:, 6]],
                key=lambda e: (e[0], e[1]))
    cur = peak = 0
    for _, d in ev:
        cur += d
        peak = max(peak, cur)
    out = {"events": n, "causality_violations": len(val.staleness_violations),
           "provenance_violations": len(val.provenance_violations), "max_staleness": int(max(stale, default=0)),
           "mean_staleness": float(np.mean(stale)) if stale else 0.0, "peak_in_flight": int(peak),
           "clusters_used": int(len(np.unique(rec[:, 7]))) if n else 0}
    if counts is not None:
        out["counts_match"] = bool(np.array_equal(pub[1:], np.asarray(counts)[1:]))
    out["ok"] = (out["causality_violations"] == 0 and out["provenance_violations"] == 0
                 and out.get("counts_match", True))
    return out


def run_async_parareal_device(coarse, fine, u0, p: int, epsilon: float | None = None, *,
                              max_events: int = 200_000, delay_frac: float = 0.0,
                              seed: int = 0, record_trace: bool = False,
                              trace_cap: int | None = None, domains: int | None = None,
                              lanes: int = 4) -> DeviceAsyncResult:
    """Asynchronous Parareal with real concurrency on the GPU (PAPER.md
    Algorithm 2): one persistent launch; thread-block clusters act as workers
    that claim slice activations, read the freshest published predecessor
    (no waiting, versioned ring buffers) and publish their update. Stops when
    every slice is drained and its last change is below epsilon, or at exact
    quiescence when epsilon is None.

    ``domains > 1`` splits the slices into that many contiguous domains with
    their own rings, mailboxes and status boards, hosted by one launch on this
    GPU: the multi-GPU protocol of ``distributed.run_async_parareal_distributed``
    (P2P push of the boundary state, distributed stop) on one device.

    2-D/3-D operators run on ``lanes`` CUDA streams instead (one activation =
    F, G and the correction of one slice as whole-GPU launches,
    async_streams.py)."""
    import time

    if p < 1:
        raise ValueError(f"need p >= 1 subintervals, got {p}")
    if epsilon is not None and epsilon <= 0.0:
        raise ValueError(f"epsilon must be positive, got {epsilon}")
    if domains is None:
        # per-domain claim queues keep the activations local (C2: kappa 110 -> 48,
        # 1.03 -> 0.40 s to eps = 1e-10 with 8 domains, profiles/r01_async_domains.jsonl)
        domains = max(1, min(8, p // 8))
    if not (fine.is_tridiagonal and coarse.is_tridiagonal):
        # 2-D/3-D operators: an activation is a whole-GPU job, orchestrated on
        # streams (async_streams.py); same stopping rules and result fields
        from .async_streams import run_async_parareal_streams
        return run_async_parareal_streams(coarse, fine, u0, p, epsilon, lanes=max(lanes, domains),
                                          domains=domains, max_events=max_events, delay_frac=delay_frac,
                                          seed=seed, record_trace=True)
    from .model import with_register_layout
    coarse = with_register_layout(coarse, fine.info.points_per_thread) if fine.is_tridiagonal else coarse
    lam = torch.empty(p + 1, coarse.dim, dtype=coarse.dtype, device=f"cuda:{coarse.device}")
    lam[0] = _u0_tensor(coarse, u0)
    _coarse_init_into(coarse, lam, p, None)
    out = torch.empty_like(lam)
    counts = np.zeros(p + 1, dtype=np.int64)
    info = np.zeros(5, dtype=np.int64)
    lib = _native.load_library()
    torch.cuda.synchronize(fine.device)
    t0 = time.perf_counter()
    cap = 0
    trace_buf = None
    if record_trace:
        cap = int(trace_cap if trace_cap is not None else min(max_events, 1_000_000))
        trace_buf = np.zeros((cap, len(TRACE_FIELDS)), dtype=np.int64)
    if not 1 <= int(domains) <= p:
        raise ValueError(f"need 1 <= domains <= p, got {domains}")
    rc = lib.pint_async_run_domains(fine.handle, coarse.handle, ctypes.c_void_p(lam.data_ptr()), int(p),
                                    int(domains), float(-1.0 if epsilon is None else epsilon), int(max_events),
                                    float(delay_frac), int(seed), ctypes.c_void_p(out.data_ptr()),
                                    counts.ctypes.data_as(ctypes.c_void_p), info.ctypes.data_as(ctypes.c_void_p),
                                    ctypes.c_void_p(trace_buf.ctypes.data if trace_buf is not None else 0), cap,
                                    ctypes.c_void_p(_device.stream_ptr(fine.device)))
    _native.check(rc, fine._ctx.handle, "pint_async_run")
    wall = time.perf_counter() - t0
    if info[2]:
        raise ValueError("block entries must be finite")
    records = trace_buf[:min(int(info[0]), cap)] if trace_buf is not None else None
    res = DeviceAsyncResult(BlockVector(out, check_finite=False), counts, info, wall, records, p, seed)
    if res.stop_reason == "max_events":
        raise HorizonExhausted(f"no stop condition met within {max_events} activations", res)
    return res
