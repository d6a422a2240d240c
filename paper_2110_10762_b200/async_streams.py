"""Asynchronous Parareal with real concurrency for any propagator pair —
the 2-D/3-D configurations (explicit stencil F, direct/CG implicit G), where
one activation is a whole-GPU job rather than one cluster's (SURVEY §8d C4/C5
async; reference semantics async_parareal.py:24-84, async_engine.py:238-365).

The host orchestrates, the device computes. ``lanes`` CUDA streams each run
one activation at a time with their own operator instances (the operators own
scratch): F(remembered) -> copy of the freshest *visible* predecessor version
-> equality flag -> G(fresh) -> correction + delta into the next ring slot of
the slice -> publish. A version becomes visible when its publish event has
completed (``cudaEventQuery``), so staleness is whatever the device schedule
produces; nobody waits for a particular version. Ring slots are recycled only
after every copy that read them has completed (stream waits on the readers'
events). Stop: drained and every last change < eps (async_parareal.py:52-58),
or exact quiescence (every slice stable on the newest predecessor version).

``domains`` splits the slices into contiguous blocks with their own lanes; a
domain's first slice reads its predecessor from a mailbox that the previous
domain's publishing lane fills with a device copy plus its own event — the
single-process form of the multi-GPU push (on several GPUs the copy is a
peer-to-peer copy into the next GPU's mailbox).
"""
from __future__ import annotations

import time

import numpy as np
import torch

from . import _device, _native
from .errors import HorizonExhausted
from .linalg import BlockVector
from .parareal import _coarse_init_into, _u0_tensor, correct_into


def clone_propagator(prop):
    """A second operator object with the same description (own scratch)."""
    import ctypes

    from .model import GPUPropagator
    d = _native.OpDesc()
    ctypes.memmove(ctypes.byref(d), ctypes.byref(prop.desc), ctypes.sizeof(d))
    return GPUPropagator(d, prop.dim, prop.dtype, prop.cost_units, prop.device, prop.rule, prop.span, prop.steps)


class _Lane:
    def __init__(self, coarse, fine, dev, n, dtype, index):
        self.index = index
        self.stream = torch.cuda.Stream(device=dev)
        self.fine = clone_propagator(fine) if index else fine
        self.coarse = clone_propagator(coarse) if index else coarse
        self.f = torch.empty(1, n, dtype=dtype, device=dev)
        self.fresh = torch.empty(1, n, dtype=dtype, device=dev)
        self.g = torch.empty(1, n, dtype=dtype, device=dev)
        self.eq = torch.zeros(1, dtype=torch.uint8, device=dev)
        self.delta = torch.zeros(1, dtype=torch.float64, device=dev)
        self.flag = torch.zeros(1, dtype=torch.int32, device=dev)
        self.host = torch.zeros(3, dtype=torch.float64).pin_memory()  # delta, non-finite, equal
        self.job = None


class StreamAsyncResult:
    """Outcome of ``run_async_parareal_streams`` (same fields as
    DeviceAsyncResult; trace rows follow async_parareal.TRACE_FIELDS with the
    lane id in the last column and host ns clocks)."""

    def __init__(self, final, counts, activations, stop_reason, wall_s, lanes, records, p):
        self.final = final
        self.per_component_counts = counts
        self.activations = activations
        self.stop_reason = stop_reason
        self.retries = 0
        self.concurrent_clusters = lanes
        self.wall_s = wall_s
        self.trace_records = records
        self.p = p

    @property
    def kappa(self) -> int:
        return int(np.max(self.per_component_counts[1:])) if len(self.per_component_counts) > 1 else 0

    def to_async_trace(self):
        from .async_parareal import device_records_to_trace
        return device_records_to_trace(self.trace_records, self.p, self.per_component_counts, self.final,
                                       self.stop_reason)


def run_async_parareal_streams(coarse, fine, u0, p: int, epsilon: float | None = None, *, lanes: int = 4,
                               domains: int = 1, ring: int = 3, max_events: int = 200_000,
                               delay_frac: float = 0.0, seed: int = 0,
                               record_trace: bool = True, claim: str = "lowest") -> StreamAsyncResult:
    if p < 1:
        raise ValueError(f"need p >= 1 subintervals, got {p}")
    if epsilon is not None and epsilon <= 0.0:
        raise ValueError(f"epsilon must be positive, got {epsilon}")
    if not 1 <= domains <= p:
        raise ValueError(f"need 1 <= domains <= p, got {domains}")
    if lanes < domains:
        raise ValueError(f"need at least one lane per domain, got lanes={lanes}, domains={domains}")
    if ring < 2:
        raise ValueError("the version ring needs at least two slots")
    if claim not in ("lowest", "round-robin"):
        raise ValueError(f"claim must be 'lowest' or 'round-robin', got {claim!r}")
    dev = f"cuda:{fine.device}"
    n, dtype = fine.dim, fine.dtype
    R = int(ring)
    # ---- state: version ring per slice (row 0 = u0, never republished)
    lam0 = torch.empty(p + 1, n, dtype=dtype, device=dev)
    lam0[0] = _u0_tensor(coarse, u0)
    _coarse_init_into(coarse, lam0, p, None)
    ring_buf = torch.empty(p + 1, R, n, dtype=dtype, device=dev)
    ring_buf[:, 0] = lam0
    remb = torch.empty(p + 1, n, dtype=dtype, device=dev)
    grem = torch.empty(p + 1, n, dtype=dtype, device=dev)
    remb[1:] = lam0[:-1]  # remembered reading = version 0 of the predecessor
    grem[1:] = lam0[1:]   # G(remembered) = G(lam0[i-1]) = lam0[i]
    # domains: contiguous blocks; block d > 0 reads its predecessor from a mailbox
    parts = [(1 + p * d // domains, p * (d + 1) // domains) for d in range(domains)]
    owner = np.zeros(p + 1, dtype=np.int64)
    for d, (lo, hi) in enumerate(parts):
        owner[lo:hi + 1] = d
    mailbox = {lo - 1: torch.empty(R, n, dtype=dtype, device=dev) for lo, _ in parts[1:]}
    for i, mb in mailbox.items():
        mb[0] = lam0[i]
    mb_events: dict = {i: {} for i in mailbox}   # slot -> publish-copy event
    torch.cuda.synchronize(dev)

    # ---- host bookkeeping (the reference's engine view)
    published = [0] * (p + 1)                 # newest visible version
    pending = {}                              # (i, v) -> event of the publish
    pub_events = [dict() for _ in range(p + 1)]  # slot -> event that wrote it
    readers = [[[] for _ in range(R)] for _ in range(p + 1)]  # events of copies reading a slot
    vrem = [0] * (p + 1)
    consumed = [-1] * (p + 1)
    stable = [False] * (p + 1)
    busy = [False] * (p + 1)
    last = np.full(p + 1, np.inf)
    last[0] = 0.0
    counts = np.zeros(p + 1, dtype=np.int64)
    records = []
    lanes_by_dom = [[] for _ in range(domains)]
    all_lanes = []
    for q in range(lanes):
        ln = _Lane(coarse, fine, dev, n, dtype, q)
        ln.domain = q % domains
        lanes_by_dom[ln.domain].append(ln)
        all_lanes.append(ln)
    tickets = [0] * domains
    spin_cycles_per_tf = 0.0
    if delay_frac > 0.0:  # injected delay U(0, delay_frac) * t_F per activation
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ln0 = all_lanes[0]
        e0.record()
        ln0.fine.apply_ptr(remb[1].data_ptr(), ln0.f.data_ptr(), 1, n)
        e1.record()
        torch.cuda.synchronize(dev)
        clock_khz = torch.cuda.get_device_properties(dev).clock_rate if hasattr(
            torch.cuda.get_device_properties(dev), "clock_rate") else 1_965_000
        spin_cycles_per_tf = e0.elapsed_time(e1) * clock_khz
    lib = _native.load_library()
    dt_code = _native.PINT_F64 if dtype == torch.float64 else _native.PINT_F32
    events = 0
    stop_reason = None
    t_begin = time.perf_counter()

    def visible(i: int) -> int:
        """Newest version of slice i whose publish has completed (polls)."""
        while (i, published[i] + 1) in pending and pending[(i, published[i] + 1)].query():
            del pending[(i, published[i] + 1)]
            published[i] += 1
        return published[i]

    def drained_all() -> bool:
        for i in range(p + 1):
            visible(i)
        return all(consumed[i] == published[i - 1] for i in range(1, p + 1))

    def done() -> bool:
        # the stop predicate on the completed (visible) state; activations
        # still in flight publish versions newer than the snapshot taken here
        if not drained_all():
            return False
        if epsilon is None:
            return all(stable[1:]) and not any(busy[1:])
        return float(np.max(last[1:])) < epsilon

    def source(i: int, v: int):
        """(tensor row, completion event) of version v of slice i-1 as seen by slice i."""
        src = i - 1
        slot = v % R
        if src in mailbox and owner[src] != owner[i]:
            return mailbox[src][slot], mb_events[src].get(slot), (src, slot, True)
        return ring_buf[src, slot], pub_events[src].get(slot), (src, slot, False)

    def dispatch(ln: _Lane, i: int) -> None:
        nonlocal events
        v = visible(i - 1)
        vr = vrem[i]
        t0 = time.perf_counter_ns()
        busy[i] = True
        st = ln.stream
        row, ev_src, key = source(i, v)
        vi = published[i] + sum(1 for (j, _) in pending if j == i)
        dst_slot = (vi + 1) % R
        with torch.cuda.stream(st):
            # the slot about to be written must not be read any more
            for ev in readers[i][dst_slot]:
                st.wait_event(ev)
            readers[i][dst_slot] = []
            if i in mailbox:
                for ev in [e for e in mb_readers[i][dst_slot]]:
                    st.wait_event(ev)
                mb_readers[i][dst_slot] = []
            ln.fine.apply_ptr(remb[i].data_ptr(), ln.f.data_ptr(), 1, n, stream=st.cuda_stream)
            if delay_frac > 0.0:
                # U(0, delay_frac) * t_F keyed by (seed, slice, activation), as in the kernel runtime
                torch.cuda._sleep(int(_unit(seed, i, int(counts[i])) * delay_frac * spin_cycles_per_tf))
            if ev_src is not None:
                st.wait_event(ev_src)
            ln.fresh[0].copy_(row, non_blocking=True)
            rd = torch.cuda.Event()
            rd.record(st)
            src, slot, is_mb = key
            (mb_readers[src][slot] if is_mb else readers[src][slot]).append(rd)
            if v == vr:
                ln.eq.fill_(1)
            else:
                rc = lib.pint_equal_flag(ln.fine._ctx.handle, dt_code, n, _ptr(ln.fresh), _ptr(remb[i]), _ptr(ln.eq),
                                         _sptr(st))
                _native.check(rc, ln.fine._ctx.handle, "pint_equal_flag")
            ln.coarse.apply_ptr(ln.fresh.data_ptr(), ln.g.data_ptr(), 1, n, stream=st.cuda_stream)
            cur = ring_buf[i, vi % R]
            dst = ring_buf[i, dst_slot]
            correct_into(ln.fine, ln.g, ln.f, grem[i:i + 1], cur.reshape(1, -1), dst.reshape(1, -1), ln.eq,
                         ln.delta, ln.flag, 1)
            grem[i].copy_(ln.g[0], non_blocking=True)
            remb[i].copy_(ln.fresh[0], non_blocking=True)
            ln.host[0:1].copy_(ln.delta, non_blocking=True)
            ln.host[1:2].copy_(ln.flag.to(torch.float64), non_blocking=True)
            ln.host[2:3].copy_(ln.eq.to(torch.float64), non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(st)
            pub_events[i][dst_slot] = ev
            if i in mailbox:  # push into the next domain's mailbox (a P2P copy across GPUs)
                mailbox[i][dst_slot].copy_(dst, non_blocking=True)
                evm = torch.cuda.Event()
                evm.record(st)
                mb_events[i][dst_slot] = evm
                ev = evm
            pending[(i, vi + 1)] = ev
        ln.job = (i, v, vr, t0, ev)

    def finish(ln: _Lane) -> None:
        nonlocal events
        i, v, vr, t0, ev = ln.job
        ln.job = None
        if ln.host[1].item() != 0.0:
            raise ValueError("block entries must be finite")
        d = float(ln.host[0].item())
        fonly = (v == vr) or ln.host[2].item() != 0.0
        last[i] = d
        vrem[i] = v
        consumed[i] = v
        stable[i] = fonly
        counts[i] += 1
        busy[i] = False
        events += 1
        if record_trace:
            records.append((i, v, vr, 1 if fonly else 0, int(np.array([d]).view(np.int64)[0]), t0,
                            time.perf_counter_ns(), ln.index))

    mb_readers = {i: [[] for _ in range(R)] for i in mailbox}

    def pick(dom: int):
        # the lowest slice of the domain with something to do first (the
        # pipeline order of the sweeps), or a round-robin ticket; both are
        # valid asynchronous schedules with the same reads and stop rule
        lo, hi = parts[dom]
        m = hi - lo + 1
        for q in range(m):
            if claim == "round-robin":
                i = lo + tickets[dom] % m
                tickets[dom] += 1
            else:
                i = lo + q
            if busy[i]:
                continue
            if stable[i] and consumed[i] == visible(i - 1):
                last[i] = 0.0  # an activation would reproduce the same value
                continue
            return i
        return None

    while True:
        progressed = False
        # Completed activations are retired in dispatch order: a consumer is only
        # dispatched after its producer's publish event completed (visible()
        # polls the events), so its record must follow the producer's even when
        # both are found complete in the same pass (the trace audit replays the
        # records as the publish order).
        ready = [ln for ln in all_lanes if ln.job is not None and ln.job[4].query()]
        ready.sort(key=lambda ln: ln.job[3])
        for ln in ready:
            finish(ln)
            progressed = True
        if done():
            stop_reason = "converged"
            break
        if events >= max_events:
            stop_reason = "max_events"
            break
        for ln in all_lanes:
            if ln.job is None:
                i = pick(ln.domain)
                if i is not None:
                    dispatch(ln, i)
                    progressed = True
        if not progressed:
            waiting = [ln.job[4] for ln in all_lanes if ln.job is not None]
            if waiting:
                waiting[0].synchronize()
            elif not pending:
                # nothing in flight and nothing to do: every slice stable & drained
                if done():
                    stop_reason = "converged"
                    break
            else:
                next(iter(pending.values())).synchronize()
    snap = list(published)  # the state the stop decision saw
    wall = time.perf_counter() - t_begin
    torch.cuda.synchronize(dev)
    final = torch.stack([ring_buf[i, snap[i] % R] for i in range(p + 1)])
    res = StreamAsyncResult(BlockVector(final, check_finite=False), counts, events, stop_reason, wall, lanes,
                            np.array(records, dtype=np.int64).reshape(-1, 8) if record_trace else None, p)
    if stop_reason == "max_events":
        raise HorizonExhausted(f"no stop condition met within {max_events} activations", res)
    return res


def _unit(seed: int, i: int, count: int) -> float:
    """splitmix64 of (seed, slice, activation) -> U[0, 1) (async_rt.cu mix64)."""
    m = (1 << 64) - 1
    z = (seed ^ ((i << 32) & m) ^ count) & m
    z = (z + 0x9E3779B97F4A7C15) & m
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    z ^= z >> 31
    return (z >> 11) * (1.0 / 9007199254740992.0)


def _ptr(t):
    import ctypes
    return ctypes.c_void_p(t.data_ptr())


def _sptr(st):
    import ctypes
    return ctypes.c_void_p(st.cuda_stream)
