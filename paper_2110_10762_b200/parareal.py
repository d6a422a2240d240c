"""Synchronous Parareal on the B200 (reference: pintlab/parareal.py:1-138).

Same names, signatures, stop rules and results as the reference:

* ``parareal_update`` — G(fresh) + F(old) - G(old) in that FP order, or
  F(old) when the two readings are bitwise equal (parareal.py:25-36);
* ``sequential_fine_solve`` / ``coarse_init`` (parareal.py:39-63);
* ``parareal_iterate`` — one full sweep, no freeze (parareal.py:66-76);
* ``run_parareal`` — frozen prefix, strict threshold, stop order
  threshold -> exact -> k_max (parareal.py:99-138).

The hot loop is restructured for the GPU without changing any value:
each sweep is one batched launch of F over all live slices (the F calls of a
sweep are independent, parareal.py:125) followed by one fused coarse-sweep
launch that carries the running iterate on-chip through the serial G chain and
applies the correction and the per-slice convergence norm in its epilogue
(pint_sync_sweep). G(old) is not recomputed: it is the previous sweep's
G(new) of the same bits (Algorithm 1's w_i^k).
"""
from __future__ import annotations

import ctypes
import os
import json
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device, _native
from .linalg import BlockVector

STOP_THRESHOLD = "threshold"
STOP_KMAX = "k_max"
STOP_EXACT = "exact"

RECORD_LIMIT_BYTES = 1 << 30  # keep every iterate only while they fit in 1 GiB


def _ctx(prop):
    return prop._ctx.handle


def _stream(prop):
    return ctypes.c_void_p(_device.stream_ptr(prop.device))


def correct_into(ctx_prop, gnew, f, gold, prev, out, f_only, delta, nonfinite, nbatch: int) -> None:
    """pint_correct on device tensors (rows of length dim)."""
    lib = _native.load_library()
    dtype = _native.PINT_F64 if out.dtype == torch.float64 else _native.PINT_F32
    dim = out.shape[-1]
    ptr = lambda t: ctypes.c_void_p(t.data_ptr() if t is not None else 0)  # noqa: E731
    rc = lib.pint_correct(_ctx(ctx_prop), dtype, int(dim), int(nbatch), ptr(gnew), ptr(f), ptr(gold), ptr(prev),
                          ptr(out), ptr(f_only), ptr(delta), ptr(nonfinite), _stream(ctx_prop))
    _native.check(rc, _ctx(ctx_prop), "pint_correct")


def correct_chain_into(ctx_prop, gnew, f, gcache, prev, out, fonly_delta, delta, nonfinite, f_only=None) -> None:
    """pint_correct_chain: one coarse-chain step of the generic sweep (F-only
    decided on the device from the predecessor's delta, G(old) cache
    refreshed in place, delta accumulated into a slot zeroed per sweep)."""
    lib = _native.load_library()
    dtype = _native.PINT_F64 if out.dtype == torch.float64 else _native.PINT_F32
    ptr = lambda t: ctypes.c_void_p(t.data_ptr() if t is not None else 0)  # noqa: E731
    rc = lib.pint_correct_chain(_ctx(ctx_prop), dtype, int(out.shape[-1]), ptr(gnew), ptr(f), ptr(gcache), ptr(prev),
                                ptr(out), ptr(f_only), ptr(fonly_delta), ptr(delta), ptr(nonfinite),
                                _stream(ctx_prop))
    _native.check(rc, _ctx(ctx_prop), "pint_correct_chain")


def parareal_update(coarse, fine, fresh_prev, old_prev):
    """One interface-state correction from two predecessor readings
    (parareal.py:25-36). Inputs may be numpy arrays or device tensors; the
    result is of the same kind."""
    is_torch = isinstance(fresh_prev, torch.Tensor) or isinstance(old_prev, torch.Tensor)
    dev = fine.device
    fresh, _ = _device.as_device_tensor(fresh_prev, dev, fine.dtype)
    old, _ = _device.as_device_tensor(old_prev, dev, fine.dtype)
    fresh = fresh.reshape(-1)
    old = old.reshape(-1)
    if torch.equal(fresh, old):
        out = fine.apply(old)
    else:
        g_f = coarse.apply(fresh)
        f_o = fine.apply(old)
        g_o = coarse.apply(old)
        out = torch.empty_like(f_o)
        correct_into(fine, g_f, f_o, g_o, None, out, None, None, None, 1)
    return out if is_torch else _device.to_host(out).astype(float)


def _u0_tensor(prop, u0) -> torch.Tensor:
    t, _ = _device.as_device_tensor(u0, prop.device, prop.dtype)
    t = t.reshape(-1)
    if t.numel() != prop.dim:
        from .errors import DimensionError
        raise DimensionError(f"initial state has dim {t.numel()}, expected {prop.dim}")
    return t


def sequential_fine_solve(fine, u0, p: int) -> BlockVector:
    """lambda_0 = u0, lambda_i = F(lambda_{i-1}) (parareal.py:39-51): the
    purely sequential fine solution every parallel variant must reproduce."""
    if p < 1:
        raise ValueError(f"need p >= 1 subintervals, got {p}")
    lam = torch.empty(p + 1, fine.dim, dtype=fine.dtype, device=f"cuda:{fine.device}")
    lam[0] = _u0_tensor(fine, u0)
    for i in range(1, p + 1):
        fine.apply_ptr(lam[i - 1].data_ptr(), lam[i].data_ptr(), 1, fine.dim)
    return BlockVector(lam, check_finite=False)


def _coarse_init_into(coarse, lam: torch.Tensor, p: int, gcache: torch.Tensor | None) -> None:
    lib = _native.load_library()
    rc = lib.pint_coarse_init(coarse.handle, ctypes.c_void_p(lam.data_ptr()), int(p),
                              ctypes.c_void_p(gcache.data_ptr() if gcache is not None else 0), _stream(coarse))
    _native.check(rc, _ctx(coarse), "pint_coarse_init")


def coarse_init(coarse, u0, p: int) -> BlockVector:
    """Initial interface states from a sequential coarse pass (parareal.py:54-63)."""
    if p < 1:
        raise ValueError(f"need p >= 1 subintervals, got {p}")
    lam = torch.empty(p + 1, coarse.dim, dtype=coarse.dtype, device=f"cuda:{coarse.device}")
    lam[0] = _u0_tensor(coarse, u0)
    _coarse_init_into(coarse, lam, p, None)
    return BlockVector(lam, check_finite=False)


def parareal_iterate(coarse, fine, lam: BlockVector, out: torch.Tensor | None = None) -> BlockVector:
    """One full sweep over all interface states, ascending in i, component 0
    pinned (parareal.py:66-76): new[i] = parareal_update(G, F, new[i-1],
    lam[i-1]) — the synchronous engine's sweep k = 1 with G(old) recomputed
    from ``lam`` (bitwise one sweep of run_parareal).

    Host in, host out: when ``lam`` holds a host tensor the sweep runs from
    host buffers (pinned uploads overlapped with the F launches that read
    them, results downloaded part by part as the coarse chain passes, the
    stream work replayed as one CUDA graph) and the result is a host
    BlockVector in ``out`` (a pinned (p+1) x N tensor, allocated when not
    given). A device ``lam`` gives a device result."""
    t = lam.tensor
    p = t.shape[0] - 1
    if p < 1:
        raise ValueError(f"need p >= 1 subintervals, got {p}")
    if t.shape[1] != fine.dim:
        from .errors import DimensionError
        raise DimensionError(f"block dim {t.shape[1]} does not match the propagator dim {fine.dim}")
    eng = _iterate_engine(coarse, fine, p)
    if t.device.type == "cpu":
        host_in = t if (t.dtype == fine.dtype and t.is_pinned() and t.is_contiguous()) else \
            t.to(fine.dtype).contiguous().pin_memory()
        if out is None:
            out = torch.empty_like(host_in).pin_memory()
        out[0].copy_(host_in[0])
        eng.prev = eng.lam_b
        eng.sweep_host(1, host_in, out, graph=True, gold_from_prev=True)
        return BlockVector(out, check_finite=False)
    eng.lam_a.copy_(t.to(device=eng.lam_a.device, dtype=fine.dtype))
    eng.lam_b[0].copy_(eng.lam_a[0])
    eng.prev = eng.lam_a
    eng.sweep(1, eng.lam_b, gold_from_prev=True)
    eng.read_delta()  # raises ValueError on a non-finite state
    return BlockVector(eng.lam_b.clone(), check_finite=False)


def _iterate_engine(coarse, fine, p: int):
    """A SyncEngine kept on the fine operator for repeated parareal_iterate
    calls with the same (coarse, p) (buffers and captured graphs reused)."""
    cache = fine.__dict__.setdefault("_iterate_engines", {})
    key = (id(coarse), int(p))
    eng = cache.get(key)
    if eng is None:
        cache.clear()
        eng = cache[key] = SyncEngine(coarse, fine, p)
    return eng


@dataclass
class SyncTrace:
    """Record of a synchronous run (parareal.py:79-96). ``iterates`` holds every
    iterate when they fit in RECORD_LIMIT_BYTES (or record_iterates=True),
    else only the initial and the final iterate; ``final`` is always the last."""

    iterates: list
    k_final: int
    stop_reason: str
    deltas: list
    final: BlockVector | None = None
    slice_deltas: list = field(default_factory=list)

    def to_json(self, include_iterates: bool = False) -> str:
        doc = {"k_final": self.k_final, "stop_reason": self.stop_reason, "deltas": list(self.deltas)}
        if include_iterates:
            doc["iterates"] = [it.data.tolist() for it in self.iterates]
        return json.dumps(doc, sort_keys=True)


class SyncEngine:
    """Device buffers and launches of the synchronous iteration.

    lam_a / lam_b  ping-pong iterates ((p+1) x dim, HBM resident)
    fv             F(prev[i-1]) for the live slices of the current sweep
    gcache         G(prev[i-1]): the previous sweep's G(new), reused as G(old)
    deltas         per-slice max |new - prev| of the current sweep
    """

    def __init__(self, coarse, fine, p: int):
        if coarse.dim != fine.dim:
            from .errors import DimensionError
            raise DimensionError("coarse and fine propagators differ in dimension")
        if coarse.device != fine.device or coarse.dtype != fine.dtype:
            raise ValueError("coarse and fine propagators must share device and dtype")
        self.coarse, self.fine, self.p = coarse, fine, int(p)
        dev = f"cuda:{fine.device}"
        n = fine.dim
        self.lam_a = torch.empty(p + 1, n, dtype=fine.dtype, device=dev)
        self.lam_b = torch.empty_like(self.lam_a)
        self.fv = torch.empty_like(self.lam_a)
        self.gcache = torch.zeros_like(self.lam_a)  # row 0 is never read
        self.deltas = torch.zeros(p + 1, dtype=torch.float64, device=dev)
        self.dmax = torch.zeros(1, dtype=torch.float64, device=dev)
        self.flag = torch.zeros(1, dtype=torch.int32, device=dev)
        self.host = torch.zeros(2, dtype=torch.float64).pin_memory() if torch.cuda.is_available() else None
        self.fused = coarse.is_tridiagonal and bool(coarse.info.fused_sweep)
        self.prev = self.lam_a
        self.lib = _native.load_library()
        # pipelining: F runs in wave-sized chunks of slices on the current
        # stream; each chunk's fused coarse sweep runs on `side` as soon as
        # its F is done, overlapping the next chunk's F
        wave = int(getattr(fine.info, "batch_wave_slices", 0)) if fine.is_tridiagonal else 0
        self.wave = wave if wave > 0 else 0
        if self.wave and os.environ.get("PINT_SWEEP_CHUNK"):
            self.wave = max(1, min(self.wave, int(os.environ["PINT_SWEEP_CHUNK"])))
        self.pipeline = self.fused and self.wave > 0
        self.side = torch.cuda.Stream(device=dev) if self.pipeline else None
        self.copy = torch.cuda.Stream(device=dev) if self.pipeline else None
        self.dcopy = torch.cuda.Stream(device=dev) if self.pipeline else None  # downloads (other PCIe direction)
        # odd F chunks go on a second stream so their clusters start as the
        # previous chunk's retire (as inside one launch)
        self.fstream = torch.cuda.Stream(device=dev) if self.pipeline else None

    def init(self, u0) -> None:
        self.lam_a[0] = _u0_tensor(self.coarse, u0)
        self.lam_b[0] = self.lam_a[0]
        _coarse_init_into(self.coarse, self.lam_a, self.p, self.gcache)
        self.prev = self.lam_a
        self.flag.zero_()

    def fine_batch(self, k: int, fine_done_event=None) -> None:
        """fv[i] = F(prev[i-1]) for i in [k, p]: one launch over all live slices."""
        p, n = self.p, self.fine.dim
        self.fine.apply_ptr(self.prev[k - 1].data_ptr(), self.fv[k].data_ptr(), p - k + 1, n)
        if fine_done_event is not None:
            fine_done_event.record(torch.cuda.current_stream(self.fine.device))

    def coarse_sweep(self, k: int, nxt: torch.Tensor, chain_in: bool = False, hi: int | None = None,
                     stream=None) -> None:
        """Fused G chain + correction + per-slice delta for slices [k, hi]
        (hi = p by default). chain_in: nxt[k-1] and deltas[k-1] already hold
        this sweep's slice k-1 (a previous chunk or another GPU's)."""
        p, prev = self.p, self.prev
        hi = p if hi is None else int(hi)
        if self.fused:
            fn = self.lib.pint_sync_sweep_chain if chain_in else self.lib.pint_sync_sweep
            st = _stream(self.coarse) if stream is None else ctypes.c_void_p(stream.cuda_stream)
            rc = fn(self.coarse.handle, ctypes.c_void_p(prev.data_ptr()), ctypes.c_void_p(nxt.data_ptr()),
                    ctypes.c_void_p(self.fv.data_ptr()), ctypes.c_void_p(self.gcache.data_ptr()), int(k), hi,
                    ctypes.c_void_p(self.deltas.data_ptr()), ctypes.c_void_p(self.flag.data_ptr()), st)
            _native.check(rc, _ctx(self.coarse), "pint_sync_sweep")
        else:
            self._generic_sweep(k, nxt, chain_in, hi)

    def reduce_delta(self, k: int, stream=None) -> None:
        st = _stream(self.fine) if stream is None else ctypes.c_void_p(stream.cuda_stream)
        rc = self.lib.pint_max_reduce(_ctx(self.fine), ctypes.c_void_p(self.deltas.data_ptr()), k - 1, self.p + 1,
                                      ctypes.c_void_p(self.dmax.data_ptr()), st)
        _native.check(rc, _ctx(self.fine), "pint_max_reduce")

    def chunks(self, k: int) -> list:
        """Live slices [k, p] in chunks of at most one wave. The boundaries are
        those of the balanced split of [1, p] (only the first chunk shrinks as
        the frozen prefix grows), so the rows a chunk of sweep k+1 reads were
        produced by the same chunk of sweep k — what lets sweep k+1's first F
        start before sweep k's chain has finished (``speculate``)."""
        if not self.pipeline or self.p <= self.wave:
            return [(k, self.p)]
        n = -(-self.p // self.wave)
        base, extra = divmod(self.p, n)
        out, a = [], 1
        for c in range(n):
            b = a + base + (1 if c < extra else 0) - 1
            if b >= k:
                out.append((max(a, k), b))
            a = b + 1
        return out

    def row_ranges(self, k: int) -> list:
        """Rows of the iterate each chunk's upload carries: a partition of
        [0, p] (chunk c's F needs rows a_c-1 .. b_c-1; its coarse sweep rows
        up to b_c)."""
        out, lo = [], 0
        chunks = self.chunks(k)
        for c, (a, b) in enumerate(chunks):
            hi = self.p if c == len(chunks) - 1 else b
            out.append((lo, hi))
            lo = hi + 1
        return out

    def sweep(self, k: int, nxt: torch.Tensor, fine_done_event=None, h2d=None, d2h=None,
              d2h_splits: int = 1, h2d_splits: int = 1, speculate: bool = False,
              gold_from_prev: bool = False) -> None:
        """Sweep k (device work only, stream-ordered): nxt <- new iterate.
        With several chunks, chunk c's coarse sweep overlaps chunk c+1's F.
        With h2d_splits > 1 every chunk's F is split into that many launches
        on their own streams and the coarse sweep follows part by part, so a
        part's F starts as soon as its rows are uploaded and its results
        leave as soon as the chain has passed them.
        h2d(r0, r1, stream) enqueues the upload of iterate rows [r0, r1]
        before the F that reads them; d2h(lo, hi, last, stream) enqueues the
        download of slices [lo, hi] once the coarse sweep has produced them
        (without F parts, the last chunk's sweep is split into d2h_splits
        launches so its download overlaps it).
        speculate: also launch sweep k+1's first-chunk F as soon as this
        sweep's first chunk has its new values (on its own stream, not joined
        into the current stream), so it runs while this sweep's chain finishes
        and the host reads the delta; the next ``sweep(k+1)`` uses it (a
        stop at k discards it).
        gold_from_prev: G(old) is recomputed from the iterate (gcache[i] <-
        G(prev[i-1]) next to each F launch) instead of taken from the previous
        sweep — a standalone sweep (parareal_iterate)."""
        chunks = self.chunks(k)
        if gold_from_prev:
            speculate = False
        spec = getattr(self, "_spec", None)
        self._spec = None
        if spec is not None and (spec[0] != k or spec[1] is not self.prev or h2d is not None):
            spec[2].synchronize()  # stale speculation (not this sweep): let it finish, recompute
            spec = None
        if len(chunks) == 1 and h2d is None and d2h is None and spec is None:
            self.fine_batch(k, fine_done_event)
            if gold_from_prev:
                self.coarse.apply_ptr(self.prev[k - 1].data_ptr(), self.gcache[k].data_ptr(), self.p - k + 1,
                                      self.fine.dim)
            self.coarse_sweep(k, nxt)
            self.reduce_delta(k)
            self.prev = nxt
            return
        main = torch.cuda.current_stream(self.fine.device)
        side = self.side if self.side is not None else main
        cp = self.copy if self.copy is not None else main
        dn = self.dcopy if getattr(self, "dcopy", None) is not None else cp
        n = self.fine.dim
        fs = [main, self.fstream if self.fstream is not None else main]
        side.wait_stream(main)
        cp.wait_stream(main)
        dn.wait_stream(main)
        fs[1].wait_stream(main)
        rows = self.row_ranges(k)
        split_f = h2d is not None and self.pipeline and h2d_splits > 1

        def split(a, b, m):
            m = max(1, min(int(m), b - a + 1))
            base, extra = divmod(b - a + 1, m)
            out = []
            for q in range(m):
                e = a + base + (1 if q < extra else 0) - 1
                out.append((a, e))
                a = e + 1
            return out

        parts = [split(a, b, h2d_splits if split_f else 1) for (a, b) in chunks]
        used = {fs[0], fs[1]}
        f_done = []
        for c, (a, b) in enumerate(chunks):
            evs = []
            r0 = rows[c][0]
            if c == 0 and spec is not None and spec[3] == (a, b):
                f_done.append([spec[2]])  # launched by the previous sweep
                continue
            for q, (pa, pb) in enumerate(parts[c]):
                if split_f:
                    # one stream per (chunk, part): a later chunk's part is not queued
                    # behind an earlier chunk's part, its clusters start as SMs free up
                    st = self._sub_stream(c * len(parts[0]) + q)
                    st.wait_stream(main)
                else:
                    st = fs[c % 2]
                used.add(st)
                if h2d is not None:
                    r1 = rows[c][1] if q == len(parts[c]) - 1 else pb - 1
                    h2d(r0, r1, cp)
                    r0 = r1 + 1
                    ev = torch.cuda.Event()
                    ev.record(cp)
                    st.wait_event(ev)
                self.fine.apply_ptr(self.prev[pa - 1].data_ptr(), self.fv[pa].data_ptr(), pb - pa + 1, n,
                                    stream=st.cuda_stream)
                if gold_from_prev:
                    self.coarse.apply_ptr(self.prev[pa - 1].data_ptr(), self.gcache[pa].data_ptr(), pb - pa + 1, n,
                                          stream=st.cuda_stream)
                ev = torch.cuda.Event()
                ev.record(st)
                evs.append(ev)
            f_done.append(evs)
        if fine_done_event is not None:
            for st in used:
                if st is not main:
                    main.wait_stream(st)
            fine_done_event.record(main)
        lo = 0
        for c, (a, b) in enumerate(chunks):
            last = c == len(chunks) - 1
            if split_f:
                pieces = [(pr, [f_done[c][q]]) for q, pr in enumerate(parts[c])]
            else:
                m = d2h_splits if (last and d2h is not None) else 1
                pieces = [(pr, f_done[c] if q == 0 else []) for q, pr in enumerate(split(a, b, m))]
            for q, ((pa, pb), evs) in enumerate(pieces):
                for ev in evs:
                    side.wait_event(ev)
                self.coarse_sweep(pa, nxt, chain_in=(c > 0 or q > 0), hi=pb, stream=side)
                final = last and q == len(pieces) - 1
                if final:
                    self.reduce_delta(k, stream=side)
                if d2h is not None:
                    ev = torch.cuda.Event()
                    ev.record(side)
                    dn.wait_event(ev)
                    d2h(lo, pb, final, dn)
                    lo = pb + 1
            if c == 0 and speculate and len(chunks) > 1 and k < self.p:
                nk = self.chunks(k + 1)
                a1, b1 = nk[0]
                if b1 <= b:  # its inputs nxt[a1-1 .. b1-1] come from this chunk
                    ev0 = torch.cuda.Event()
                    ev0.record(side)
                    sp = self._spec_stream()
                    sp.wait_event(ev0)
                    self.fine.apply_ptr(nxt[a1 - 1].data_ptr(), self.fv[a1].data_ptr(), b1 - a1 + 1, n,
                                        stream=sp.cuda_stream)
                    evs = torch.cuda.Event()
                    evs.record(sp)
                    self._spec = (k + 1, nxt, evs, (a1, b1))
        for st in used:
            if st is not main:
                main.wait_stream(st)
        main.wait_stream(side)
        main.wait_stream(cp)
        main.wait_stream(dn)
        self.prev = nxt

    def finish(self) -> None:
        """Join a speculative launch that the run did not use into the current
        stream: its F results are discarded, but the buffers it writes must
        not be released (or reused by the caching allocator) before it ends."""
        spec = getattr(self, "_spec", None)
        self._spec = None
        if spec is not None:
            torch.cuda.current_stream(self.fine.device).wait_event(spec[2])

    def _spec_stream(self):
        st = getattr(self, "_spec_st", None)
        if st is None:
            st = self._spec_st = torch.cuda.Stream(device=f"cuda:{self.fine.device}")
        return st

    def _sub_stream(self, q: int):
        """Streams of the first chunk's split F launches (independent, so each
        part's clusters start as soon as its rows are uploaded)."""
        subs = getattr(self, "_subs", None)
        if subs is None:
            subs = self._subs = []
        while len(subs) <= q:
            subs.append(torch.cuda.Stream(device=f"cuda:{self.fine.device}"))
        return subs[q]

    def sweep_host(self, k: int, host_prev: torch.Tensor, host_next: torch.Tensor, d2h_splits: int = 4,
                   h2d_splits: int = 8, graph: bool = False, gold_from_prev: bool = False) -> float:
        """One sweep from host (pinned) buffers: host_prev -> device iterate ->
        sweep -> host_next. Uploads run ahead of the F launches that read
        them; with h2d_splits > 1 each chunk's F runs as that many launches
        that start as their rows arrive, and the coarse sweep and the
        downloads follow part by part (C2 on B200: h2d 52 GB/s, d2h 29 GB/s,
        so the last part's download is the exposed tail; 8 parts, each on its
        own stream, measured best: 4.34 ms vs 4.54 unsplit, scripts/e2e_probe.py).
        ``graph=True`` captures the sweep's stream work (copies and launches on
        all streams) once per buffer pairing into a CUDA graph and replays it,
        so repeated sweeps cost one graph launch of host time. Returns the delta."""
        dev_prev = self.lam_a if self.prev is not self.lam_a else self.lam_b
        nxt = self.lam_b if dev_prev is self.lam_a else self.lam_a
        if graph:
            key = (k, host_prev.data_ptr(), host_next.data_ptr(), d2h_splits, h2d_splits, dev_prev is self.lam_a,
                   gold_from_prev)
            graphs = self.__dict__.setdefault("_graphs", {})
            g = graphs.get(key)
            if g is None:
                g = self._capture(lambda: self._host_sweep_work(k, dev_prev, nxt, host_prev, host_next, d2h_splits,
                                                                h2d_splits, gold_from_prev))
                graphs[key] = g
            g.replay()
            self.prev = nxt
        else:
            self._host_sweep_work(k, dev_prev, nxt, host_prev, host_next, d2h_splits, h2d_splits, gold_from_prev)
        torch.cuda.current_stream(self.fine.device).synchronize()
        if self.host[1].item() != 0.0:
            raise ValueError("block entries must be finite")
        return float(self.host[0].item())

    def _capture(self, work):
        """CUDA graph of ``work()`` (stream-ordered work that forks to and
        joins back from the engine's side streams)."""
        dev = f"cuda:{self.fine.device}"
        g = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream(device=dev)
        cap.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.graph(g, stream=cap, capture_error_mode="thread_local"):
            work()
        torch.cuda.current_stream(dev).wait_stream(cap)
        return g

    def _host_sweep_work(self, k, dev_prev, nxt, host_prev, host_next, d2h_splits, h2d_splits,
                         gold_from_prev=False) -> None:

        def h2d(r0, r1, st):
            with torch.cuda.stream(st):
                dev_prev[r0:r1 + 1].copy_(host_prev[r0:r1 + 1], non_blocking=True)

        def d2h(r0, r1, final, st):
            with torch.cuda.stream(st):
                host_next[r0:r1 + 1].copy_(nxt[r0:r1 + 1], non_blocking=True)
                if final:
                    self.host[:1].copy_(self.dmax, non_blocking=True)
                    self.host[1:2].copy_(self.flag.to(torch.float64), non_blocking=True)

        self.prev = dev_prev
        self.sweep(k, nxt, h2d=h2d, d2h=d2h, d2h_splits=d2h_splits, h2d_splits=h2d_splits,
                   gold_from_prev=gold_from_prev)

    def launches_per_sweep(self, k: int = 1) -> int:
        """Our kernel launches per sweep (fused path: F batch and coarse sweep
        per chunk, max-reduce)."""
        return 2 * len(self.chunks(k)) + 1 if self.fused else 1 + 3 * self.p

    def launches_per_host_sweep(self, k: int = 1, d2h_splits: int = 4, h2d_splits: int = 8) -> int:
        """As launches_per_sweep, for sweep_host (every chunk's F split into
        h2d_splits launches with the coarse sweep following part by part;
        without a pipeline, one F launch and d2h_splits sweep launches)."""
        if not self.fused:
            return 1 + 3 * self.p
        ch = self.chunks(k)
        if self.pipeline and h2d_splits > 1:
            parts = sum(min(h2d_splits, b - a + 1) for a, b in ch)
            return 2 * parts + 1
        a, b = ch[-1]
        return 2 * len(ch) - 1 + min(d2h_splits, b - a + 1) + 1

    def _generic_sweep(self, k: int, nxt: torch.Tensor, chain_in: bool = False, hi: int | None = None) -> None:
        """Coarse chain + correction for coarse operators without a fused
        sweep kernel (2-D/3-D direct or CG coarse): same values, two launches
        per slice (G, then pint_correct_chain: the F-only branch from the
        predecessor's delta, the G(old) cache refreshed in place)."""
        p, prev = self.p, self.prev
        hi = p if hi is None else int(hi)
        if not chain_in:
            nxt[k - 1].copy_(prev[k - 1])
        # slice k-1 is frozen (delta 0 => F-only for slice k) unless its new value came in on the chain
        self.deltas[k if chain_in else k - 1:hi + 1].zero_()
        g = self._gbuf(nxt)
        for i in range(k, hi + 1):
            self.coarse.apply_ptr(nxt[i - 1].data_ptr(), g.data_ptr(), 1, self.fine.dim)
            correct_chain_into(self.fine, g[0], self.fv[i], self.gcache[i], prev[i], nxt[i], self.deltas[i - 1:i],
                               self.deltas[i:i + 1], self.flag)

    def _gbuf(self, like: torch.Tensor) -> torch.Tensor:
        if getattr(self, "_g", None) is None or self._g.device != like.device:
            self._g = torch.empty(1, self.fine.dim, dtype=self.fine.dtype, device=like.device)
        return self._g

    def read_delta(self) -> float:
        """Host read of the sweep's delta (the one sync per sweep)."""
        if bool(self.flag.item()):
            raise ValueError("block entries must be finite")
        return float(self.dmax.item())


class LeanSyncEngine:
    """Synchronous iteration in place: one iterate, the G(old) cache and a
    chunk of F results — 2 state copies instead of SyncEngine's 4, for
    problems whose state fills HBM (C5: 129 slices x 512^3 fp32 = 66 GB per
    copy; 2 copies fit a 180 GB B200, 4 do not). Same arithmetic as
    SyncEngine's generic sweep (parareal.py:119-127 semantics): F of a chunk
    runs from the old values (the chunk-boundary row is saved before the
    chain overwrites it), the chain then corrects slice by slice into the F
    row (the correction reads F before writing each element) and copies it
    into the iterate."""

    def __init__(self, coarse, fine, p: int, chunk: int | None = None):
        if coarse.dim != fine.dim:
            from .errors import DimensionError
            raise DimensionError("coarse and fine propagators differ in dimension")
        self.coarse, self.fine, self.p = coarse, fine, int(p)
        dev = f"cuda:{fine.device}"
        n = fine.dim
        esz = 8 if fine.dtype == torch.float64 else 4
        if chunk is None:
            chunk = max(1, min(self.p, (8 << 30) // max(1, n * esz)))
        self.chunk = int(chunk)
        self.lam_a = torch.empty(p + 1, n, dtype=fine.dtype, device=dev)
        self.lam_b = self.lam_a  # in place: the next iterate overwrites this one
        self.gcache = torch.zeros_like(self.lam_a)
        self.fv = torch.empty(self.chunk, n, dtype=fine.dtype, device=dev)
        self.saved = torch.empty(1, n, dtype=fine.dtype, device=dev)
        self.g = torch.empty(1, n, dtype=fine.dtype, device=dev)
        self.deltas = torch.zeros(p + 1, dtype=torch.float64, device=dev)
        self.dmax = torch.zeros(1, dtype=torch.float64, device=dev)
        self.flag = torch.zeros(1, dtype=torch.int32, device=dev)
        self.prev = self.lam_a
        self.lib = _native.load_library()

    def init(self, u0) -> None:
        self.lam_a[0] = _u0_tensor(self.coarse, u0)
        _coarse_init_into(self.coarse, self.lam_a, self.p, self.gcache)
        self.flag.zero_()

    def sweep(self, k: int, nxt: torch.Tensor, speculate: bool = False, **_) -> None:
        lam, n, p = self.lam_a, self.fine.dim, self.p
        if nxt is not lam:
            raise ValueError("the lean engine updates its iterate in place")
        self.deltas.zero_()
        a = k
        while a <= p:
            b = min(p, a + self.chunk - 1)
            m = b - a + 1
            # F from the old values: row a-1 is frozen (a == k) or was saved
            # before the previous chunk's chain overwrote it
            src0 = lam[a - 1] if a == k else self.saved[0]
            self.fine.apply_ptr(src0.data_ptr(), self.fv[0].data_ptr(), 1, n)
            if m > 1:
                self.fine.apply_ptr(lam[a].data_ptr(), self.fv[1].data_ptr(), m - 1, n)
            if b < p:
                self.saved[0].copy_(lam[b])
            for i in range(a, b + 1):
                self.coarse.apply_ptr(lam[i - 1].data_ptr(), self.g.data_ptr(), 1, n)
                # in place: lam[i] is read (delta) before it is overwritten, element by element;
                # F-only iff slice i-1 did not move (its delta of this sweep is 0; slice k-1 is frozen)
                correct_chain_into(self.fine, self.g[0], self.fv[i - a], self.gcache[i], lam[i], lam[i],
                                   self.deltas[i - 1:i], self.deltas[i:i + 1], self.flag)
            a = b + 1
        rc = self.lib.pint_max_reduce(_ctx(self.fine), ctypes.c_void_p(self.deltas.data_ptr()), k - 1, p + 1,
                                      ctypes.c_void_p(self.dmax.data_ptr()), _stream(self.fine))
        _native.check(rc, _ctx(self.fine), "pint_max_reduce")
        self.prev = lam

    def read_delta(self) -> float:
        if bool(self.flag.item()):
            raise ValueError("block entries must be finite")
        return float(self.dmax.item())


def _pick_engine(coarse, fine, p: int, engine: str | None):
    if engine == "lean":
        return LeanSyncEngine(coarse, fine, p)
    if engine in (None, "auto") and not coarse.is_tridiagonal:
        esz = 8 if fine.dtype == torch.float64 else 4
        need = 4 * (p + 1) * fine.dim * esz
        free, _ = torch.cuda.mem_get_info(fine.device)
        if need > 0.8 * free:
            return LeanSyncEngine(coarse, fine, p)
    return SyncEngine(coarse, fine, p)


def run_parareal(coarse, fine, u0, p: int, epsilon: float, k_max: int | None = None, *,
                 record_iterates: bool | None = None, engine: str | None = None) -> SyncTrace:
    """Iterate from the coarse initialization until a stop condition fires
    (parareal.py:99-138): "threshold" when the sweep-to-sweep change drops
    strictly below epsilon, "exact" at k == p, "k_max" at the budget.
    Components i < k are frozen (already exact). ``engine="lean"`` (chosen
    automatically when four state copies would not fit in HBM) updates one
    iterate in place (LeanSyncEngine)."""
    if epsilon < 0.0:
        raise ValueError(f"epsilon must be nonnegative, got {epsilon}")
    cap = p if k_max is None else min(int(k_max), p)
    if cap < 1:
        raise ValueError(f"iteration budget must allow k >= 1, got k_max={k_max}")
    eng = _pick_engine(coarse, fine, p, engine)
    eng.init(u0)
    esz = 8 if fine.dtype == torch.float64 else 4
    if record_iterates is None:
        record_iterates = (cap + 1) * (p + 1) * fine.dim * esz <= RECORD_LIMIT_BYTES
    lean = isinstance(eng, LeanSyncEngine)
    if lean and record_iterates and (cap + 1) * (p + 1) * fine.dim * esz > RECORD_LIMIT_BYTES:
        record_iterates = False
    # the lean engine exists for states that fill HBM: no initial snapshot
    iterates = [] if (lean and not record_iterates) else [BlockVector(eng.lam_a.clone(), check_finite=False)]
    deltas: list[float] = []
    slice_deltas: list = []
    stop_reason = STOP_KMAX
    k = 0
    try:
        while k < cap:
            k += 1
            nxt = eng.lam_b if eng.prev is eng.lam_a else eng.lam_a
            if record_iterates and nxt is not eng.prev:
                nxt.copy_(eng.prev)
            # sweep k+1's first F starts while this sweep's chain and the host's
            # delta read finish (discarded if this sweep stops the iteration)
            eng.sweep(k, nxt, speculate=k < cap)
            delta = eng.read_delta()
            deltas.append(delta)
            slice_deltas.append(eng.deltas.to("cpu").numpy().copy())
            if record_iterates:
                iterates.append(BlockVector(nxt.clone(), check_finite=False))
            if delta < epsilon:
                stop_reason = STOP_THRESHOLD
                break
            if k == p:
                stop_reason = STOP_EXACT
                break
            if k == cap:
                stop_reason = STOP_KMAX
                break
    finally:
        # a speculative F may still be writing engine buffers (also on an exception)
        if hasattr(eng, "finish"):
            eng.finish()
    # the engine is not reused: hand its iterate over (lean) or copy it out
    final = BlockVector(eng.prev if lean else eng.prev.clone(), check_finite=False)
    if not record_iterates:
        iterates.append(final)
    return SyncTrace(iterates=iterates, k_final=k, stop_reason=stop_reason, deltas=deltas, final=final,
                     slice_deltas=slice_deltas)
