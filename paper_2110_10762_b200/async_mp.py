"""Multi-GPU asynchronous Parareal for whole-GPU activations — the 2-D/3-D
configurations C4/C5 (explicit stencil F, direct implicit G), one process per
GPU (Algorithm 2; reference semantics async_parareal.py:24-84 and
async_engine.py:238-365, which are single-process).

Rank r owns the contiguous slices ``async_partition(p, W)[r] = lo..hi`` and
holds ONLY their states (a version ring of R slots per slice, the remembered
predecessor reading and its G) plus the predecessor's mailbox: memory per rank
is (nloc + 1) * (R + 2) state copies, never the whole (p + 1) x N iterate.

Data path (no NCCL, no barrier, no host round trip between GPUs):

* the activation of slice i runs on one of the rank's CUDA streams ("lanes"):
  F(remembered) -> read of the freshest predecessor version -> equality flag
  -> G(fresh) -> correction + delta into the slice's next ring slot;
* the predecessor of the rank's first slice lives on the previous GPU. That
  GPU pushes every new version of its last slice straight into this rank's
  mailbox ring with SM stores over NVLink (CUDA IPC peer memory) and then
  release-stores the version word at system scope (``pint_mailbox_push``);
  this rank reads the freshest version under a seqlock
  (``pint_mailbox_read``). Nobody waits for a particular version, so the
  staleness is what the hardware schedule produces (the paper's async model);
* termination without a global barrier: every rank posts its status
  {done, consumed ghost version, last published version of its last slice,
  publish count} into every rank's status board (seqlocked slots, system-scope
  release) whenever it becomes done or stops being done; a done rank
  double-collects its board and, when every rank is done, every ghost version
  consumed equals the predecessor's published one and nothing changed between
  the two collects, the cut is consistent and the stop predicate held on it
  (async_parareal.py:52-58 ``drained and max(last) < eps``, or exact
  quiescence) — it raises the stop word on every board.

NCCL (or gloo) is used afterwards only: the final reductions (stop code,
counts, wall time) and, on request, gathering the final iterate to rank 0.

``transport`` and ``ops`` isolate the device (CUDA IPC + the C ABI kernels,
the GPU propagators) so the protocol runs unchanged over CPU test doubles
(tests/async_mp_doubles.py; gloo world sizes 2 and 3).
"""
from __future__ import annotations

import ctypes
import time

import numpy as np
import torch

from . import _native
from .distributed import async_partition
from .errors import HorizonExhausted

# board slot words (after the sequence word)
W_DONE, W_CONSUMED, W_PUBHI, W_PUBCOUNT, W_EVENTS, W_CODE, W_SPARE = range(7)
STOP_CONVERGED, STOP_HORIZON, STOP_NONFINITE = 1, 2, 3




# ============================================================ device pieces
class _CAI:
    """Zero-copy torch view of raw device memory (__cuda_array_interface__)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"data": (int(ptr), False), "shape": tuple(shape), "typestr": typestr,
                                         "version": 3, "strides": None}


_TYPESTR = {torch.float64: "<f8", torch.float32: "<f4", torch.int64: "<i8", torch.int32: "<i4",
            torch.uint32: "<u4"}


class CudaTransport:
    """Shared device workspaces exported through CUDA IPC, and the mailbox /
    board kernels of the C ABI (csrc/mailbox.cu)."""

    def __init__(self, prop):
        self.lib = _native.load_library()
        self.prop = prop
        self.ctx = prop._ctx.handle
        self.device = int(prop.device)
        self._opened = []
        self._owned = []
        self._exports = {}  # handle -> pointer of this process's own exported workspaces

    def _chk(self, rc, what):
        _native.check(rc, self.ctx, what)

    # ---- memory
    def alloc(self, nbytes: int) -> int:
        p = ctypes.c_void_p()
        self._chk(self.lib.pint_shared_alloc(self.ctx, int(nbytes), ctypes.byref(p)), "pint_shared_alloc")
        self._owned.append(p.value)
        return int(p.value)

    def view(self, ptr: int, shape, dtype) -> torch.Tensor:
        return torch.as_tensor(_CAI(ptr, shape, _TYPESTR[dtype]), device=f"cuda:{self.device}")

    def export(self, ptr: int) -> bytes:
        buf = (ctypes.c_ubyte * 64)()
        self._chk(self.lib.pint_ipc_export(self.ctx, ctypes.c_void_p(ptr), buf), "pint_ipc_export")
        self._exports[bytes(buf)] = int(ptr)
        return bytes(buf)

    def open(self, handle: bytes, own_ptr: int, own_handle: bytes) -> int:
        if handle == own_handle:  # a process cannot open its own allocation
            return own_ptr
        if handle in self._exports:  # another workspace of this same process
            return self._exports[handle]
        buf = (ctypes.c_ubyte * 64).from_buffer_copy(handle)
        p = ctypes.c_void_p()
        self._chk(self.lib.pint_ipc_open(self.ctx, buf, ctypes.byref(p)), "pint_ipc_open")
        self._opened.append(p.value)
        return int(p.value)

    def close(self) -> None:
        torch.cuda.synchronize(self.device)
        for p in self._opened:
            self.lib.pint_ipc_close(self.ctx, ctypes.c_void_p(p))
        for p in self._owned:
            self.lib.pint_shared_free(self.ctx, ctypes.c_void_p(p))
        self._opened, self._owned = [], []

    # ---- streams
    def stream(self):
        return torch.cuda.Stream(device=self.device)

    def event(self, stream):
        ev = torch.cuda.Event()
        ev.record(stream)
        return ev

    def stream_ctx(self, stream):
        return torch.cuda.stream(stream)

    @staticmethod
    def sptr(stream) -> ctypes.c_void_p:
        return ctypes.c_void_p(stream.cuda_stream)

    # ---- kernels
    def push(self, dst_ptr: int, src: torch.Tensor, ver_ptr: int, version: int, ctr_ptr: int, stream) -> None:
        nbytes = src.numel() * src.element_size()
        self._chk(self.lib.pint_mailbox_push(self.ctx, ctypes.c_void_p(dst_ptr), ctypes.c_void_p(src.data_ptr()),
                                             nbytes, ctypes.c_void_p(ver_ptr), int(version),
                                             ctypes.c_void_p(ctr_ptr), self.sptr(stream)), "pint_mailbox_push")

    def read_mailbox(self, ring_ptr: int, slot_bytes: int, nslots: int, ver_ptr: int, dst: torch.Tensor,
                     scratch: torch.Tensor, stream) -> None:
        """scratch: int64[3] on the device = (vsel, v_out, torn)."""
        nbytes = dst.numel() * dst.element_size()
        sp = scratch.data_ptr()
        self._chk(self.lib.pint_mailbox_read(self.ctx, ctypes.c_void_p(ring_ptr), int(slot_bytes), int(nslots),
                                             ctypes.c_void_p(ver_ptr), ctypes.c_void_p(dst.data_ptr()), nbytes,
                                             ctypes.c_void_p(sp), ctypes.c_void_p(sp + 8),
                                             ctypes.c_void_p(sp + 16), self.sptr(stream)), "pint_mailbox_read")

    def post(self, slot_ptr: int, seq: int, words, stream) -> None:
        w = (ctypes.c_int64 * 7)(*[int(x) for x in words])
        self._chk(self.lib.pint_board_post(self.ctx, ctypes.c_void_p(slot_ptr), int(seq), w, self.sptr(stream)),
                  "pint_board_post")

    def read_board(self, board_ptr: int, nslots: int, out: torch.Tensor, host: torch.Tensor, stream) -> np.ndarray:
        self._chk(self.lib.pint_board_read(self.ctx, ctypes.c_void_p(board_ptr), int(nslots),
                                           ctypes.c_void_p(out.data_ptr()), self.sptr(stream)), "pint_board_read")
        with torch.cuda.stream(stream):
            host.copy_(out, non_blocking=True)
        stream.synchronize()
        return host.numpy().reshape(nslots, 8).copy()

    def read_word(self, t: torch.Tensor, host: torch.Tensor, stream) -> int:
        with torch.cuda.stream(stream):
            host.copy_(t, non_blocking=True)
        stream.synchronize()
        return int(host[0])

    def sleep_cycles(self, cycles: int, stream) -> None:
        with torch.cuda.stream(stream):
            torch.cuda._sleep(int(cycles))

    def wait_version(self, ver_ptr: int, value: int, timed_out: torch.Tensor, stream, timeout_s: float = 30.0) -> None:
        """Stream-ordered wait (one-thread device poll) for a peer's version."""
        self._chk(self.lib.pint_mailbox_wait(self.ctx, ctypes.c_void_p(ver_ptr), int(value), float(timeout_s),
                                             ctypes.c_void_p(timed_out.data_ptr()), self.sptr(stream)),
                  "pint_mailbox_wait")

    def synchronize(self) -> None:
        torch.cuda.synchronize(self.device)


class GpuOps:
    """The activation's compute on the GPU propagators (C ABI kernels)."""

    def __init__(self, coarse, fine):
        from .async_streams import clone_propagator
        self._clone = clone_propagator
        self.coarse, self.fine = coarse, fine
        self.n, self.dtype = fine.dim, fine.dtype
        self.lib = _native.load_library()
        self.dt_code = _native.PINT_F64 if self.dtype == torch.float64 else _native.PINT_F32

    def lane_ops(self, index: int):
        """Per-lane operator instances (operators own their scratch)."""
        if index == 0:
            return self.coarse, self.fine
        return self._clone(self.coarse), self._clone(self.fine)

    def apply(self, prop, src: torch.Tensor, dst: torch.Tensor, stream) -> None:
        prop.apply_ptr(src.data_ptr(), dst.data_ptr(), 1, self.n, stream=stream.cuda_stream)

    def equal(self, a: torch.Tensor, b: torch.Tensor, eq: torch.Tensor, stream) -> None:
        ctx = self.fine._ctx.handle
        rc = self.lib.pint_equal_flag(ctx, self.dt_code, self.n, ctypes.c_void_p(a.data_ptr()),
                                      ctypes.c_void_p(b.data_ptr()), ctypes.c_void_p(eq.data_ptr()),
                                      ctypes.c_void_p(stream.cuda_stream))
        _native.check(rc, ctx, "pint_equal_flag")

    def correct(self, g, f, gold, cur, dst, eq, delta, flag, stream) -> None:
        from .parareal import correct_into
        with torch.cuda.stream(stream):
            correct_into(self.fine, g, f, gold, cur, dst, eq, delta, flag, 1)


# ================================================================ runtime
class MPAsyncResult:
    """Outcome on one rank. ``rows`` = this rank's final states of slices
    lo..hi ((nloc, N) device tensor); ``final`` = the whole (p+1) x N iterate
    on rank 0 when gathered, else None."""

    def __init__(self, **kw):
        self.__dict__.update(kw)

    @property
    def kappa(self) -> int:
        return int(np.max(self.counts[1:])) if len(self.counts) > 1 else 0


class _Lane:
    def __init__(self, rt, index):
        self.index = index
        self.stream = rt.tp.stream()
        self.coarse, self.fine = rt.ops.lane_ops(index)
        n, dt, dev = rt.n, rt.dtype, rt.dev
        self.f = torch.empty(1, n, dtype=dt, device=dev)
        self.fresh = torch.empty(1, n, dtype=dt, device=dev)
        self.g = torch.empty(1, n, dtype=dt, device=dev)
        self.eq = torch.zeros(1, dtype=torch.uint8, device=dev)
        self.delta = torch.zeros(1, dtype=torch.float64, device=dev)
        self.flag = torch.zeros(1, dtype=torch.int32, device=dev)
        self.mb = torch.zeros(3, dtype=torch.int64, device=dev)        # vsel, v_out, torn
        self.ctr = torch.zeros(1, dtype=torch.int32, device=dev)       # push completion counter
        self.host = torch.zeros(6, dtype=torch.float64, pin_memory=rt.pinned)  # delta, nonfinite, eq, v, torn
        self.job = None


class _Runtime:
    def __init__(self, coarse, fine, u0, p, epsilon, lanes, ring, max_events, delay_frac, seed, record_trace,
                 rank, world, transport, ops, exchange, coarse_init_rows):
        self.p, self.eps = int(p), epsilon
        self.rank, self.world = rank, world
        self.tp, self.ops = transport, ops
        self.exchange = exchange
        self.lo, self.hi = async_partition(p, world)[rank]
        self.nloc = self.hi - self.lo + 1
        self.n, self.dtype = fine.dim, fine.dtype
        self.dev = ops.device_str if hasattr(ops, "device_str") else f"cuda:{fine.device}"
        self.pinned = self.dev.startswith("cuda")
        self.R = int(ring)
        self.max_events, self.delay_frac, self.seed = int(max_events), float(delay_frac), int(seed)
        self.record_trace = record_trace
        self.claim = "lowest"
        self.timeout_s = None
        esz = torch.empty(0, dtype=self.dtype).element_size()
        self.row_bytes = self.n * esz
        self.slot_bytes = (self.row_bytes + 255) // 256 * 256
        # ---- this rank's states only: rows lo-1 .. hi of the coarse initial iterate
        lam0 = coarse_init_rows(coarse, u0, self.lo - 1, self.hi)  # (nloc+1) x n
        nl, R, n = self.nloc, self.R, self.n
        self.ring = torch.empty(nl + 1, R, n, dtype=self.dtype, device=self.dev)
        self.ring[:, 0] = lam0
        self.remb = torch.empty(nl + 1, n, dtype=self.dtype, device=self.dev)
        self.grem = torch.empty(nl + 1, n, dtype=self.dtype, device=self.dev)
        self.remb[1:] = lam0[:-1]   # remembered reading: version 0 of the predecessor
        self.grem[1:] = lam0[1:]    # G(remembered) = G(lam0[i-1]) = lam0[i]
        # ---- shared workspace: [mailbox version | board (W+1 slots) | mailbox ring R x slot]
        W = world
        self.board_off = 256
        self.mb_off = self.board_off + ((W + 1) * 64 + 255) // 256 * 256
        ws_bytes = self.mb_off + R * self.slot_bytes
        self.ws = self.tp.alloc(ws_bytes)
        self.mb_ver = self.tp.view(self.ws, (1,), torch.int64)
        self.board = self.tp.view(self.ws + self.board_off, ((W + 1) * 8,), torch.int64)
        self.mb_ring_ptr = self.ws + self.mb_off
        if rank > 0:
            # version 0 of the predecessor slice (bitwise the peer's: same chain, same kernels)
            slot0 = self.tp.view(self.mb_ring_ptr, (n,), self.dtype)
            slot0.copy_(lam0[0])
        self.tp.synchronize()
        my_handle = self.tp.export(self.ws)
        handles = exchange.all_gather_bytes(my_handle)
        self.peer_ws = [self.tp.open(h, self.ws, my_handle) for h in handles]
        self.post_seq = [0] * W
        self.lanes = [_Lane(self, q) for q in range(max(1, int(lanes)))]
        self.ctl = self.tp.stream()
        self.board_out = torch.zeros((W + 1) * 8, dtype=torch.int64, device=self.dev)
        self.board_host = torch.zeros((W + 1) * 8, dtype=torch.int64, pin_memory=self.pinned)
        self.word_host = torch.zeros(1, dtype=torch.int64, pin_memory=self.pinned)
        self.spin_cycles_per_tf = 0.0
        if self.delay_frac > 0.0:
            self._calibrate_delay()
        self.tp.synchronize()

    # ------------------------------------------------------------ helpers
    def _calibrate_delay(self):
        ln = self.lanes[0]
        t0 = time.perf_counter()
        with self.tp.stream_ctx(ln.stream):
            self.ops.apply(ln.fine, self.remb[1], ln.f[0], ln.stream)
        ln.stream.synchronize()
        t_f = time.perf_counter() - t0
        clock_khz = 1_965_000
        self.spin_cycles_per_tf = t_f * 1e3 * clock_khz

    def _peer_board_slot(self, dest: int, writer: int) -> int:
        return self.peer_ws[dest] + self.board_off + 64 * writer

    def _post_all(self, words):
        """Post this rank's status into every rank's board (own included);
        returns after the posts are visible (the stream is synchronised), so a
        status is always published before any activation it permits."""
        for d in range(self.world):
            self.tp.post(self._peer_board_slot(d, self.rank), self.post_seq[d], words, self.ctl)
            self.post_seq[d] += 2
        self.ctl.synchronize()

    def _post_stop(self, code: int):
        words = [code, 0, 0, 0, 0, 0, 0]
        for d in range(self.world):
            # any rank may raise the stop word; identical contents, seq 0 -> 2
            self.tp.post(self._peer_board_slot(d, self.world), 0, words, self.ctl)
        self.ctl.synchronize()

    def _board(self) -> np.ndarray:
        return self.tp.read_board(self.ws + self.board_off, self.world + 1, self.board_out, self.board_host, self.ctl)

    def _ghost_version(self) -> int:
        """Newest version of the predecessor slice visible in the mailbox."""
        if self.rank == 0:
            return 0
        return self.tp.read_word(self.mb_ver, self.word_host, self.ctl)

    # ------------------------------------------------------------ main loop
    def run(self):
        lo, hi, nl, R, n = self.lo, self.hi, self.nloc, self.R, self.n
        W, eps = self.world, self.eps
        ops, tp = self.ops, self.tp
        published = [0] * (nl + 1)
        pending = {}
        pub_events = [dict() for _ in range(nl + 1)]
        readers = [[[] for _ in range(R)] for _ in range(nl + 1)]
        vrem = [0] * (nl + 1)
        consumed = [-1] * (nl + 1)
        stable = [False] * (nl + 1)
        busy = [False] * (nl + 1)
        last = np.full(nl + 1, np.inf)
        counts = np.zeros(nl + 1, dtype=np.int64)
        records = []
        events = 0
        pubcount = 0
        ticket = 0
        ghost = [0]
        posted_done = None
        stop_code = 0
        nonfinite = False
        t_begin = time.perf_counter()

        def visible(li: int) -> int:
            if li == 0:
                return ghost[0] if self.rank > 0 else 0
            while (li, published[li] + 1) in pending and pending[(li, published[li] + 1)].query():
                del pending[(li, published[li] + 1)]
                published[li] += 1
            return published[li]

        def drained() -> bool:
            for li in range(1, nl + 1):
                visible(li)
            return all(consumed[li] == visible(li - 1) for li in range(1, nl + 1))

        def idle() -> bool:
            return all(ln.job is None for ln in self.lanes) and not pending

        def local_done() -> bool:
            if not drained() or not idle():  # drained() also retires completed publishes
                return False
            if eps is None:
                return all(stable[1:])
            return float(np.max(last[1:])) < eps

        def dispatch(ln: _Lane, li: int) -> None:
            i = lo + li - 1
            from_mailbox = li == 1 and self.rank > 0
            v = None if from_mailbox else visible(li - 1)
            vr = vrem[li]
            t0 = time.perf_counter_ns()
            busy[li] = True
            st = ln.stream
            vi = published[li] + sum(1 for (j, _) in pending if j == li)
            dst_slot = (vi + 1) % R
            with tp.stream_ctx(st):
                for ev in readers[li][dst_slot]:
                    st.wait_event(ev)
                readers[li][dst_slot] = []
                ops.apply(ln.fine, self.remb[li], ln.f[0], st)
                if self.delay_frac > 0.0:
                    tp.sleep_cycles(int(_unit(self.seed, i, int(counts[li])) * self.delay_frac *
                                        self.spin_cycles_per_tf), st)
                if from_mailbox:
                    tp.read_mailbox(self.mb_ring_ptr, self.slot_bytes, R, self.ws, ln.fresh[0],
                                    ln.mb, st)
                    ops.equal(ln.fresh[0], self.remb[li], ln.eq, st)
                else:
                    src_slot = v % R
                    ev_src = pub_events[li - 1].get(src_slot)
                    if ev_src is not None:
                        st.wait_event(ev_src)
                    ln.fresh[0].copy_(self.ring[li - 1, src_slot], non_blocking=True)
                    rd = tp.event(st)
                    readers[li - 1][src_slot].append(rd)
                    if v == vr:
                        ln.eq.fill_(1)
                    else:
                        ops.equal(ln.fresh[0], self.remb[li], ln.eq, st)
                ops.apply(ln.coarse, ln.fresh[0], ln.g[0], st)
                cur = self.ring[li, vi % R]
                dst = self.ring[li, dst_slot]
                ops.correct(ln.g, ln.f, self.grem[li:li + 1], cur.reshape(1, -1), dst.reshape(1, -1), ln.eq,
                            ln.delta, ln.flag, st)
                self.grem[li].copy_(ln.g[0], non_blocking=True)
                self.remb[li].copy_(ln.fresh[0], non_blocking=True)
                if li == nl and self.rank + 1 < W:
                    # push the new version into the next GPU's mailbox (P2P stores + release)
                    nxt = self.peer_ws[self.rank + 1]
                    tp.push(nxt + self.mb_off + ((vi + 1) % R) * self.slot_bytes, dst, nxt, vi + 1,
                            ln.ctr.data_ptr(), st)
                ln.host[0:1].copy_(ln.delta, non_blocking=True)
                ln.host[1:2].copy_(ln.flag.to(torch.float64), non_blocking=True)
                ln.host[2:3].copy_(ln.eq.to(torch.float64), non_blocking=True)
                ln.host[3:5].copy_(ln.mb[1:3].to(torch.float64), non_blocking=True)
                ev = tp.event(st)
                pub_events[li][dst_slot] = ev
                pending[(li, vi + 1)] = ev
            ln.job = (li, v, vr, t0, ev, from_mailbox)

        def finish(ln: _Lane) -> None:
            nonlocal events, pubcount, nonfinite
            li, v, vr, t0, ev, from_mailbox = ln.job
            ln.job = None
            h = ln.host.numpy() if hasattr(ln.host, "numpy") else ln.host
            if h[1] != 0.0:
                nonfinite = True
            if from_mailbox:
                if h[4] != 0.0:
                    raise RuntimeError("mailbox read overtaken by the producer (ring too small for the push rate)")
                v = int(h[3])
            d = float(h[0])
            fonly = (v == vr) or h[2] != 0.0
            last[li] = d
            vrem[li] = v
            consumed[li] = v
            stable[li] = bool(fonly)
            counts[li] += 1
            busy[li] = False
            events += 1
            pubcount += 1
            if self.record_trace:
                records.append((lo + li - 1, v, vr, 1 if fonly else 0, int(np.array([d]).view(np.int64)[0]), t0,
                                time.perf_counter_ns(), ln.index + 65536 * self.rank))

        def pick():
            # lowest slice with something to do first (the pipeline order of the
            # sweeps; any order is a valid asynchronous schedule); "round-robin"
            # walks a ticket over the slices instead
            nonlocal ticket
            for q in range(nl):
                if self.claim == "round-robin":
                    li = 1 + ticket % nl
                    ticket += 1
                else:
                    li = 1 + q
                if busy[li]:
                    continue
                if stable[li] and consumed[li] == visible(li - 1):
                    last[li] = 0.0  # an activation would reproduce the same value
                    continue
                if eps is not None and last[li] < eps and consumed[li] == visible(li - 1):
                    continue  # nothing new to consume and already below the threshold: stay put
                return li
            return None

        while True:
            progressed = False
            # retire in dispatch order so a consumer's record follows its
            # producer's (see async_streams: the audit replays record order)
            ready = [ln for ln in self.lanes if ln.job is not None and ln.job[4].query()]
            ready.sort(key=lambda ln: ln.job[3])
            for ln in ready:
                finish(ln)
                progressed = True
            if nonfinite and stop_code == 0:
                stop_code = STOP_NONFINITE
                self._post_stop(STOP_NONFINITE)
            if self.rank > 0:
                ghost[0] = self._ghost_version()
            done = local_done()
            if done != posted_done:
                cons0 = consumed[1] if self.rank > 0 else 0
                self._post_all([1 if done else 0, cons0, visible(nl), pubcount, events, 0, 0])
                posted_done = done
            bd = self._board()
            stop_slot = bd[W]
            if stop_slot[0] == 2:
                stop_code = int(stop_slot[1 + 0])
                break
            if done and self._consistent(bd) and self._consistent_again(bd):
                self._post_stop(STOP_CONVERGED)
                continue
            if self.timeout_s is not None and stop_code == 0 and time.perf_counter() - t_begin > self.timeout_s:
                stop_code = STOP_HORIZON  # wall-clock budget spent: stop every rank like a horizon
                self._post_stop(STOP_HORIZON)
                continue
            if events >= self.max_events and stop_code == 0:
                stop_code = STOP_HORIZON
                self._post_stop(STOP_HORIZON)
                continue
            if not done:
                for ln in self.lanes:
                    if ln.job is None:
                        li = pick()
                        if li is not None:
                            dispatch(ln, li)
                            progressed = True
            if not progressed:
                time.sleep(20e-6)  # lanes busy or nothing to do: poll again
        wall = time.perf_counter() - t_begin
        # the cut the stop decision saw: every rank idle, so nothing newer exists
        for ln in self.lanes:
            if ln.job is not None:
                ln.job[4].synchronize()
                finish(ln)
        snap = [visible(li) for li in range(nl + 1)]
        tp.synchronize()
        rows = torch.stack([self.ring[li, snap[li] % R] for li in range(1, nl + 1)])
        return dict(rows=rows, counts=counts, events=events, stop_code=stop_code, wall=wall,
                    records=np.array(records, dtype=np.int64).reshape(-1, 8), nonfinite=nonfinite)

    def _consistent(self, bd: np.ndarray) -> bool:
        W = self.world
        for r in range(W):
            s = bd[r]
            if s[0] <= 0 or s[0] % 2 or s[1 + W_DONE] != 1:
                return False
            if r > 0 and s[1 + W_CONSUMED] != bd[r - 1][1 + W_PUBHI]:
                return False
        return True

    def _consistent_again(self, bd: np.ndarray) -> bool:
        """Second collect: nobody re-posted in between (same sequence words)."""
        bd2 = self._board()
        return bool(np.array_equal(bd2[:self.world, 0], bd[:self.world, 0])) and self._consistent(bd2)

    def close(self):
        self.tp.close()


def _unit(seed: int, i: int, count: int) -> float:
    """splitmix64 of (seed, slice, activation) -> U[0, 1) (as async_rt.cu mix64)."""
    m = (1 << 64) - 1
    z = (seed ^ ((i << 32) & m) ^ count) & m
    z = (z + 0x9E3779B97F4A7C15) & m
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    z ^= z >> 31
    return (z >> 11) * (1.0 / 9007199254740992.0)


class TorchExchange:
    """Host plumbing over torch.distributed (handle exchange and the final
    reductions only — never on the data path)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group

    def all_gather_bytes(self, b: bytes) -> list[bytes]:
        out = [None] * self.dist.get_world_size(self.group)
        self.dist.all_gather_object(out, b, group=self.group)
        return out

    def all_gather_object(self, obj) -> list:
        out = [None] * self.dist.get_world_size(self.group)
        self.dist.all_gather_object(out, obj, group=self.group)
        return out

    def barrier(self):
        self.dist.barrier(group=self.group)


def device_coarse_init_rows(coarse, u0, first: int, last: int) -> torch.Tensor:
    """Rows first..last of the coarse initial iterate (parareal.py:54-63),
    chained from u0 with two working rows; the rank keeps only its rows."""
    from .parareal import _u0_tensor
    dev = f"cuda:{coarse.device}"
    out = torch.empty(last - first + 1, coarse.dim, dtype=coarse.dtype, device=dev)
    cur = torch.empty(1, coarse.dim, dtype=coarse.dtype, device=dev)
    nxt = torch.empty_like(cur)
    cur[0] = _u0_tensor(coarse, u0)
    if first == 0:
        out[0] = cur[0]
    for i in range(1, last + 1):
        coarse.apply_ptr(cur.data_ptr(), nxt.data_ptr(), 1, coarse.dim)
        cur, nxt = nxt, cur
        if i >= first:
            out[i - first] = cur[0]
    return out


def run_async_parareal_mp(coarse, fine, u0, p: int, epsilon: float | None = None, *, lanes: int = 2,
                          ring: int = 3, max_events: int = 200_000, delay_frac: float = 0.0, seed: int = 0,
                          record_trace: bool = False, gather: bool = False, group=None, transport=None, ops=None,
                          exchange=None, coarse_init_rows=None, claim: str = "lowest",
                          timeout_s: float | None = None) -> MPAsyncResult:
    """Asynchronous Parareal across processes/GPUs (see the module docstring).

    Every rank calls it with the same arguments. Returns this rank's
    ``MPAsyncResult`` (its rows; the gathered ``final`` on rank 0 when
    ``gather``). ``epsilon=None`` stops on exact quiescence. Raises
    ``HorizonExhausted`` when a rank reaches ``max_events`` activations first,
    ``ValueError`` on non-finite states (async_parareal.py:61-84 semantics).
    ``claim``: which ready slice a free lane takes — "lowest" (the pipeline
    order of the sweeps, default) or "round-robin" (a ticket over the slices);
    both are valid asynchronous schedules with the same reads and stop rule.
    ``timeout_s``: a wall-clock budget after which every rank stops as on the
    activation horizon (``HorizonExhausted``)."""
    import torch.distributed as dist
    if epsilon is not None and epsilon <= 0.0:
        raise ValueError(f"epsilon must be positive, got {epsilon}")
    if ring < 3:
        raise ValueError("the version ring needs at least three slots (seqlocked mailbox)")
    exchange = exchange or TorchExchange(group)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if p < world:
        raise ValueError(f"need at least one slice per rank, got p={p}, world={world}")
    transport = transport or CudaTransport(fine)
    ops = ops or GpuOps(coarse, fine)
    coarse_init_rows = coarse_init_rows or device_coarse_init_rows
    if claim not in ("lowest", "round-robin"):
        raise ValueError(f"claim must be 'lowest' or 'round-robin', got {claim!r}")
    rt = _Runtime(coarse, fine, u0, p, epsilon, lanes, ring, max_events, delay_frac, seed, record_trace, rank, world,
                  transport, ops, exchange, coarse_init_rows)
    rt.claim = claim
    rt.timeout_s = timeout_s
    exchange.barrier()  # every mailbox and board is initialised before any rank may push or post
    out = rt.run()
    exchange.barrier()  # no rank frees its workspace while a peer may still store into it
    info = exchange.all_gather_object({"counts": out["counts"], "events": out["events"], "wall": out["wall"],
                                       "code": out["stop_code"], "nonfinite": out["nonfinite"],
                                       "records": out["records"] if record_trace else None,
                                       "lo": rt.lo, "hi": rt.hi})
    counts = np.zeros(p + 1, dtype=np.int64)
    for d in info:
        counts[d["lo"]:d["hi"] + 1] = d["counts"][1:]
    code = max(d["code"] for d in info)
    final = None
    if gather:
        final = _gather_rows(out["rows"], rt, u0, coarse, exchange, p)
    rt.close()
    res = MPAsyncResult(rows=out["rows"], slices=(rt.lo, rt.hi), final=final, counts=counts,
                        activations=int(sum(d["events"] for d in info)),
                        stop_reason={STOP_CONVERGED: "converged", STOP_HORIZON: "max_events",
                                     STOP_NONFINITE: "nonfinite"}.get(code, "unknown"),
                        wall_s=float(max(d["wall"] for d in info)),
                        trace=np.concatenate([d["records"] for d in info]) if record_trace else None)
    if any(d["nonfinite"] for d in info):
        raise ValueError("block entries must be finite")
    if code == STOP_HORIZON:
        raise HorizonExhausted(f"no stop condition met within {max_events} activations per rank", res)
    return res


def _gather_rows(rows: torch.Tensor, rt: _Runtime, u0, coarse, exchange, p: int):
    """The whole iterate on rank 0 (row 0 = u0); other ranks return None.
    Host-staged through the exchange: meant for checking moderate sizes —
    at C5 scale keep the shards (``rows``)."""
    parts = exchange.all_gather_object(rows.detach().to("cpu"))
    if rt.rank != 0:
        return None
    from .parareal import _u0_tensor
    full = torch.empty(p + 1, rows.shape[1], dtype=rows.dtype, device=rows.device)
    full[0] = _u0_tensor(coarse, u0) if rows.device.type == "cuda" else torch.as_tensor(u0, dtype=rows.dtype)
    for (lo, hi), part in zip(async_partition(p, rt.world), parts):
        full[lo:hi + 1] = part.to(full.device)
    return full
