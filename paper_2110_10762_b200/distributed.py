"""Multi-GPU synchronous Parareal: contiguous time-slice shards, one process
per GPU (torch.distributed, NCCL over NVLink/NVSwitch).

Rank r owns global slices r*p_local+1 .. (r+1)*p_local; its local row 0 holds
global slice r*p_local (owned by rank r-1). Per sweep k (PAPER.md:675-708,
Algorithm 1, and parareal.py:119-127):

  1. F over the rank's live slices — independent, one batched launch;
  2. receive the NEW value of the boundary slice (and its delta, which
     decides the F-only branch of the first local slice) from rank r-1;
  3. fused coarse chain + correction + deltas over the local slices;
  4. send the last local slice's new value and delta to rank r+1;
  5. one 16-byte MAX all-reduce of (delta, non-finite flag).

Wavefront overlap (Algorithm 1: "processor i-1 starts
applying F before processor i"): as soon as rank r's own chain segment of
sweep k is done, F of sweep k+1 over its slices is launched on a side stream
(its inputs are all local by then: the rank's new rows and the boundary row
received in step 2), so it runs while the downstream ranks are still in
their chain of sweep k and while the delta is reduced; a stop at k discards
it (``finish``).

The only data-path exchange is the 1-D chain edge lambda_{i-1} -> lambda_i
that crosses each GPU boundary once per sweep. By default it
goes over peer memory (``MailboxEdge``, K7): rank r's GPU pushes the boundary
slice and its delta straight into rank r+1's mailbox with SM stores and a
system-scope release of the sweep number (``pint_mailbox_push``), and rank
r+1's stream waits for that version with a one-thread device poll
(``pint_mailbox_wait``; a host poll when two ranks share a device, e.g. the
one-GPU tests) before its chain — no NCCL on the data path. ``edge="nccl"``
keeps the NCCL send/recv. Everything else stays on the owning GPU. The inner
engine and the transport are pluggable so the protocol is unit-tested on CPU
with gloo.
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def init_process_group() -> None:
    if dist.is_initialized():
        return
    backend = "nccl" if torch.cuda.is_available() else "gloo"
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    if backend == "nccl":
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
    dist.init_process_group(backend=backend)


def destroy() -> None:
    if dist.is_initialized():
        dist.destroy_process_group()


def barrier() -> None:
    if dist.is_initialized():
        if dist.get_backend() == "nccl":
            dist.barrier(device_ids=[torch.cuda.current_device()])
        else:
            dist.barrier()


def _red_device():
    return torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")


def max_over_ranks(x: float) -> float:
    t = torch.tensor([float(x)], dtype=torch.float64, device=_red_device())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class MailboxEdge:
    """The chain edge of the sharded synchronous sweep over peer memory.
    Two slots of [boundary row | its delta] in every rank's shared workspace,
    guarded by one version word = the message sequence number (1 = the coarse
    initial value, then one per sweep; both ends count their messages, so
    repeated sweeps with the same k — the bench — stay ordered). A slot is
    rewritten two messages later, after the per-sweep delta all-reduce that
    the consumer can only pass once it has read it — so no flow control."""

    def __init__(self, like: torch.Tensor, rank: int, world: int, transport, exchange, wait: str = "auto"):
        self.tp, self.rank, self.world = transport, rank, world
        n, dt = like.shape[-1], like.dtype
        esz = like.element_size()
        self.row_pad = (n * esz + 255) // 256 * 256
        self.slot = self.row_pad + 256
        self.ws = transport.alloc(256 + 2 * self.slot)
        self.ver = transport.view(self.ws, (1,), torch.int64)
        self.rows = [transport.view(self.ws + 256 + q * self.slot, (n,), dt) for q in range(2)]
        self.dls = [transport.view(self.ws + 256 + q * self.slot + self.row_pad, (1,), torch.float64)
                    for q in range(2)]
        dev = like.device
        self.stage = torch.zeros(self.slot, dtype=torch.uint8, device=dev)
        self.stage_row = self.stage[:n * esz].view(dt)
        self.stage_dl = self.stage[self.row_pad:self.row_pad + 8].view(torch.float64)
        self.ctr = torch.zeros(1, dtype=torch.int32, device=dev)
        self.timed_out = torch.zeros(1, dtype=torch.int32, device=dev)
        self.word_host = torch.zeros(1, dtype=torch.int64, pin_memory=dev.type == "cuda")
        handle = transport.export(self.ws)
        handles = exchange.all_gather_bytes(handle)
        self.peer_next = transport.open(handles[rank + 1], self.ws, handle) if rank + 1 < world else None
        if wait == "auto":
            import socket
            where = exchange.all_gather_object((socket.gethostname(), str(dev)))
            wait = "device" if dev.type == "cuda" and len(set(where)) == world else "host"
        self.wait = wait
        self.sent = 0
        self.received = 0

    def recv(self, k: int, row0: torch.Tensor, delta0: torch.Tensor) -> None:
        """Consumer: this sweep's new boundary row and delta from rank-1
        (k = 0: the coarse initial value); message sequence numbers 1, 2, ..."""
        self.received += 1
        k = self.received
        if self.wait == "device":
            self.tp.wait_version(self.ver.data_ptr(), k, self.timed_out, torch.cuda.current_stream(row0.device))
        else:
            st = torch.cuda.current_stream(row0.device) if row0.device.type == "cuda" else None
            while self.tp.read_word(self.ver, self.word_host, st) < k:
                pass
        q = k % 2
        row0.copy_(self.rows[q])
        delta0.copy_(self.dls[q])

    def send(self, k: int, row: torch.Tensor, delta: torch.Tensor) -> None:
        """Producer: push the boundary row and delta into rank+1's slot k % 2,
        then publish its sequence number (SM stores + system-scope release)."""
        self.sent += 1
        k = self.sent
        self.stage_row.copy_(row)
        self.stage_dl.copy_(delta)
        st = torch.cuda.current_stream(row.device) if row.device.type == "cuda" else None
        self.tp.push(self.peer_next + 256 + (k % 2) * self.slot, self.stage, self.peer_next, k, self.ctr.data_ptr(),
                     st)

    def check(self) -> None:
        if int(self.timed_out.item()) != 0:
            raise RuntimeError("chain edge: the previous rank's boundary state did not arrive (mailbox wait timed out)")

    def close(self) -> None:
        self.tp.close()


class ShardedSyncEngine:
    """One rank's share of the synchronous iteration. ``engine`` provides the
    local device work (default: parareal.SyncEngine on this rank's GPU);
    ``edge`` the chain edge ("mailbox": peer memory, K7; "nccl": send/recv;
    or a MailboxEdge built with a test transport)."""

    def __init__(self, coarse, fine, p_local: int, rank: int, world: int, engine=None, edge="mailbox"):
        if engine is None:
            from .parareal import SyncEngine
            engine = SyncEngine(coarse, fine, p_local)
        self.eng = engine
        self.p = int(p_local)
        self.rank = int(rank)
        self.world = int(world)
        dev = self.eng.lam_a.device
        # the per-sweep reduction lives where the process group reduces (NCCL: the GPU; gloo: the host)
        red_dev = _red_device() if dist.is_initialized() else dev
        self._red = torch.zeros(2, dtype=torch.float64, device=red_dev)
        self._spec = None
        self._side = torch.cuda.Stream(device=dev) if dev.type == "cuda" else None
        if edge == "mailbox" and world > 1:
            from .async_mp import CudaTransport, TorchExchange
            edge = MailboxEdge(self.eng.lam_a[0], rank, world, CudaTransport(fine), TorchExchange())
        self.edge = edge if isinstance(edge, MailboxEdge) else None

    # views of the inner engine (bench resets the iterate through these)
    @property
    def lam_a(self):
        return self.eng.lam_a

    @property
    def lam_b(self):
        return self.eng.lam_b

    @property
    def prev(self):
        return self.eng.prev

    @prev.setter
    def prev(self, v):
        self.eng.prev = v

    def launches_per_sweep(self) -> int:
        return self.eng.launches_per_sweep()

    def init(self, u0) -> None:
        """Coarse initialisation, chained across ranks (parareal.py:54-63)."""
        eng = self.eng
        if self.rank == 0:
            eng.init(u0)
        else:
            if self.edge is not None:
                self.edge.recv(0, eng.lam_a[0], eng.deltas[0:1])
            else:
                dist.recv(eng.lam_a[0], src=self.rank - 1)
            eng.init(eng.lam_a[0])
        if self.rank + 1 < self.world:
            if self.edge is not None:
                self.edge.send(0, eng.lam_a[self.p], eng.deltas[self.p:self.p + 1])
            else:
                dist.send(eng.lam_a[self.p].contiguous(), dst=self.rank + 1)

    def _k_loc(self, k: int) -> int:
        return max(1, k - self.rank * self.p)

    def _launch_spec(self, k_loc: int):
        """F of the next sweep over this rank's live slices, off the critical path."""
        if self._side is None:  # host engine (tests): runs in order
            self.eng.fine_batch(k_loc)
            return None
        main = torch.cuda.current_stream(self._side.device)
        self._side.wait_stream(main)
        with torch.cuda.stream(self._side):
            self.eng.fine_batch(k_loc)
        ev = torch.cuda.Event()
        ev.record(self._side)
        return ev

    def finish(self) -> None:
        """Join a speculative F the run did not use (its buffers stay alive)."""
        spec, self._spec = self._spec, None
        if spec is not None and spec[1] is not None:
            torch.cuda.current_stream(self._side.device).wait_event(spec[1])

    def sweep(self, k: int, nxt: torch.Tensor, fine_done_event=None, speculate: bool = False) -> None:
        """Global sweep k on this rank's shard; nxt receives the new iterate.
        speculate: launch sweep k+1's F right after this rank's chain."""
        eng = self.eng
        k_loc = self._k_loc(k)
        live = k_loc <= self.p
        spec, self._spec = self._spec, None
        if live:
            if spec is not None and spec[0] == k:
                if spec[1] is not None:
                    torch.cuda.current_stream(self._side.device).wait_event(spec[1])
                if fine_done_event is not None:
                    fine_done_event.record()
            else:
                if spec is not None and spec[1] is not None:
                    torch.cuda.current_stream(self._side.device).wait_event(spec[1])
                eng.fine_batch(k_loc, fine_done_event)
        elif fine_done_event is not None:
            fine_done_event.record()
        chain_in = False
        if self.rank > 0:
            if self.edge is not None:
                self.edge.recv(k, nxt[0], eng.deltas[0:1])
            else:
                w1 = dist.irecv(nxt[0], src=self.rank - 1)
                w2 = dist.irecv(eng.deltas[0:1], src=self.rank - 1)
                w1.wait()
                w2.wait()
            chain_in = k_loc == 1
        if live:
            eng.coarse_sweep(k_loc, nxt, chain_in=chain_in)
            eng.reduce_delta(k_loc)
        else:
            nxt.copy_(eng.prev)
            eng.deltas.zero_()
            eng.dmax.zero_()
        if speculate and self._k_loc(k + 1) <= self.p:
            # this rank's rows of sweep k are final: F(k+1) can start now
            eng.prev = nxt
            self._spec = (k + 1, self._launch_spec(self._k_loc(k + 1)))
        if self.rank + 1 < self.world:
            if self.edge is not None:
                self.edge.send(k, nxt[self.p], eng.deltas[self.p:self.p + 1])
            else:
                s1 = dist.isend(nxt[self.p].contiguous(), dst=self.rank + 1)
                s2 = dist.isend(eng.deltas[self.p:self.p + 1].contiguous(), dst=self.rank + 1)
                s1.wait()
                s2.wait()
        self._red[0:1].copy_(eng.dmax)
        self._red[1:2].copy_(eng.flag.to(torch.float64))
        dist.all_reduce(self._red, op=dist.ReduceOp.MAX)
        eng.prev = nxt

    def read_delta(self) -> float:
        if self.edge is not None:
            self.edge.check()
        vals = self._red.to("cpu")
        if vals[1] != 0.0:
            raise ValueError("block entries must be finite")
        return float(vals[0])


def run_parareal_sharded(coarse, fine, u0, p_local: int, epsilon: float, k_max: int | None = None,
                         engine=None, edge="mailbox") -> dict:
    """Synchronous Parareal over all ranks (P = p_local * world slices) with
    the reference's stop rules (parareal.py:99-138). Returns this rank's final
    shard and the global stop bookkeeping."""
    rank, world = dist.get_rank(), dist.get_world_size()
    p = p_local * world
    if epsilon < 0.0:
        raise ValueError(f"epsilon must be nonnegative, got {epsilon}")
    cap = p if k_max is None else min(int(k_max), p)
    if cap < 1:
        raise ValueError(f"iteration budget must allow k >= 1, got k_max={k_max}")
    sh = ShardedSyncEngine(coarse, fine, p_local, rank, world, engine=engine, edge=edge)
    sh.init(u0)
    deltas, k, stop = [], 0, "k_max"
    try:
        while k < cap:
            k += 1
            nxt = sh.lam_b if sh.prev is sh.lam_a else sh.lam_a
            sh.sweep(k, nxt, speculate=k < cap)
            d = sh.read_delta()
            deltas.append(d)
            if d < epsilon:
                stop = "threshold"
                break
            if k == p:
                stop = "exact"
                break
            if k == cap:
                stop = "k_max"
                break
    finally:
        sh.finish()
    return {"k_final": k, "stop_reason": stop, "deltas": deltas, "shard": sh.prev.clone()}


# ================================================= asynchronous, across GPUs
def async_partition(p: int, world: int) -> list[tuple[int, int]]:
    """Contiguous slice ranges (lo, hi), 1-based inclusive, one per rank —
    the same split the C runtime uses (async_rt.cu, pint_async_run_domains)."""
    if world < 1 or p < world:
        raise ValueError(f"need 1 <= world <= p, got world={world}, p={p}")
    return [(1 + p * r // world, p * (r + 1) // world) for r in range(world)]


class NativeAsyncDomain:
    """One rank's domain of the device async runtime (include/pint_abi.h,
    pint_async_domain_*): a workspace with the rank's version rings, a ghost
    mailbox for the predecessor slice and a status board, exported to the
    peers as a CUDA IPC handle. The kernel pushes the rank's last slice into
    the next rank's mailbox with P2P stores (async_rt.cu)."""

    HANDLE_BYTES = 64

    def __init__(self, coarse, fine, p: int, lo: int, hi: int, world: int, index: int, trace_cap: int = 0):
        import ctypes

        from . import _native
        self._ct = ctypes
        self.lib = _native.load_library()
        self._native = _native
        self.fine, self.coarse = fine, coarse
        self.ctx = fine._ctx.handle
        self.lo, self.hi, self.nloc = lo, hi, hi - lo + 1
        self.trace_cap = int(trace_cap)
        h = ctypes.c_void_p()
        rc = self.lib.pint_async_domain_create(fine.handle, coarse.handle, int(p), int(lo), int(hi), int(world),
                                               int(index), 0, self.trace_cap, ctypes.byref(h))
        _native.check(rc, self.ctx, "pint_async_domain_create")
        self.handle = h

    def ipc_handle(self) -> bytes:
        buf = (self._ct.c_ubyte * self.HANDLE_BYTES)()
        rc = self.lib.pint_async_domain_ipc_handle(self.handle, buf)
        self._native.check(rc, self.ctx, "pint_async_domain_ipc_handle")
        return bytes(buf)

    def connect(self, handles: list[bytes], nloc_all: list[int]) -> None:
        import numpy as np
        blob = b"".join(handles)
        arr = (self._ct.c_ubyte * len(blob)).from_buffer_copy(blob)
        nl = np.asarray(nloc_all, dtype=np.int64)
        rc = self.lib.pint_async_domain_connect(self.handle, arr, nl.ctypes.data_as(self._ct.c_void_p))
        self._native.check(rc, self.ctx, "pint_async_domain_connect")

    def reset(self, rows: torch.Tensor) -> None:
        from . import _device
        rc = self.lib.pint_async_domain_reset(self.handle, self._ct.c_void_p(rows.data_ptr()),
                                              self._ct.c_void_p(_device.stream_ptr(self.fine.device)))
        self._native.check(rc, self.ctx, "pint_async_domain_reset")

    def launch(self, epsilon: float, max_events: int, delay_frac: float, seed: int) -> None:
        from . import _device
        arr = (self._ct.c_void_p * 1)(self.handle.value)
        rc = self.lib.pint_async_domain_launch(1, arr, float(epsilon), int(max_events), float(delay_frac),
                                               int(seed), self._ct.c_void_p(_device.stream_ptr(self.fine.device)))
        self._native.check(rc, self.ctx, "pint_async_domain_launch")

    def synchronize(self) -> None:
        torch.cuda.synchronize(self.fine.device)

    def collect(self, rows_out: torch.Tensor):
        import numpy as np

        from . import _device
        counts = np.zeros(self.nloc + 1, dtype=np.int64)
        info = np.zeros(6, dtype=np.int64)
        trace = np.zeros((max(self.trace_cap, 1), 8), dtype=np.int64)
        rc = self.lib.pint_async_domain_collect(self.handle, self._ct.c_void_p(rows_out.data_ptr()),
                                                counts.ctypes.data_as(self._ct.c_void_p),
                                                info.ctypes.data_as(self._ct.c_void_p),
                                                trace.ctypes.data_as(self._ct.c_void_p), self.trace_cap,
                                                self._ct.c_void_p(_device.stream_ptr(self.fine.device)))
        self._native.check(rc, self.ctx, "pint_async_domain_collect")
        return counts, info, trace[:self.trace_cap]

    def close(self) -> None:
        if getattr(self, "handle", None):
            self.lib.pint_async_domain_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def run_async_parareal_distributed(coarse, fine, u0, p: int, epsilon: float | None = None, *,
                                   max_events: int = 200_000, delay_frac: float = 0.0, seed: int = 0,
                                   record_trace: bool = False, trace_cap: int | None = None,
                                   domain_factory=None, coarse_init_rows=None, gather: bool = True) -> dict:
    """Asynchronous Parareal over all ranks (Algorithm 2; reference
    run_async_parareal, async_parareal.py:61-84), one domain of contiguous
    slices per GPU. The data path is peer memory only: each rank's kernel
    pushes its last slice into the next rank's mailbox with P2P stores and the
    stop decision is taken on device from the status boards. NCCL reduces the
    outcome afterwards (stop code, non-finite flag, activation counts, the
    trace) and gathers the final iterate.

    Memory per rank: only the rank's rows (lo-1 .. hi) of the coarse initial
    iterate are formed (the chain from u0 is run up to hi with two working
    rows), and the final iterate is gathered to rank 0 (``gather``) instead of
    being assembled on every rank.

    Returns {"rows": this rank's final slices lo..hi, "final": (p+1) x N
    tensor on rank 0 when ``gather`` (None elsewhere), "counts",
    "activations", "stop_reason", "kappa", "wall_s", "trace", "slices"}.
    ``domain_factory(coarse, fine, p, lo, hi, world, rank, trace_cap)`` and
    ``coarse_init_rows(coarse, u0, first, last) -> rows first..last`` replace
    the native pieces (the CPU tests drive the protocol with test doubles)."""
    import time

    import numpy as np

    rank, world = dist.get_rank(), dist.get_world_size()
    if epsilon is not None and epsilon <= 0.0:
        raise ValueError(f"epsilon must be positive, got {epsilon}")
    parts = async_partition(p, world)
    lo, hi = parts[rank]
    if getattr(fine, "is_tridiagonal", False):
        from .model import with_register_layout
        coarse = with_register_layout(coarse, fine.info.points_per_thread)
    if coarse_init_rows is None:
        from .async_mp import device_coarse_init_rows as coarse_init_rows
    # rows lo-1 .. hi, chained from u0 on every rank: bitwise identical, no exchange
    lam = coarse_init_rows(coarse, u0, lo - 1, hi)
    dev = lam.device
    cap = int(trace_cap if trace_cap is not None else min(max_events, 1_000_000)) if record_trace else 0
    factory = domain_factory or NativeAsyncDomain
    dom = factory(coarse, fine, p, lo, hi, world, rank, cap)
    # exchange the workspace handles (host plumbing; 64 bytes per rank)
    hb = torch.tensor(list(dom.ipc_handle()), dtype=torch.uint8, device=_red_device())
    allh = [torch.zeros_like(hb) for _ in range(world)]
    dist.all_gather(allh, hb)
    handles = [bytes(t.cpu().tolist()) for t in allh]
    dom.connect(handles, [h_ - l_ + 1 for l_, h_ in parts])
    dom.reset(lam.contiguous())
    barrier()  # every mailbox and board is reset before any rank may push
    t0 = time.perf_counter()
    dom.launch(-1.0 if epsilon is None else float(epsilon), max_events, delay_frac, seed)
    dom.synchronize()
    wall = time.perf_counter() - t0
    barrier()  # no rank frees its workspace while a peer may still store into it
    rows = torch.empty(hi - lo + 2, lam.shape[1], dtype=lam.dtype, device=dev)
    counts, info, trace = dom.collect(rows)
    barrier()
    dom.close()
    # ---- the final convergence reduction (NCCL)
    red = torch.tensor([float(info[1]), float(info[2]), wall], dtype=torch.float64, device=_red_device())
    dist.all_reduce(red, op=dist.ReduceOp.MAX)
    stop_code, nonfinite, wall_max = int(red[0].item()), int(red[1].item()), float(red[2].item())
    cnt = torch.zeros(p + 1, dtype=torch.int64, device=_red_device())
    cnt[lo:hi + 1] = torch.as_tensor(counts[1:], device=cnt.device)
    dist.all_reduce(cnt, op=dist.ReduceOp.SUM)
    full = _gather_final(rows, parts, p, rank, world) if gather else None
    tr = None
    if cap > 0:
        tt = torch.as_tensor(trace, device=_red_device())
        dist.all_reduce(tt, op=dist.ReduceOp.SUM)  # each record was written by exactly one rank
        n = min(int(info[0]), cap)
        tr = tt[:n].cpu().numpy()
    if nonfinite:
        raise ValueError("block entries must be finite")
    counts_all = cnt.cpu().numpy()
    out = {"rows": rows[1:], "final": None if full is None else full.to(dev), "counts": counts_all, "activations": int(info[0]),
           "stop_reason": {1: "converged", 2: "max_events"}.get(stop_code, "unknown"),
           "kappa": int(counts_all[1:].max()), "wall_s": wall_max, "trace": tr, "slices": (lo, hi)}
    return out


def _gather_final(rows: torch.Tensor, parts, p: int, rank: int, world: int):
    """The final iterate on rank 0 only: every rank sends its owned rows
    (padded to the largest shard so the collective has one shape); row 0 =
    u0 from rank 0. Nothing of size (p+1) x N is allocated on other ranks."""
    dev = _red_device()
    width = max(h - l + 1 for l, h in parts)
    mine = torch.zeros(width, rows.shape[1], dtype=rows.dtype, device=dev)
    lo, hi = parts[rank]
    mine[:hi - lo + 1] = rows[1:].to(dev)
    bufs = [torch.empty_like(mine) for _ in range(world)] if rank == 0 else None
    dist.gather(mine, gather_list=bufs, dst=0)
    if rank != 0:
        return None
    full = torch.empty(p + 1, rows.shape[1], dtype=rows.dtype, device=dev)
    full[0] = rows[0].to(dev)
    for (l_, h_), b in zip(parts, bufs):
        full[l_:h_ + 1] = b[:h_ - l_ + 1]
    return full
