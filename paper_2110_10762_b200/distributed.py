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

The only data-path exchange is the 1-D chain edge lambda_{i-1} -> lambda_i
that crosses each GPU boundary once per sweep: one N*8-byte
NCCL send/recv. Everything else stays on the owning GPU. The inner engine is
pluggable so the protocol is unit-tested on CPU with gloo.
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


class ShardedSyncEngine:
    """One rank's share of the synchronous iteration. ``engine`` provides the
    local device work (default: parareal.SyncEngine on this rank's GPU)."""

    def __init__(self, coarse, fine, p_local: int, rank: int, world: int, engine=None):
        if engine is None:
            from .parareal import SyncEngine
            engine = SyncEngine(coarse, fine, p_local)
        self.eng = engine
        self.p = int(p_local)
        self.rank = int(rank)
        self.world = int(world)
        dev = self.eng.lam_a.device
        self._red = torch.zeros(2, dtype=torch.float64, device=dev)

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
            dist.recv(eng.lam_a[0], src=self.rank - 1)
            eng.init(eng.lam_a[0])
        if self.rank + 1 < self.world:
            dist.send(eng.lam_a[self.p].contiguous(), dst=self.rank + 1)

    def sweep(self, k: int, nxt: torch.Tensor, fine_done_event=None) -> None:
        """Global sweep k on this rank's shard; nxt receives the new iterate."""
        eng = self.eng
        k_loc = max(1, k - self.rank * self.p)
        live = k_loc <= self.p
        if live:
            eng.fine_batch(k_loc, fine_done_event)
        elif fine_done_event is not None:
            fine_done_event.record()
        chain_in = False
        if self.rank > 0:
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
        if self.rank + 1 < self.world:
            s1 = dist.isend(nxt[self.p].contiguous(), dst=self.rank + 1)
            s2 = dist.isend(eng.deltas[self.p:self.p + 1].contiguous(), dst=self.rank + 1)
            s1.wait()
            s2.wait()
        self._red[0:1].copy_(eng.dmax)
        self._red[1:2].copy_(eng.flag.to(torch.float64))
        dist.all_reduce(self._red, op=dist.ReduceOp.MAX)
        eng.prev = nxt

    def read_delta(self) -> float:
        vals = self._red.to("cpu")
        if vals[1] != 0.0:
            raise ValueError("block entries must be finite")
        return float(vals[0])


def run_parareal_sharded(coarse, fine, u0, p_local: int, epsilon: float, k_max: int | None = None,
                         engine=None) -> dict:
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
    sh = ShardedSyncEngine(coarse, fine, p_local, rank, world, engine=engine)
    sh.init(u0)
    deltas, k, stop = [], 0, "k_max"
    while k < cap:
        k += 1
        nxt = sh.lam_b if sh.prev is sh.lam_a else sh.lam_a
        sh.sweep(k, nxt)
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
    return {"k_final": k, "stop_reason": stop, "deltas": deltas, "shard": sh.prev.clone()}
