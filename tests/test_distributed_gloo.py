"""Multi-rank synchronous Parareal protocol (paper_2110_10762_b200/distributed.py)
on CPU: world_size 2 and 3 over gloo, with an oracle-backed test double of the
per-rank device engine. The sharded run must reproduce the single-process
run bitwise (same k, stop reason, deltas, iterate)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import heat_oracle as H


class CPUEngine:
    """Same interface as parareal.SyncEngine, numpy oracle propagators."""

    def __init__(self, coarse, fine, p):
        n = fine.n
        self.coarse, self.fine, self.p = coarse, fine, p
        z = lambda: torch.zeros(p + 1, n, dtype=torch.float64)  # noqa: E731
        self.lam_a, self.lam_b, self.fv, self.gcache = z(), z(), z(), z()
        self.deltas = torch.zeros(p + 1, dtype=torch.float64)
        self.dmax = torch.zeros(1, dtype=torch.float64)
        self.flag = torch.zeros(1, dtype=torch.int32)
        self.prev = self.lam_a

    def init(self, u0):
        self.lam_a[0] = torch.as_tensor(np.asarray(u0, dtype=float))
        self.lam_b[0] = self.lam_a[0]
        for i in range(1, self.p + 1):
            self.lam_a[i] = torch.from_numpy(self.coarse.apply(self.lam_a[i - 1].numpy()))
        self.gcache.copy_(self.lam_a)
        self.prev = self.lam_a

    def fine_batch(self, k, fine_done_event=None):
        self.fv[k:] = torch.from_numpy(self.fine.apply_batch(self.prev[k - 1:self.p].numpy()))

    def coarse_sweep(self, k, nxt, chain_in=False):
        prev = self.prev
        if not chain_in:
            nxt[k - 1] = prev[k - 1]
            self.deltas[k - 1] = 0.0
        for i in range(k, self.p + 1):
            g = torch.from_numpy(self.coarse.apply(nxt[i - 1].numpy()))
            fonly = (float(self.deltas[i - 1]) == 0.0) if (chain_in or i > k) else True
            v = self.fv[i].clone() if fonly else (g + self.fv[i]) - self.gcache[i]
            self.deltas[i] = float((v - prev[i]).abs().max())
            self.gcache[i] = g
            nxt[i] = v

    def reduce_delta(self, k):
        self.dmax[0] = self.deltas[k - 1:].max()

    def launches_per_sweep(self):
        return 0


def problem(n=64):
    a_d, a_o, c = H.heat1d_coeffs(n, 1.0, 0.5, -0.25)
    return H.Tridiag1D(n, a_d, a_o, c, 0.05, 1), H.Tridiag1D(n, a_d, a_o, c, 0.05, 20), H.sine_u0_1d(n, 8, 0)


def _worker(rank, world, port, p_local, eps, out, edge="nccl"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2110_10762_b200 import distributed as D
    coarse, fine, u0 = problem()
    eng = CPUEngine(coarse, fine, p_local)
    if edge == "mailbox":
        # the peer-memory chain edge (K7) over the shared-memory test transport
        import sys
        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        from async_mp_doubles import ShmTransport

        from paper_2110_10762_b200.async_mp import TorchExchange
        edge = D.MailboxEdge(eng.lam_a[0], rank, world, ShmTransport(), TorchExchange(), wait="host")
    res = D.run_parareal_sharded(coarse, fine, u0, p_local, eps, engine=eng, edge=edge)
    shards = [torch.zeros_like(res["shard"]) for _ in range(world)]
    dist.all_gather(shards, res["shard"])
    if rank == 0:
        full = torch.cat([shards[0]] + [s[1:] for s in shards[1:]]).numpy()
        np.savez(out, full=full, k=res["k_final"], stop=res["stop_reason"], deltas=np.array(res["deltas"]))
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("edge", ["nccl", "mailbox"])
@pytest.mark.parametrize("world,p_local,eps", [(2, 4, 1e-9), (3, 3, 0.0), (2, 5, 1e-4)])
def test_sharded_run_equals_single_process(tmp_path, world, p_local, eps, edge):
    out = str(tmp_path / "res.npz")
    mp.start_processes(_worker, args=(world, _free_port(), p_local, eps, out, edge), nprocs=world, join=True,
                       start_method="spawn")
    got = np.load(out)
    coarse, fine, u0 = problem()
    ref = H.run_parareal(coarse, fine, u0, p_local * world, eps)
    assert int(got["k"]) == ref.k_final
    assert str(got["stop"]) == ref.stop_reason
    assert np.array_equal(got["deltas"], np.array(ref.deltas))
    assert np.array_equal(got["full"], ref.iterates[-1])


# ------------------------------------------------ asynchronous, across ranks
class FakeAsyncDomain:
    """Test double of distributed.NativeAsyncDomain: checks the handle
    exchange and the call order, and 'runs' the domain by landing on the
    exact-quiescence answer (the sequential fine solution),
    one activation per slice, trace records at global event = slice."""

    calls = []

    def __init__(self, coarse, fine, p, lo, hi, world, rank, cap):
        self.fine, self.p, self.lo, self.hi, self.world, self.rank, self.cap = fine, p, lo, hi, world, rank, cap
        self.state = "created"

    def ipc_handle(self):
        return bytes([self.rank + 1]) * 64

    def connect(self, handles, nloc_all):
        assert self.state == "created"
        assert [h for h in handles] == [bytes([x + 1]) * 64 for x in range(self.world)]
        assert sum(nloc_all) == self.p and nloc_all[self.rank] == self.hi - self.lo + 1
        self.state = "connected"

    def reset(self, rows):
        assert self.state == "connected" and rows.shape[0] == self.hi - self.lo + 2
        self.rows = rows.clone()
        self.state = "reset"

    def launch(self, eps, max_events, delay, seed):
        assert self.state == "reset"
        seq = H.sequential_fine_solve(self.fine, self.u0, self.p)
        self.result = torch.from_numpy(seq[self.lo - 1:self.hi + 1].copy())
        self.state = "launched"

    def synchronize(self):
        pass

    def collect(self, rows_out):
        assert self.state == "launched"
        rows_out.copy_(self.result)
        nloc = self.hi - self.lo + 1
        counts = np.ones(nloc + 1, dtype=np.int64)
        counts[0] = 0
        info = np.array([self.p, 1, 0, 0, 1, nloc], dtype=np.int64)
        trace = np.zeros((self.cap, 8), dtype=np.int64)
        for gi in range(self.lo, self.hi + 1):
            if gi - 1 < self.cap:
                trace[gi - 1, 0] = gi
                trace[gi - 1, 3] = 1
                trace[gi - 1, 7] = self.rank * 65536
        return counts, info, trace

    def close(self):
        self.state = "closed"


def _async_worker(rank, world, port, p, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2110_10762_b200 import distributed as D
    coarse, fine, u0 = problem()

    def factory(*args):
        d = FakeAsyncDomain(*args)
        d.u0 = u0
        return d

    def cinit_rows(c, u, first, last):
        lam = np.zeros((last + 1, len(u)))
        lam[0] = u
        for i in range(1, last + 1):
            lam[i] = c.apply(lam[i - 1])
        return torch.from_numpy(lam[first:])

    res = D.run_async_parareal_distributed(coarse, fine, u0, p, None, record_trace=True, trace_cap=p,
                                           domain_factory=factory, coarse_init_rows=cinit_rows)
    final = res["final"].numpy() if res["final"] is not None else np.zeros(0)
    np.savez(out + f".{rank}.npz", final=final, rows=res["rows"].numpy(), counts=res["counts"], trace=res["trace"],
             stop=res["stop_reason"], kappa=res["kappa"], slices=np.array(res["slices"]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,p", [(2, 6), (3, 7), (4, 4)])
def test_async_distributed_protocol(tmp_path, world, p):
    from paper_2110_10762_b200.distributed import async_partition
    out = str(tmp_path / "a")
    mp.start_processes(_async_worker, args=(world, _free_port(), p, out), nprocs=world, join=True,
                       start_method="spawn")
    coarse, fine, u0 = problem()
    seq = H.sequential_fine_solve(fine, u0, p)
    parts = async_partition(p, world)
    for r in range(world):
        got = np.load(out + f".{r}.npz")
        lo, hi = parts[r]
        assert np.array_equal(got["rows"], seq[lo:hi + 1])  # each rank holds only its own slices
        if r == 0:
            assert np.array_equal(got["final"], seq)  # gathered to rank 0
        else:
            assert got["final"].size == 0
        assert np.array_equal(got["counts"], np.r_[0, np.ones(p, dtype=np.int64)])
        assert str(got["stop"]) == "converged" and int(got["kappa"]) == 1
        assert tuple(got["slices"]) == parts[r]
        assert np.array_equal(got["trace"][:, 0], np.arange(1, p + 1))  # merged from all ranks
        owners = got["trace"][:, 7] // 65536
        assert all(parts[o][0] <= i <= parts[o][1] for o, i in zip(owners, got["trace"][:, 0]))


def test_async_partition_matches_the_device_split():
    from paper_2110_10762_b200.distributed import async_partition
    for p in range(1, 40):
        for w in range(1, min(p, 9) + 1):
            parts = async_partition(p, w)
            assert parts[0][0] == 1 and parts[-1][1] == p
            assert all(parts[i][1] + 1 == parts[i + 1][0] for i in range(w - 1))
            sizes = [h - l + 1 for l, h in parts]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        async_partition(3, 4)
