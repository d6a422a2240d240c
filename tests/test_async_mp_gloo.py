"""Multi-process asynchronous runtime (paper_2110_10762_b200/async_mp.py) on
CPU: world sizes 1, 2 and 3 over gloo, each rank a real OS process holding
only its slices, the predecessor pushed through a shared-memory mailbox
(seqlocked) and termination decided from status boards — the device
transport/propagators replaced by tests/async_mp_doubles.py. Checks the
reference's async properties (async_parareal.py:61-84; test_async_parareal.py
78-88): exact quiescence lands bitwise on the sequential fine solution, the
eps stop is drained with every last change below eps."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, p, n, eps, lanes, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from async_mp_doubles import CpuOps, FakeProp, ShmTransport

        from paper_2110_10762_b200.async_mp import run_async_parareal_mp
        ops = CpuOps(n)
        prop = FakeProp(n)
        s = np.arange(1, n + 1) / (n + 1)
        u0 = np.sin(np.pi * s) + 0.3 * np.sin(3 * np.pi * s)
        res = run_async_parareal_mp(prop, prop, u0, p, eps, lanes=lanes, transport=ShmTransport(), ops=ops,
                                    coarse_init_rows=ops.coarse_init_rows, gather=True, record_trace=True)
        rows = res.rows.numpy()
        np.save(os.path.join(out_dir, f"rows{rank}.npy"), rows)
        if rank == 0:
            seq = ops.fine_seq(torch.as_tensor(u0), p).numpy()
            np.save(os.path.join(out_dir, "final.npy"), res.final.numpy())
            np.save(os.path.join(out_dir, "seq.npy"), seq)
            np.save(os.path.join(out_dir, "counts.npy"), res.counts)
            with open(os.path.join(out_dir, "stop.txt"), "w") as f:
                f.write(f"{res.stop_reason} {res.activations} {len(res.trace)}")
    finally:
        dist.destroy_process_group()


def _run(tmp_path, world, p, n=24, eps=None, lanes=2):
    port = _free_port()
    mp.spawn(_worker, args=(world, port, p, n, eps, lanes, str(tmp_path)), nprocs=world, join=True)
    final = np.load(tmp_path / "final.npy")
    seq = np.load(tmp_path / "seq.npy")
    stop, acts, ntr = open(tmp_path / "stop.txt").read().split()
    return final, seq, stop, int(acts), int(ntr), np.load(tmp_path / "counts.npy")


@pytest.fixture(autouse=True)
def _path():
    here = os.path.dirname(os.path.abspath(__file__))
    root = os.path.dirname(here)
    old = os.environ.get("PYTHONPATH", "")
    os.environ["PYTHONPATH"] = os.pathsep.join([here, root, old])
    yield
    os.environ["PYTHONPATH"] = old


@pytest.mark.parametrize("world,p", [(1, 6), (2, 8), (3, 9), (3, 5)])
def test_quiescence_equals_sequential_fine_bitwise(tmp_path, world, p):
    final, seq, stop, acts, ntr, counts = _run(tmp_path, world, p)
    assert stop == "converged"
    assert np.array_equal(final, seq)  # finite termination, bitwise (test_async_parareal.py:78-88)
    assert ntr == acts and counts[1:].min() >= 1
    assert counts[1:].sum() == acts


@pytest.mark.parametrize("world,p", [(2, 8), (3, 9)])
def test_eps_stop_is_drained_and_below_eps(tmp_path, world, p):
    eps = 1e-6
    final, seq, stop, acts, ntr, counts = _run(tmp_path, world, p, eps=eps)
    assert stop == "converged"
    # the stop predicate held on a consistent cut: the final iterate is a
    # fixed point of the two-slot update up to eps-sized changes
    err = np.max(np.abs(final - seq))
    assert err < 1e3 * eps, err


def _edge_worker(rank, world, port, p, n, mode, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from async_mp_doubles import CpuOps, FakeProp, ShmTransport

        from paper_2110_10762_b200.async_mp import run_async_parareal_mp
        from paper_2110_10762_b200.errors import HorizonExhausted
        ops = CpuOps(n, steps=400, r_f=2.0) if mode == "nonfinite" else CpuOps(n)
        prop = FakeProp(n)
        s = np.arange(1, n + 1) / (n + 1)
        u0 = np.sin(np.pi * s) + 0.3 * np.sin(3 * np.pi * s) + 0.01 * np.sin(n * np.pi * s / 2)
        kw = {"max_events": 3} if mode == "horizon" else {}
        try:
            run_async_parareal_mp(prop, prop, u0, p, None, lanes=2, transport=ShmTransport(), ops=ops,
                                  coarse_init_rows=ops.coarse_init_rows, **kw)
            got = "none"
        except HorizonExhausted as exc:
            got = f"horizon {exc.trace.stop_reason}"
        except ValueError as exc:
            got = f"value {exc}"
        with open(os.path.join(out_dir, f"r{rank}.txt"), "w") as f:
            f.write(got)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["horizon", "nonfinite"])
def test_every_rank_stops_on_horizon_and_nonfinite(tmp_path, mode):
    """A rank that exhausts its activation budget, or produces a non-finite
    state, raises the stop word on every board: every rank ends and raises
    the reference's exception (HorizonExhausted / ValueError,
    async_engine.py:362-365, linalg.py:74-75) instead of hanging."""
    world, p = 2, 8
    mp.spawn(_edge_worker, args=(world, _free_port(), p, 24, mode, str(tmp_path)), nprocs=world, join=True)
    got = [open(tmp_path / f"r{r}.txt").read() for r in range(world)]
    if mode == "horizon":
        assert all(g == "horizon max_events" for g in got), got
    else:
        assert all(g.startswith("value") and "finite" in g for g in got), got
