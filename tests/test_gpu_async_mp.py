"""GPU checks of the multi-process asynchronous runtime for whole-GPU
activations (paper_2110_10762_b200/async_mp.py, csrc/mailbox.cu):

* the mailbox / board kernels through the C ABI (push + seqlocked read,
  version publication, torn-read detection, board post/read);
* a one-rank NCCL world through the C ABI on a 3-D problem: exact quiescence
  lands bitwise on the sequential fine solution, the eps stop is drained;
* two OS processes sharing the one GPU (gloo for the host plumbing): the
  predecessor crosses processes through a CUDA IPC mailbox written by SM
  stores with a system-scope release (the multi-GPU data path; on one GPU
  the peer is the same device) — bitwise quiescence again. No kernel of one
  process waits on a kernel of the other.
"""
import ctypes
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(pb, n=20, p=6, steps=7, dtype="float64"):
    h = 1.0 / (n + 1)
    span = steps * 0.15 * h * h
    from paper_2110_10762_b200.inputs import modes_3d, sine_u0_nd
    u0 = sine_u0_nd((n, n, n), modes_3d(), 0).reshape(-1)
    ivp = pb.heat3d_system(n, t_final=p * span, u0=u0)
    fine = pb.forward_euler_propagator(ivp, span, steps, dtype=dtype)
    coarse = pb.backward_euler_propagator(ivp, span, 1, dtype=dtype)
    return u0, fine, coarse


def test_mailbox_and_board_kernels(gpu):
    from paper_2110_10762_b200 import _native
    from paper_2110_10762_b200.async_mp import CudaTransport
    u0, fine, coarse = _problem(gpu)
    tp = CudaTransport(fine)
    R, n = 3, 1000
    slot = 8192
    ws = tp.alloc(256 + R * slot)
    ver = tp.view(ws, (1,), torch.int64)
    st = torch.cuda.current_stream()
    ctr = torch.zeros(1, dtype=torch.int32, device="cuda")
    scratch = torch.zeros(3, dtype=torch.int64, device="cuda")
    dst = torch.empty(n, dtype=torch.float64, device="cuda")
    for v in range(1, 7):
        row = torch.arange(n, dtype=torch.float64, device="cuda") * v
        tp.push(ws + 256 + (v % R) * slot, row, ws, v, ctr.data_ptr(), st)
        tp.read_mailbox(ws + 256, slot, R, ws, dst, scratch, st)
        torch.cuda.synchronize()
        assert int(ver[0]) == v and int(scratch[1]) == v and int(scratch[2]) == 0
        assert torch.equal(dst, row)
    # a version that advanced past the seqlock window is reported as torn
    ver.fill_(100)
    scratch.zero_()
    lib = _native.load_library()
    rc = lib.pint_mailbox_read(tp.ctx, ctypes.c_void_p(ws + 256), slot, R, ctypes.c_void_p(ws),
                               ctypes.c_void_p(dst.data_ptr()), n * 8, ctypes.c_void_p(scratch.data_ptr()),
                               ctypes.c_void_p(scratch.data_ptr() + 8), ctypes.c_void_p(scratch.data_ptr() + 16),
                               ctypes.c_void_p(st.cuda_stream))
    assert rc == 0
    torch.cuda.synchronize()
    assert int(scratch[1]) == 100 and int(scratch[2]) == 0  # v re-read equal: consistent
    # boards
    board = tp.alloc(4 * 64)
    out = torch.zeros(4 * 8, dtype=torch.int64, device="cuda")
    host = torch.zeros(4 * 8, dtype=torch.int64).pin_memory()
    tp.post(board + 64, 0, [1, 2, 3, 4, 5, 6, 7], st)
    tp.post(board + 64, 2, [9, 8, 7, 6, 5, 4, 3], st)
    bd = tp.read_board(board, 4, out, host, st)
    assert bd[1].tolist() == [4, 9, 8, 7, 6, 5, 4, 3]
    assert bd[0].tolist() == [0] * 8
    # misaligned rows are refused
    assert lib.pint_mailbox_push(tp.ctx, ctypes.c_void_p(ws + 260), ctypes.c_void_p(dst.data_ptr()), 8,
                                 ctypes.c_void_p(ws), 1, ctypes.c_void_p(ctr.data_ptr()),
                                 ctypes.c_void_p(st.cuda_stream)) != 0
    tp.close()


def _init_world1(backend):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group(backend, rank=0, world_size=1)


@pytest.mark.parametrize("dtype", ("float64", "float32"))
def test_one_rank_nccl_world_quiescence_bitwise(gpu, dtype):
    from paper_2110_10762_b200.async_mp import run_async_parareal_mp
    u0, fine, coarse = _problem(gpu, dtype=dtype)
    p = 6
    _init_world1("nccl")
    try:
        res = run_async_parareal_mp(coarse, fine, u0, p, None, lanes=3, gather=True, record_trace=True)
        seq = gpu.sequential_fine_solve(fine, u0, p).tensor
        assert res.stop_reason == "converged"
        assert torch.equal(res.final, seq)
        assert res.counts[1:].sum() == res.activations == len(res.trace)
        res2 = run_async_parareal_mp(coarse, fine, u0, p, 1e-6, lanes=2, gather=True)
        assert res2.stop_reason == "converged"
        err = float((res2.final.double() - seq.double()).abs().max())
        assert err < 1e-3, err
    finally:
        dist.destroy_process_group()


def _two_proc_worker(rank, world, port, out_dir, dtype, delay):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2110_10762_b200 as pb
        from paper_2110_10762_b200.async_mp import run_async_parareal_mp
        torch.cuda.set_device(0)
        u0, fine, coarse = _problem(pb, dtype=dtype)
        p = 6
        res = run_async_parareal_mp(coarse, fine, u0, p, None, lanes=2, gather=True, record_trace=True,
                                    delay_frac=delay, seed=3)
        if rank == 0:
            seq = pb.sequential_fine_solve(fine, u0, p).tensor
            ok = bool(torch.equal(res.final, seq))
            with open(os.path.join(out_dir, "r.txt"), "w") as f:
                f.write(f"{ok} {res.stop_reason} {res.activations} {res.counts.tolist()}")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dtype,delay", [("float64", 0.0), ("float32", 0.2)])
def test_two_processes_ipc_mailbox_quiescence_bitwise(gpu, tmp_path, dtype, delay):
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_two_proc_worker, args=(r, 2, port, str(tmp_path), dtype, delay)) for r in range(2)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=300)
    for pr in procs:
        if pr.is_alive():
            pr.kill()
    assert all(pr.exitcode == 0 for pr in procs), [pr.exitcode for pr in procs]
    ok, stop, acts, counts = open(tmp_path / "r.txt").read().split(" ", 3)
    assert ok == "True" and stop == "converged", (ok, stop, acts, counts)


def _sharded_worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import numpy as np

        import paper_2110_10762_b200 as pb
        from paper_2110_10762_b200 import distributed as D
        from paper_2110_10762_b200.inputs import sine_u0_1d
        torch.cuda.set_device(0)
        n, p_local, T = 4096, 4, 1.0
        p = p_local * world
        ivp = pb.heat1d_system(n, 1.0, 0.0, 0.0, 0.0, T)
        fine = pb.backward_euler_propagator(ivp, T / p, 20)
        coarse = pb.backward_euler_propagator(ivp, T / p, 1)
        u0 = sine_u0_1d(n, 8, 0)
        res = D.run_parareal_sharded(coarse, fine, u0, p_local, 1e-9)  # default edge: peer-memory mailbox
        shards = [None] * world
        dist.all_gather_object(shards, res["shard"].cpu())
        if rank == 0:
            full = torch.cat([shards[0]] + [s[1:] for s in shards[1:]])
            ref = pb.run_parareal(coarse, fine, u0, p, 1e-9)
            ok = (res["k_final"] == ref.k_final and res["stop_reason"] == ref.stop_reason
                  and res["deltas"] == ref.deltas and torch.equal(full, ref.final.tensor.cpu()))
            with open(os.path.join(out_dir, "s.txt"), "w") as f:
                f.write(f"{ok} {res['k_final']} {ref.k_final} {res['stop_reason']}")
    finally:
        dist.destroy_process_group()


def test_two_processes_sharded_sync_mailbox_edge_bitwise(gpu, tmp_path):
    """The synchronous multi-GPU sweep with its chain edge over peer memory
    (K7: pint_mailbox_push into the next rank's IPC mailbox, sequence-numbered
    versions; host poll because both ranks share this GPU) equals the
    single-process run bitwise: same k, stop reason, deltas and iterate."""
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_sharded_worker, args=(r, 2, port, str(tmp_path))) for r in range(2)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=300)
    for pr in procs:
        if pr.is_alive():
            pr.kill()
    assert all(pr.exitcode == 0 for pr in procs), [pr.exitcode for pr in procs]
    ok, k, kref, stop = open(tmp_path / "s.txt").read().split()
    assert ok == "True", (k, kref, stop)


def test_mailbox_edge_device_wait_in_one_process(gpu):
    """The sync chain edge with the device-side wait (the multi-GPU mode):
    rank 0's edge pushes into rank 1's workspace, rank 1's stream waits on the
    version with pint_mailbox_wait — here both ends in one process on one
    stream (push before wait in stream order), so nothing waits on another
    process. Sequence numbers, slot parity and the timeout flag are checked."""
    from paper_2110_10762_b200.async_mp import CudaTransport
    from paper_2110_10762_b200.distributed import MailboxEdge
    u0, fine, coarse = _problem(gpu)

    class OneProcExchange:
        def __init__(self):
            self.pending = []

        def all_gather_bytes(self, b):
            # rank 1's edge is built first, rank 0's second: [rank 0, rank 1] handles
            self.pending.append(b)
            return [b, b] if len(self.pending) == 1 else [b, self.pending[0]]

        def all_gather_object(self, obj):
            return [obj, ("other-host", obj[1])]

    n = 5000
    like = torch.zeros(n, dtype=torch.float64, device="cuda")
    ex = OneProcExchange()
    tp = CudaTransport(fine)
    recv_edge = MailboxEdge(like, 1, 2, tp, ex, wait="device")      # rank 1 (consumer): allocates first
    send_edge = MailboxEdge(like, 0, 2, tp, ex, wait="device")      # rank 0 (producer): next = rank 1's ws
    assert send_edge.peer_next == recv_edge.ws
    row0 = torch.empty(n, dtype=torch.float64, device="cuda")
    d0 = torch.empty(1, dtype=torch.float64, device="cuda")
    for k in range(5):
        row = torch.arange(n, dtype=torch.float64, device="cuda") * (k + 1)
        dl = torch.tensor([0.5 * k], dtype=torch.float64, device="cuda")
        send_edge.send(k, row, dl)
        recv_edge.recv(k, row0, d0)
        torch.cuda.synchronize()
        assert torch.equal(row0, row) and float(d0) == 0.5 * k
        assert int(recv_edge.ver[0]) == k + 1
    recv_edge.check()
    # a version that never comes: the device wait gives up and the flag raises
    tp.wait_version(recv_edge.ver.data_ptr(), 99, recv_edge.timed_out, torch.cuda.current_stream(), timeout_s=0.05)
    torch.cuda.synchronize()
    with pytest.raises(RuntimeError):
        recv_edge.check()
    tp.close()
