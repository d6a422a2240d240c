"""CPU test doubles for the multi-process asynchronous runtime
(paper_2110_10762_b200/async_mp.py): a shared-memory transport standing in
for CUDA IPC + the mailbox/board kernels, and elementwise CPU propagators
standing in for the GPU operators. The runtime's host protocol (scheduling,
mailbox versions, seqlocks, status boards, termination) runs unchanged on
top of them in real OS processes (gloo), so the protocol is exercised with
real concurrency here; the device versions are checked on the GPU."""
from __future__ import annotations

import contextlib
import uuid
from multiprocessing import shared_memory

import numpy as np
import torch

_BASE = 1 << 40  # "pointer" = region id * 2^40 + byte offset


class _Stream:
    def synchronize(self):
        pass

    def wait_event(self, ev):
        pass


class _Event:
    def query(self):
        return True

    def synchronize(self):
        pass


class ShmTransport:
    def __init__(self):
        self._regions = {}   # id -> SharedMemory
        self._names = {}     # id -> name
        self._owned = []
        self._next = 1

    def _reg(self, shm) -> int:
        rid = self._next
        self._next += 1
        self._regions[rid] = shm
        return rid * _BASE

    def _buf(self, ptr: int):
        rid, off = divmod(ptr, _BASE)
        return self._regions[rid].buf, off

    def alloc(self, nbytes: int) -> int:
        shm = shared_memory.SharedMemory(create=True, size=int(nbytes), name="pint_" + uuid.uuid4().hex[:20])
        shm.buf[:nbytes] = bytes(nbytes)
        self._owned.append(shm)
        return self._reg(shm)

    def view(self, ptr: int, shape, dtype) -> torch.Tensor:
        buf, off = self._buf(ptr)
        count = int(np.prod(shape))
        return torch.frombuffer(buf, dtype=dtype, count=count, offset=off).view(*shape)

    def export(self, ptr: int) -> bytes:
        rid, _ = divmod(ptr, _BASE)
        return self._regions[rid].name.encode()

    def open(self, handle: bytes, own_ptr: int, own_handle: bytes) -> int:
        if handle == own_handle:
            return own_ptr
        return self._reg(shared_memory.SharedMemory(name=handle.decode()))

    def close(self):
        for rid, shm in list(self._regions.items()):
            try:
                shm.close()
            except BufferError:
                pass
        for shm in self._owned:
            try:
                shm.unlink()
            except FileNotFoundError:
                pass
        self._regions = {}

    def _i64(self, ptr: int, count: int) -> np.ndarray:
        buf, off = self._buf(ptr)
        return np.frombuffer(buf, dtype=np.int64, count=count, offset=off)

    # streams: the CPU executes each call as it is issued
    def stream(self):
        return _Stream()

    def event(self, stream):
        return _Event()

    def stream_ctx(self, stream):
        return contextlib.nullcontext()

    def sleep_cycles(self, cycles, stream):
        pass

    def synchronize(self):
        pass

    # mailbox / boards
    def push(self, dst_ptr, src: torch.Tensor, ver_ptr, version, ctr_ptr, stream):
        buf, off = self._buf(dst_ptr)
        raw = src.contiguous().view(torch.uint8).numpy().tobytes()
        buf[off:off + len(raw)] = raw
        self._i64(ver_ptr, 1)[0] = version  # after the data (x86: stores are not reordered)

    def read_mailbox(self, ring_ptr, slot_bytes, nslots, ver_ptr, dst: torch.Tensor, scratch, stream):
        ver = self._i64(ver_ptr, 1)
        v = int(ver[0])
        buf, off = self._buf(ring_ptr + (v % nslots) * slot_bytes)
        nbytes = dst.numel() * dst.element_size()
        data = bytes(buf[off:off + nbytes])
        v2 = int(ver[0])
        dst.view(torch.uint8).copy_(torch.frombuffer(bytearray(data), dtype=torch.uint8))
        scratch[1] = v
        scratch[2] = 1 if v2 > v + nslots - 2 else 0

    def post(self, slot_ptr, seq, words, stream):
        s = self._i64(slot_ptr, 8)
        s[0] = seq + 1
        s[1:] = np.asarray(words, dtype=np.int64)
        s[0] = seq + 2

    def read_board(self, board_ptr, nslots, out, host, stream):
        b = self._i64(board_ptr, 8 * nslots)
        res = np.zeros((nslots, 8), dtype=np.int64)
        for q in range(nslots):
            for _ in range(1_000_000):
                a = int(b[8 * q])
                w = b[8 * q + 1:8 * q + 8].copy()
                c = int(b[8 * q])
                if a == c and a % 2 == 0:
                    res[q, 0] = a
                    res[q, 1:] = w
                    break
            else:
                res[q, 0] = -1
        return res

    def read_word(self, t: torch.Tensor, host, stream) -> int:
        return int(t[0])


class CpuOps:
    """F = S explicit heat steps (r_f), G = one explicit step (r_g), both
    elementwise torch ops (deterministic across processes); the correction
    in the reference's order (G(f) + F(o)) - G(o)."""

    device_str = "cpu"

    def __init__(self, n: int, steps: int = 12, r_f: float = 0.2, r_g: float = 0.45):
        self.n, self.steps, self.r_f, self.r_g = n, steps, r_f, r_g

    def lane_ops(self, index):
        return ("G", self.r_g, 1), ("F", self.r_f, self.steps)

    @staticmethod
    def step(x: torch.Tensor, r: float) -> torch.Tensor:
        left = torch.nn.functional.pad(x[:-1], (1, 0))
        right = torch.nn.functional.pad(x[1:], (0, 1))
        return x + r * ((left + right) - 2.0 * x)

    def run(self, prop, x: torch.Tensor) -> torch.Tensor:
        _, r, steps = prop
        for _ in range(steps):
            x = self.step(x, r)
        return x

    def apply(self, prop, src, dst, stream):
        dst.copy_(self.run(prop, src.clone()))

    def equal(self, a, b, eq, stream):
        eq.fill_(1 if torch.equal(a, b) else 0)

    def correct(self, g, f, gold, cur, dst, eq, delta, flag, stream):
        out = f.clone() if int(eq[0]) else (g + f) - gold
        delta[0] = float((out - cur).abs().max())
        if not bool(torch.isfinite(out).all()):
            flag[0] = 1
        dst.copy_(out)

    # the reference quantities the test compares against
    def fine_seq(self, u0: torch.Tensor, p: int) -> torch.Tensor:
        rows = [u0.clone()]
        for _ in range(p):
            rows.append(self.run(("F", self.r_f, self.steps), rows[-1].clone()))
        return torch.stack(rows)

    def coarse_init_rows(self, coarse, u0, first: int, last: int) -> torch.Tensor:
        x = torch.as_tensor(np.asarray(u0, dtype=np.float64)).clone()
        rows = []
        for i in range(0, last + 1):
            if i >= first:
                rows.append(x.clone())
            x = self.run(("G", self.r_g, 1), x)
        return torch.stack(rows)


class FakeProp:
    """Just the attributes the runtime reads from a propagator."""

    def __init__(self, n: int):
        self.dim = n
        self.dtype = torch.float64
        self.device = "cpu"
