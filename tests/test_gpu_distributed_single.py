"""The multi-GPU drivers on a world of one GPU (NCCL backend): the sharded
synchronous iteration and the asynchronous domain runtime run their real
device plumbing (NCCL reductions on device tensors, the domain workspace
exported as a CUDA IPC handle, all-gathered, connected, reset, launched and
collected through the C ABI). World sizes > 1 are covered on CPU by
tests/test_distributed_gloo.py (one GPU is available here)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture
def nccl_world():
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()), RANK="0", WORLD_SIZE="1", LOCAL_RANK="0")
    from paper_2110_10762_b200 import distributed as D
    D.init_process_group()
    assert dist.get_backend() == "nccl"
    yield D
    D.destroy()


def test_sharded_sync_equals_single_process(gpu, nccl_world):
    D = nccl_world
    from paper_2110_10762_b200.inputs import sine_u0_1d
    n, p = 1024, 16
    u0 = sine_u0_1d(n, 8, 0)
    ivp = gpu.heat1d_system(n, 1.0, 0.0, 0.0, 0.0, 1.0)
    fine = gpu.backward_euler_propagator(ivp, 1 / p, 100)
    coarse = gpu.backward_euler_propagator(ivp, 1 / p, 1)
    res = D.run_parareal_sharded(coarse, fine, u0, p, 1e-10)
    ref = gpu.run_parareal(coarse, fine, u0, p, 1e-10)
    assert res["k_final"] == ref.k_final == 14 and res["stop_reason"] == ref.stop_reason
    assert res["deltas"] == ref.deltas
    assert np.array_equal(res["shard"].cpu().numpy(), ref.final.data)


def test_async_domain_runtime_through_the_c_abi(gpu, nccl_world):
    D = nccl_world
    from paper_2110_10762_b200.inputs import sine_u0_1d
    n, p = 1024, 16
    u0 = sine_u0_1d(n, 8, 0)
    ivp = gpu.heat1d_system(n, 1.0, 0.0, 0.0, 0.0, 1.0)
    fine = gpu.backward_euler_propagator(ivp, 1 / p, 100)
    coarse = gpu.backward_euler_propagator(ivp, 1 / p, 1)
    seq = gpu.sequential_fine_solve(fine, u0, p).data
    out = D.run_async_parareal_distributed(coarse, fine, u0, p, None, record_trace=True, trace_cap=100_000)
    assert out["stop_reason"] == "converged"
    assert np.array_equal(out["final"].cpu().numpy(), seq)
    assert out["slices"] == (1, p)
    audit = gpu.audit_device_trace(out["trace"], p, out["counts"])
    assert audit["ok"], audit
    eps = D.run_async_parareal_distributed(coarse, fine, u0, p, 1e-10)
    assert eps["stop_reason"] == "converged"
    assert np.max(np.abs(eps["final"].cpu().numpy() - seq)) < 1e-8
