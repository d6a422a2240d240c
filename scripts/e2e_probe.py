"""e2e (host-buffer) sweep at C2 for several upload/download split settings.

    python scripts/e2e_probe.py
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2110_10762_b200 as pb  # noqa: E402
from paper_2110_10762_b200.inputs import sine_u0_1d  # noqa: E402
from paper_2110_10762_b200.parareal import SyncEngine  # noqa: E402

n, p = 65536, 64
ivp = pb.heat1d_system(n, 1.0, 0.0, 0.0, 0.0, 1.0)
fine = pb.backward_euler_propagator(ivp, 1 / p, 1000)
coarse = pb.backward_euler_propagator(ivp, 1 / p, 1)
eng = SyncEngine(coarse, fine, p)
eng.init(sine_u0_1d(n, 32, 0))
base_g = eng.gcache.clone()
host_in = eng.lam_a.cpu().pin_memory()
host_out = torch.empty_like(host_in).pin_memory()
t = torch.empty(1 << 22, dtype=torch.float64, device="cuda")
# raw copy bandwidth
for name, src, dst in (("h2d", host_in, eng.lam_b), ("d2h", eng.lam_b, host_out)):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 5
    print(json.dumps({"copy": name, "ms": dt * 1e3, "GB_s": host_in.numel() * 8 / dt / 1e9}), flush=True)
for graph in (False, True):
    for h2d_splits, d2h_splits in ((1, 1), (1, 4), (2, 4), (4, 4), (8, 8)):
        ms = []
        for it in range(8):
            eng.gcache.copy_(base_g)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            eng.sweep_host(1, host_in, host_out, d2h_splits=d2h_splits, h2d_splits=h2d_splits, graph=graph)
            torch.cuda.synchronize()
            if it >= 3:
                ms.append((time.perf_counter() - t0) * 1e3)
        print(json.dumps({"graph": graph, "h2d_splits": h2d_splits, "d2h_splits": d2h_splits,
                          "ms": sum(ms) / len(ms), "GPt_s": p * 1000 * n / (sum(ms) / len(ms) * 1e-3) / 1e9}),
              flush=True)
