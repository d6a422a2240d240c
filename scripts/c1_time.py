"""BASELINE configs[0] (C1: N = 1024, P = 16, F = 100 BE steps, G = 1 BE step,
fp64, eps = 1e-10) — the reference's own CPU-runnable case — on the GPU:
sync time to tolerance (warm), k, error against the long-double truth, and
the device async runtime.

    python scripts/c1_time.py
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2110_10762_b200 as pb  # noqa: E402
from paper_2110_10762_b200.inputs import sine_u0_1d  # noqa: E402

n, p = 1024, 16
u0 = sine_u0_1d(n, 8, 0)
ivp = pb.heat1d_system(n, 1.0, 0.0, 0.0, 0.0, 1.0)
fine = pb.backward_euler_propagator(ivp, 1 / p, 100)
coarse = pb.backward_euler_propagator(ivp, 1 / p, 1)
pb.run_parareal(coarse, fine, u0, p, 1e-10, record_iterates=False)
times = []
for _ in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tr = pb.run_parareal(coarse, fine, u0, p, 1e-10, record_iterates=False)
    torch.cuda.synchronize()
    times.append(time.perf_counter() - t0)
seq = pb.sequential_fine_solve(fine, u0, p).data
err = float(np.max(np.abs(tr.final.data - seq)))
res = pb.run_async_parareal_device(coarse, fine, u0, p, 1e-10)
print(json.dumps({"config": "C1", "n": n, "slices": p, "sync_seconds_median": float(np.median(times)),
                  "k": tr.k_final, "stop": tr.stop_reason, "max_abs_vs_seq_fine": err,
                  "async_device_seconds": res.wall_s, "async_kappa": res.kappa,
                  "reference_cpu_seconds_survey_probe": 1.17}), flush=True)
