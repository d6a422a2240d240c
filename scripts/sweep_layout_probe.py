"""Fused coarse sweep (tri1d_sweep_kernel) at C2 with the coarse operator in
the 32- and 16-points-per-thread layouts (16: twice the threads, 8 warps per
SM in the 16-CTA cluster). CUDA-event time per launch over 64 slices.

    python scripts/sweep_layout_probe.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2110_10762_b200 as pb  # noqa: E402
from paper_2110_10762_b200.inputs import sine_u0_1d  # noqa: E402
from paper_2110_10762_b200.model import with_register_layout  # noqa: E402
from paper_2110_10762_b200.parareal import SyncEngine  # noqa: E402

N, P = 65536, 64
ivp = pb.heat1d_system(N, 1.0, 0.0, 0.0, 0.0, 1.0)
fine = pb.backward_euler_propagator(ivp, 1.0 / P, 1000)
coarse = pb.backward_euler_propagator(ivp, 1.0 / P, 1)
out = {}
for ch in (32, 16):
    g = with_register_layout(coarse, ch)
    eng = SyncEngine(g, fine, P)
    eng.init(sine_u0_1d(N, 32, 0))
    eng.fine_batch(1)
    torch.cuda.synchronize()
    for _ in range(2):
        eng.coarse_sweep(1, eng.lam_b)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        eng.coarse_sweep(1, eng.lam_b)
    e1.record()
    torch.cuda.synchronize()
    out[ch] = eng.lam_b.clone()
    print(json.dumps({"points_per_thread": ch, "sweep_ms": e0.elapsed_time(e1) / 5,
                      "us_per_slice": e0.elapsed_time(e1) / 5 / P * 1e3, "threads": g.info.threads_per_slice,
                      "sweep_cluster": g.info.sweep_cluster}), flush=True)
d = (out[32] - out[16]).abs().max().item()
print(json.dumps({"max_abs_diff_layouts": d, "max_abs": out[32].abs().max().item()}))
