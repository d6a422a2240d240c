"""F batch (C2 slice: N = 65,536, BE) per-step time vs live slices: 1 CTA/SM
(P = 18), 2 CTAs/SM (P = 37), two waves (P = 64). Separates per-slice
latency from FP64-pipe contention between co-resident clusters."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2110_10762_b200 as pb  # noqa: E402

steps = 1000
N = 65536
ivp = pb.heat1d_system(N, 1.0, 0.0, 0.0, 0.0, 1.0)
F = pb.backward_euler_propagator(ivp, 1.0 / 64, steps)
clk = 1.965e9
for P in (1, 2, 9, 18, 19, 27, 37, 38, 48, 64, 74):
    x = torch.randn(P, N, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    F.apply_batch(x, out=y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        F.apply_batch(x, out=y)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"P={P:3d} CTAs={P * F.info.batch_cluster:4d} {ms:7.3f} ms  {P * N * steps / ms / 1e6:7.1f} GPt/s  "
          f"cycles/step={ms * 1e-3 / steps * clk:7.0f}", flush=True)
