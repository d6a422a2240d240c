"""C2 fine batch (64 slices x 1000 BE steps) with 32 vs 16 points per thread:
CUDA-event time per F batch, resident slices per wave.

    python scripts/fine_layout_probe.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2110_10762_b200 as pb  # noqa: E402
from paper_2110_10762_b200.model import with_register_layout  # noqa: E402

N, P = 65536, 64
ivp = pb.heat1d_system(N, 1.0, 0.0, 0.0, 0.0, 1.0)
fine = pb.backward_euler_propagator(ivp, 1.0 / P, 1000)
x = torch.rand(P, N, dtype=torch.float64, device="cuda")
for ch in (32, 16):
    f = with_register_layout(fine, ch)
    y = torch.empty_like(x)
    for nb in (1, 16, 32, 64):
        f.apply_batch(x[:nb], out=y[:nb])
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            f.apply_batch(x[:nb], out=y[:nb])
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(json.dumps({"points_per_thread": ch, "slices": nb, "ms": ms, "GPt_s": nb * 1000 * N / ms / 1e6,
                          "wave_slices": f.info.batch_wave_slices, "cluster": f.info.batch_cluster}), flush=True)
