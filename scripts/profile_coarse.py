"""Apply the n-D direct coarse solve a few times at the C3/C4 shapes (for an
ncu launch list / full capture of its kernels).

    python scripts/profile_coarse.py [c3_f64|c3_f32|c4_f32] [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2110_10762_b200 as pb  # noqa: E402

CFG = {"c3_f64": ((1024, 1024), 100, "float64"), "c3_f32": ((1024, 1024), 100, "float32"),
       "c4_f32": ((256, 256, 256), 30, "float32")}

if __name__ == "__main__":
    name = sys.argv[1] if len(sys.argv) > 1 else "c3_f64"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    shape, cfl_coarse, dtype = CFG[name]
    n = shape[0]
    h = 1.0 / (n + 1)
    ivp = (pb.heat2d_system if len(shape) == 2 else pb.heat3d_system)(n, t_final=1.0)
    G = pb.backward_euler_propagator(ivp, cfl_coarse * h * h, 1, dtype=dtype)
    x = torch.randn(1, ivp.dim, dtype=G.dtype, device="cuda")
    y = torch.empty_like(x)
    for _ in range(reps):
        G.apply_batch(x, out=y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        G.apply_batch(x, out=y)
    e1.record()
    torch.cuda.synchronize()
    print(f"{name}: {e0.elapsed_time(e1) / reps:.3f} ms per solve")
