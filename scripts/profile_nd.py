"""One explicit fine application at a C3/C4 shape (for ncu captures of the
wavefront stencil kernels).

    python scripts/profile_nd.py [c3_f64|c3_f32|c4_f32] [slices] [steps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2110_10762_b200 as pb  # noqa: E402

CFG = {"c3_f64": ((1024, 1024), 0.2, "float64"), "c3_f32": ((1024, 1024), 0.2, "float32"),
       "c4_f32": ((256, 256, 256), 0.15, "float32")}

if __name__ == "__main__":
    name = sys.argv[1] if len(sys.argv) > 1 else "c4_f32"
    p = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 8
    shape, cfl, dtype = CFG[name]
    n = shape[0]
    h = 1.0 / (n + 1)
    ivp = (pb.heat2d_system if len(shape) == 2 else pb.heat3d_system)(n, t_final=1.0)
    F = pb.forward_euler_propagator(ivp, steps * cfl * h * h, steps, dtype=dtype)
    x = torch.randn(p, ivp.dim, dtype=F.dtype, device="cuda")
    y = torch.empty_like(x)
    F.apply_batch(x, out=y)
    torch.cuda.synchronize()
    print("ok")
