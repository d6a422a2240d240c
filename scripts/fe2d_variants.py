"""Time the 2-D explicit stencil variants (PINT_FE2D_VARIANT) at the C3 shape
and check they are bitwise equal.

    python scripts/fe2d_variants.py [dtype] [slices] [steps]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2110_10762_b200 as pb  # noqa: E402

if __name__ == "__main__":
    dtype = sys.argv[1] if len(sys.argv) > 1 else "float64"
    p = int(sys.argv[2]) if len(sys.argv) > 2 else 32
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 48
    n = int(os.environ.get("FE2D_N", 1024))
    h = 1.0 / (n + 1)
    ivp = pb.heat2d_system(n, t_final=1.0)
    x = None
    ref = None
    for v in [int(t) for t in os.environ.get("FE2D_VARIANTS", "0,1,2").split(",")]:
        os.environ["PINT_FE2D_VARIANT"] = str(v)
        F = pb.forward_euler_propagator(ivp, steps * 0.2 * h * h, steps, dtype=dtype)
        if x is None and os.environ.get("FE2D_SINE"):
            from paper_2110_10762_b200 import inputs
            x = torch.tensor(inputs.sine_u0((n, n), seed=0), dtype=F.dtype, device="cuda").repeat(p, 1)
        if x is None:
            x = torch.rand(p, ivp.dim, dtype=F.dtype, device="cuda", generator=torch.Generator("cuda").manual_seed(0))
        y = torch.empty_like(x)
        for _ in range(2):
            F.apply_batch(x, out=y)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            F.apply_batch(x, out=y)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        if ref is None:
            ref = y.clone()
        upd = p * steps * n * n
        print(json.dumps({"variant": v, "dtype": dtype, "n": n, "slices": p, "steps": steps, "ms": ms,
                          "GPt_s": upd / ms / 1e6, "bitwise_equal_v0": bool(torch.equal(y, ref))}), flush=True)
