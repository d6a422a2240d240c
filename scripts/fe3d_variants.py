"""Time the 3-D explicit stencil tilings (stencil3d.cu variants; 0 = the
first-generation fe3d_wave) at the C4 shape and check they are bitwise equal.

    python scripts/fe3d_variants.py [dtype] [slices] [steps]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2110_10762_b200 as pb  # noqa: E402

if __name__ == "__main__":
    dtype = sys.argv[1] if len(sys.argv) > 1 else "float32"
    p = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 24
    n = int(os.environ.get("FE3D_N", 256))
    variants = [0, 3, 6, 8, 9, 12, 13, 14] if dtype == "float32" else [0, 4, 5, 7, 8]
    if os.environ.get("FE3D_VARIANTS"):
        variants = [int(v) for v in os.environ["FE3D_VARIANTS"].split(",")]
    h = 1.0 / (n + 1)
    ivp = pb.heat3d_system(n, t_final=1.0)
    g = torch.Generator(device="cuda").manual_seed(0)
    ref = None
    for v in variants:
        os.environ["PINT_FE3D_VARIANT"] = str(v)
        F = pb.forward_euler_propagator(ivp, steps * 0.15 * h * h, steps, dtype=dtype)
        x = torch.rand(p, ivp.dim, dtype=F.dtype, device="cuda", generator=g) if ref is None else x
        y = torch.empty_like(x)
        for _ in range(2):
            F.apply_batch(x, out=y)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 5
        e0.record()
        for _ in range(reps):
            F.apply_batch(x, out=y)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        upd = p * steps * n ** 3
        if ref is None:
            ref = y.clone()
        same = bool(torch.equal(y, ref))
        maxdiff = float((y - ref).abs().max())
        esz = 4 if dtype == "float32" else 8
        print(json.dumps({"variant": v, "dtype": dtype, "n": n, "slices": p, "steps": steps, "ms": ms,
                          "GPt_s": upd / ms / 1e6, "alg_hbm_frac": upd / ms / 1e6 * 2 * esz / 6442.2,
                          "bitwise_equal_v0": same, "max_abs_diff": maxdiff}), flush=True)
