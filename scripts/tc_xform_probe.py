"""Direct n-D coarse solve with the sine transforms on the tensor cores
(3xTF32, tc_xform.cu) vs the SIMT GEMMs: accuracy (against the fp64 solve of
the same system and as a normwise backward error) and time per solve.

    python scripts/tc_xform_probe.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2110_10762_b200 as pb  # noqa: E402
from paper_2110_10762_b200 import inputs  # noqa: E402

for shape in ((256, 256, 256), (512, 512, 512), (1024, 1024), (64, 64, 64), (128, 128)):
    n = shape[0]
    h = 1.0 / (n + 1)
    steps = 200 if len(shape) == 3 else 500
    cfl = 0.15 if len(shape) == 3 else 0.2
    span = steps * cfl * h * h
    mk = pb.heat3d_system if len(shape) == 3 else pb.heat2d_system
    u0 = inputs.sine_u0(shape, seed=0)
    ivp = mk(n, t_final=span, u0=u0)
    b = torch.tensor(u0, dtype=torch.float64, device="cuda").reshape(1, -1)
    b += 1e-3 * torch.rand_like(b)
    g64 = pb.backward_euler_propagator(ivp, span, 1, dtype="float64")
    x64 = g64.apply_batch(b)
    out = {"shape": list(shape)}
    for tc in ("0", "1"):
        os.environ["PINT_TC_XFORM"] = tc
        g32 = pb.backward_euler_propagator(ivp, span, 1, dtype="float32")
        b32 = b.float()
        y = torch.empty_like(b32)
        g32.apply_batch(b32, out=y)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            g32.apply_batch(b32, out=y)
        e1.record()
        torch.cuda.synchronize()
        err = float((y.double() - x64).abs().max() / x64.abs().max())
        # backward error of the fp32 answer in the fp64 operator: ||(I - dT L) y - b|| / (||A|| ||y|| + ||b||)
        tag = "tc" if tc == "1" else "simt"
        out[f"{tag}_ms"] = e0.elapsed_time(e1) / 5
        out[f"{tag}_rel_err_vs_fp64"] = err
    print(json.dumps(out), flush=True)
