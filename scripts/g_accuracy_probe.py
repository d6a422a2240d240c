"""Accuracy of one direct implicit coarse solve (2-D/3-D, fp32/fp64) against
the exact DST-I solve of the oracle, per variant (modal sweep chunked or not,
tensor-core transforms or SIMT). Diagnostic for the fp32 coarse chain."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2110_10762_b200 as pb  # noqa: E402
from oracle import heat_oracle as H  # noqa: E402
from oracle.nd_truth import SpectralND  # noqa: E402

for ndim, n, steps, cfl in ((2, 1024, 500, 0.2), (3, 256, 200, 0.15)):
    h = 1.0 / (n + 1)
    span = steps * cfl * h * h
    shape = (n,) * ndim
    u0 = H.sine_u0_nd(shape, H.modes_2d() if ndim == 2 else H.modes_3d(), 0).reshape(-1)
    mk = pb.heat2d_system if ndim == 2 else pb.heat3d_system
    ivp = mk(n, t_final=32 * span, u0=u0)
    G = SpectralND(shape, h, span)
    want = G.apply(u0)
    rows = [u0]
    for _ in range(4):
        rows.append(G.apply(rows[-1]))
    for dtype in ("float32", "float64"):
        for env in ({}, {"PINT_MODAL_CHUNKED": "0"}, {"PINT_TC_XFORM": "0"}):
            for k, v in env.items():
                os.environ[k] = v
            g = pb.backward_euler_propagator(ivp, span, 1, dtype=dtype)
            x = torch.tensor(u0, device="cuda", dtype=g.dtype)
            got = g.apply(x).double().cpu().numpy()
            chain = [x]
            for _ in range(4):
                chain.append(g.apply(chain[-1]))
            ch = [float(np.linalg.norm(c.double().cpu().numpy() - r) / np.linalg.norm(r)) for c, r in zip(chain, rows)]
            print(json.dumps({"ndim": ndim, "dtype": dtype, "env": env,
                              "one_solve_rel_l2": float(np.linalg.norm(got - want) / np.linalg.norm(want)),
                              "chain_rel_l2": ch}), flush=True)
            for k in env:
                os.environ.pop(k)
