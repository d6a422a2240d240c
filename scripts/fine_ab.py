"""A/B timing of the C2 fine batch (64 slices x 1000 BE steps, N = 65,536)
under environment switches given as NAME=VALUE arguments (one line each)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2110_10762_b200 as pb  # noqa: E402
from paper_2110_10762_b200 import inputs  # noqa: E402

N, P, S = 65536, 64, 1000
u0 = torch.tensor(inputs.sine_u0_1d(N, 32, 0), device="cuda")
x = u0.repeat(P, 1)
ref = None
for spec in sys.argv[1:] or ["BASE=1"]:
    k, v = spec.split("=")
    os.environ[k] = v
    ivp = pb.heat1d_system(N, 1.0, 0.0, 0.0, 0.0, 1.0)
    fine = pb.backward_euler_propagator(ivp, 1.0 / P, S)
    y = torch.empty_like(x)
    fine.apply_batch(x, out=y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms = []
    for _ in range(5):
        e0.record()
        fine.apply_batch(x, out=y)
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    ref = y.clone() if ref is None else ref
    print(json.dumps({"env": spec, "ms": sorted(ms)[2], "GPt_s": P * S * N / sorted(ms)[2] / 1e6,
                      "bitwise_equal_first": bool(torch.equal(y, ref))}), flush=True)
    del fine
    os.environ.pop(k)
