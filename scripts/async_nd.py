"""C4 (256^3 fp32, P = 64, S = 200 forward-Euler, G = 1 backward-Euler direct
solve) asynchronous Parareal on CUDA streams vs the synchronous iteration:
time to tolerance, kappa / k, activations, error against the sequential fine
solve. ``domains`` emulates the per-GPU slice blocks (mailbox push) on one GPU.

    python scripts/async_nd.py [eps]
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2110_10762_b200 as pb  # noqa: E402
from paper_2110_10762_b200 import inputs  # noqa: E402


def main():
    eps = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-5
    n, p, steps, cfl = int(os.environ.get("ND_N", 256)), int(os.environ.get("ND_P", 64)), 200, 0.15
    h = 1.0 / (n + 1)
    span = steps * cfl * h * h
    u0 = inputs.sine_u0((n, n, n), seed=0)
    ivp = pb.heat3d_system(n, t_final=p * span, u0=u0)
    fine = pb.forward_euler_propagator(ivp, span, steps, dtype="float32")
    coarse = pb.backward_euler_propagator(ivp, span, 1, dtype="float32")
    seq = pb.sequential_fine_solve(fine, u0, p).tensor
    torch.cuda.synchronize()
    pb.run_parareal(coarse, fine, u0, p, eps, k_max=1, record_iterates=False)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tr = pb.run_parareal(coarse, fine, u0, p, eps, record_iterates=False)
    torch.cuda.synchronize()
    ts = time.perf_counter() - t0
    err = float((tr.final.tensor - seq).abs().max())
    print(json.dumps({"mode": "sync", "seconds": ts, "k": tr.k_final, "stop": tr.stop_reason,
                      "max_abs_vs_seq_fine": err}), flush=True)
    for lanes, domains, delay in ((4, 1, 0.0), (8, 1, 0.0), (8, 8, 0.0), (8, 8, 0.2)):
        res = pb.run_async_parareal_device(coarse, fine, u0, p, eps, lanes=lanes, domains=domains,
                                           delay_frac=delay, seed=1)
        audit = pb.audit_device_trace(res.trace_records, p, res.per_component_counts)
        err = float((res.final.tensor - seq).abs().max()) if hasattr(res.final, "tensor") else \
            float(np.max(np.abs(res.final.data - seq.cpu().numpy())))
        print(json.dumps({"mode": "async-streams", "lanes": lanes, "domains": domains, "delay_frac": delay,
                          "seconds": res.wall_s, "kappa": res.kappa, "activations": res.activations,
                          "stop": res.stop_reason, "max_abs_vs_seq_fine": err, "audit_ok": audit["ok"],
                          "max_staleness": audit["max_staleness"], "peak_in_flight": audit["peak_in_flight"]}),
              flush=True)


if __name__ == "__main__":
    main()
