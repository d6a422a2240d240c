"""BASELINE C5 (512^3 fp32, P = 128, S = 100 forward-Euler, G = 1 backward-
Euler direct solve, eps = 1e-6) synchronous Parareal on ONE B200 with the
in-place engine (2 state copies = 132 GB; the standard 4-copy engine would
need 264 GB). Time to tolerance, k, peak HBM, and the error against the
sequential fine solve computed slice by slice (streamed, one state).

    python scripts/c5_lean.py [eps]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2110_10762_b200 as pb  # noqa: E402
from paper_2110_10762_b200 import inputs  # noqa: E402


def main():
    eps = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-6
    n, p, steps, cfl = int(os.environ.get("C5_N", 512)), int(os.environ.get("C5_P", 128)), 100, 0.15
    h = 1.0 / (n + 1)
    span = steps * cfl * h * h
    u0 = inputs.sine_u0((n, n, n), seed=0)
    ivp = pb.heat3d_system(n, t_final=p * span, u0=u0)
    fine = pb.forward_euler_propagator(ivp, span, steps, dtype="float32")
    coarse = pb.backward_euler_propagator(ivp, span, 1, dtype="float32")
    torch.cuda.reset_peak_memory_stats()
    torch.cuda.synchronize()
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from bench import ClockSampler
    with ClockSampler(torch.cuda.current_device()) as clk:
        t0 = time.perf_counter()
        tr = pb.run_parareal(coarse, fine, u0, p, eps, record_iterates=False)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    peak = torch.cuda.max_memory_allocated() / 2**30
    final = tr.final.tensor
    x = torch.tensor(u0, dtype=torch.float32, device="cuda").reshape(1, -1)
    y = torch.empty_like(x)
    err = 0.0
    for i in range(1, p + 1):
        fine.apply_batch(x, out=y)
        x, y = y, x
        err = max(err, float((final[i] - x[0]).abs().max()))
    print(json.dumps({"config": "C5", "shape": [n, n, n], "slices": p, "fine_steps": steps, "dtype": "float32",
                      "epsilon": eps, "seconds": wall, "k": tr.k_final, "stop": tr.stop_reason,
                      "deltas": tr.deltas, "peak_hbm_gib": peak, "max_abs_vs_seq_fine": err,
                      "engine": "lean (in place, 2 state copies)", "clocks": clk.summary()}), flush=True)


if __name__ == "__main__":
    main()
