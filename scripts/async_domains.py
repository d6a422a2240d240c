"""C2 device async runtime with the slices split into 1/2/4/8 domains hosted by
one launch (the multi-GPU protocol on one GPU): time to tolerance, kappa,
activations, seqlock retries and the error against the sequential fine solve.

    python scripts/async_domains.py [eps]
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_10762_b200 as pb  # noqa: E402
from paper_2110_10762_b200 import inputs as H  # noqa: E402  (seeded synthetic inputs)


def main():
    eps = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-10
    n, p = 65536, 64
    u0 = H.sine_u0_1d(n, 32, 0)
    ivp = pb.heat1d_system(n, 1.0, 0.0, 0.0, 0.0, 1.0)
    fine = pb.backward_euler_propagator(ivp, 1 / p, 1000)
    coarse = pb.backward_euler_propagator(ivp, 1 / p, 1)
    seq = pb.sequential_fine_solve(fine, u0, p).data
    claims = [int(c) for c in os.environ.get("CLAIMS", "0").split(",")]
    doms = [int(c) for c in os.environ.get("DOMAINS", "1,2,4,8").split(",")]
    for claim in claims:
      os.environ["PINT_ASYNC_CLAIM"] = str(claim)
      for domains in doms:
        for mode in ("eps", "quiescence"):
            e = eps if mode == "eps" else None
            pb.run_async_parareal_device(coarse, fine, u0, p, e, domains=domains)  # warm
            res = pb.run_async_parareal_device(coarse, fine, u0, p, e, domains=domains, record_trace=True)
            audit = pb.audit_device_trace(res.trace_records, p, res.per_component_counts)
            err = float(np.max(np.abs(res.final.data - seq)))
            print(json.dumps({"claim": claim, "domains": domains, "mode": mode, "epsilon": e, "seconds": res.wall_s,
                              "kappa": res.kappa, "activations": res.activations, "retries": res.retries,
                              "clusters": res.concurrent_clusters, "max_abs_vs_seq_fine": err,
                              "audit_ok": audit["ok"], "max_staleness": audit["max_staleness"],
                              "peak_in_flight": audit["peak_in_flight"]}), flush=True)


if __name__ == "__main__":
    main()
