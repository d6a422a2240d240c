"""Per-activation durations of the device async runtime at C2 (from the
device trace: t_start = before F, t_publish = after the correction)."""
import json
import sys

import numpy as np

import paper_2110_10762_b200 as pb
from paper_2110_10762_b200.async_parareal import TRACE_FIELDS
from paper_2110_10762_b200.inputs import sine_u0_1d

n, p = 65536, 64
domains = int(sys.argv[1]) if len(sys.argv) > 1 else 8
ivp = pb.heat1d_system(n, 1.0, 0.0, 0.0, 0.0, 1.0)
fine = pb.backward_euler_propagator(ivp, 1 / p, 1000)
coarse = pb.backward_euler_propagator(ivp, 1 / p, 1)
u0 = sine_u0_1d(n, 32, 0)
pb.run_async_parareal_device(coarse, fine, u0, p, 1e-10, domains=domains)  # warm
res = pb.run_async_parareal_device(coarse, fine, u0, p, 1e-10, domains=domains, record_trace=True)
rec = res.trace_records
i0, i1 = TRACE_FIELDS.index("t_start_ns"), TRACE_FIELDS.index("t_publish_ns")
dur = (rec[:, i1] - rec[:, i0]) / 1e6
t0 = rec[:, i0].min()
span = (rec[:, i1].max() - t0) / 1e6
# in-flight count sampled on a 0.1 ms grid
grid = np.arange(0, span, 0.1)
st, en = (rec[:, i0] - t0) / 1e6, (rec[:, i1] - t0) / 1e6
infl = [(np.sum((st <= g) & (en > g))) for g in grid]
print(json.dumps({"domains": domains, "wall_s": res.wall_s,
                  "kappa": int(res.kappa), "activations": int(len(rec)), "span_ms": span,
                  "dur_ms_median": float(np.median(dur)), "dur_ms_p10": float(np.percentile(dur, 10)),
                  "dur_ms_p90": float(np.percentile(dur, 90)), "inflight_mean": float(np.mean(infl)),
                  "inflight_max": int(np.max(infl)), "clusters": res.concurrent_clusters}))
