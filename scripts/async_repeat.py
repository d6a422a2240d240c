"""C2 device-async runtime repeated in one process: wall time, kappa and
activations per run (variance probe)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2110_10762_b200 as pb
from paper_2110_10762_b200 import inputs

N, P, S = 65536, 64, 1000
u0 = inputs.sine_u0_1d(N, 32, 0)
ivp = pb.heat1d_system(N, 1.0, 0.0, 0.0, 0.0, 1.0)
fine = pb.backward_euler_propagator(ivp, 1.0 / P, S)
coarse = pb.backward_euler_propagator(ivp, 1.0 / P, 1)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
for r in range(n):
    t0 = time.perf_counter()
    res = pb.run_async_parareal_device(coarse, fine, u0, P, 1e-10)
    torch.cuda.synchronize()
    print(json.dumps({"run": r, "wall_s": res.wall_s, "outer_s": time.perf_counter() - t0, "kappa": res.kappa,
                      "activations": res.activations, "stop": res.stop_reason}), flush=True)
