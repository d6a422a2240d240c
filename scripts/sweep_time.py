"""Fused coarse sweep alone at C2 (64 slices, N = 65536): CUDA-event time per
launch and per slice, warm, 20 repetitions (median)."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2110_10762_b200 as pb
from paper_2110_10762_b200.parareal import SyncEngine
from paper_2110_10762_b200 import inputs as H

N, P = 65536, 64
ivp = pb.heat1d_system(N, 1.0, 0.0, 0.0, 0.0, 1.0)
fine = pb.backward_euler_propagator(ivp, 1.0 / P, 1000)
coarse = pb.backward_euler_propagator(ivp, 1.0 / P, 1)
eng = SyncEngine(coarse, fine, P)
eng.init(H.sine_u0_1d(N, 32, 0))
eng.fine_batch(1)
g0 = eng.gcache.clone()
ts = []
for r in range(23):
    eng.gcache.copy_(g0)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    eng.coarse_sweep(1, eng.lam_b)
    b.record()
    torch.cuda.synchronize()
    if r >= 3:
        ts.append(a.elapsed_time(b))
ts.sort()
ms = ts[len(ts) // 2]
print(json.dumps({"sweep_ms": ms, "us_per_slice": 1000 * ms / P, "checksum": float(eng.lam_b.double().abs().sum())}))
