"""Run the C2 hot-path kernels once each (for ncu): F batch over 64 slices
(1000 BE steps, N=65536) and the fused coarse sweep. Usage:
  python scripts/profile_c2.py [fine|sweep|both] [--steps S]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2110_10762_b200 as pb
from paper_2110_10762_b200.parareal import SyncEngine
from paper_2110_10762_b200 import inputs as H  # seeded synthetic inputs

what = sys.argv[1] if len(sys.argv) > 1 else "both"
steps = int(sys.argv[sys.argv.index("--steps") + 1]) if "--steps" in sys.argv else 1000
N, P = 65536, 64
ivp = pb.heat1d_system(N, 1.0, 0.0, 0.0, 0.0, 1.0)
fine = pb.backward_euler_propagator(ivp, 1.0 / P, steps)
coarse = pb.backward_euler_propagator(ivp, 1.0 / P, 1)
eng = SyncEngine(coarse, fine, P)
eng.init(H.sine_u0_1d(N, 32, 0))
torch.cuda.synchronize()
if what in ("fine", "both"):
    eng.fine_batch(1)
if what in ("sweep", "both"):
    eng.coarse_sweep(1, eng.lam_b)
    eng.reduce_delta(1)
torch.cuda.synchronize()
print("ok", eng.read_delta())
