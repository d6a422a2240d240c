"""Per-phase clock64 timing of one fine step (debug library built with
-DPINT_PHASE_TIMING): PINT_LIB_PATH=scripts/libpint_timing.so python scripts/phase_timing.py"""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2110_10762_b200 as pb
from paper_2110_10762_b200 import _native

N, P, S = int(os.environ.get("N", 65536)), int(os.environ.get("P", 64)), 1000
ivp = pb.heat1d_system(N, 1.0, 0.0, 0.0, 0.0, 1.0)
F = pb.backward_euler_propagator(ivp, 1.0 / 64, S)
lib = _native.load_library()
lib.pint_debug_phase_timing.argtypes = [ctypes.c_void_p, ctypes.c_int]
info = F.info
ncta = P * info.batch_cluster
nwarps = ncta * (info.threads_per_slice // info.batch_cluster // 32)
buf = torch.zeros(nwarps * 8, dtype=torch.int64, device="cuda")
lib.pint_debug_phase_timing(ctypes.c_void_p(buf.data_ptr()), 500)
x = torch.randn(P, N, dtype=torch.float64, device="cuda")
F.apply_batch(x); torch.cuda.synchronize()
b = buf.cpu().numpy().reshape(nwarps, 8)[:, :7].astype(np.int64)
ok = b[:, 0] > 0
b = b[ok]
d = np.diff(b, axis=1)
names = ["forward+dot", "b+PCR", "y1/pw/bcast", "exchange wait", "level2+s", "back(+scale)"]
print(f"N={N} warps sampled {len(b)}; cycles per phase (median / p90):")
for i, nm in enumerate(names):
    print(f"  {nm:14s} {np.median(d[:, i]):8.0f} {np.percentile(d[:, i], 90):8.0f}")
print(f"  total step     {np.median(b[:, 6] - b[:, 0]):8.0f}")
