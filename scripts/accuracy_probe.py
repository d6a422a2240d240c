"""Accuracy probe: GPU 1-D propagator vs the numpy kernel emulator, LAPACK and
a long-double Thomas truth (C1 operators)."""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
import paper_2110_10762_b200 as pb
from oracle import heat_oracle as H
import tri1d_emulator as EM

def truth_step(x, D, E):
    n = len(x); D = np.longdouble(D); E = np.longdouble(E)
    cp = np.zeros(n, dtype=np.longdouble); dp = np.zeros(n, dtype=np.longdouble)
    cp[0] = E / D; dp[0] = x[0] / D
    for i in range(1, n):
        m = D - E * cp[i - 1]; cp[i] = E / m; dp[i] = (x[i] - E * dp[i - 1]) / m
    out = np.zeros(n, dtype=np.longdouble); out[-1] = dp[-1]
    for i in range(n - 2, -1, -1): out[i] = dp[i] - cp[i] * out[i + 1]
    return out

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
a_d, a_o, c = H.heat1d_coeffs(n)
u0 = H.sine_u0_1d(n, 8, 0)
ivp = pb.heat1d_system(n, 1.0, 0.0, 0.0, 0.0, 1.0)
for name, span, steps in (("G", 1 / 16, 1), ("F2", 1 / 1600, 2), ("F5", 5 / 1600, 5), ("F", 1 / 16, 100)):
    P = EM.export_plan(n, a_d, a_o, 0.0, 0.0, span, steps)
    ora = H.Tridiag1D(n, a_d, a_o, c, span, steps)
    gpu = pb.backward_euler_propagator(ivp, span, steps)
    xg = gpu.apply(u0)
    xe = u0.copy(); xt = u0.astype(np.longdouble); xo = u0.copy()
    for s in range(steps):
        xe = EM.step(xe, P); xt = truth_step(xt, P["D"], P["E"]); xo = ora.step(xo)
    xt = xt.astype(np.float64); nt = np.linalg.norm(xt)
    e = lambda a: np.linalg.norm(a - xt) / nt
    print(f"{name}: gpu {e(xg):.2e} emu {e(xe):.2e} lapack {e(xo):.2e} gpu-vs-emu {np.linalg.norm(xg-xe)/nt:.2e} maxabs {np.max(np.abs(xg-xe)):.2e} at {np.argmax(np.abs(xg-xe))}")
