"""Numerical prototype (CPU, numpy fp64) of the constant-coefficient twisted
chunk solve planned for the 1-D backward-Euler fine kernel: emulates the
device's per-thread arithmetic (same operation order, fma emulated through
long double where it matters little) and compares S steps against the
long-double truth."""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from oracle import heat_oracle as H
from oracle.truth import TruthTridiag1D
import scipy.linalg as sl

ld = np.longdouble

def plan(D, E, CH=32):
    D = ld(D); E = ld(E)
    m = CH - 1; k = m // 2
    c = (D + np.sqrt(D * D - 4 * E * E)) / 2
    lam = -E / c
    mu = lam * lam
    kap = 1 / c
    kap_m = 1 / (c * (1 - mu))
    rho = np.array([lam ** abs(j - k) for j in range(m)], dtype=ld)
    # exact chunk matrix and twisted constant matrix
    Kc = np.zeros((m, m), dtype=ld)
    for j in range(m):
        Kc[j, j] = D
        if j: Kc[j, j - 1] = E
        if j < m - 1: Kc[j, j + 1] = E
    delta = D - c
    Tt = Kc.copy(); Tt[0, 0] -= delta; Tt[m - 1, m - 1] -= delta
    Kci = np.linalg.inv(Kc.astype(np.float64)).astype(ld)
    # refine inverse in long double (one Newton step)
    I = np.eye(m, dtype=ld)
    for _ in range(3):
        Kci = Kci + Kci @ (I - Kc @ Kci)
    Tti = np.linalg.inv(Tt.astype(np.float64)).astype(ld)
    for _ in range(3):
        Tti = Tti + Tti @ (I - Tt @ Tti)
    a = Tti[0, 0]; b = Tti[0, m - 1]
    M = np.linalg.inv(np.array([[1 + delta * a, delta * b], [delta * b, 1 + delta * a]], dtype=np.float64)).astype(ld)
    lk = lam ** k
    # z0~ = lk*(kap*P + zk~), zk~ = kap_m * w
    al = M[0, 0] * lk * kap; be = M[0, 1] * lk * kap; ga = (M[0, 0] + M[0, 1]) * lk * kap_m
    vL0 = Kci[0, 0] * (-E); vR0 = Kci[0, m - 1] * (-E)
    g = np.array([-E * lam ** (2 * j - k) for j in range(k)], dtype=ld)  # top half contamination (psi_j += g_j sigma')
    Cm = kap_m * (-E) * lk
    return dict(m=m, k=k, c=c, lam=lam, mu=mu, kap=kap, kap_m=kap_m, rho=rho, al=al, be=be, ga=ga,
                sA=1 - lam * vL0, sB=-lam * vR0, lamv=lam, g=g, Cm=Cm, Kci=Kci, D=D, E=E)

def f(x):
    return np.float64(x)

def step(chi, sep, P_, Rsolve):
    """chi: [T, m] scaled interior, sep: [T] raw separators. returns new."""
    m, k = P_["m"], P_["k"]
    mu = f(P_["mu"]); kap = f(P_["kap"]); kap_m = f(P_["kap_m"])
    T = chi.shape[0]
    psi = chi.copy()
    for j in range(1, k):
        psi[:, j] = mu * psi[:, j - 1] + chi[:, j]
    for j in range(m - 2, k, -1):
        psi[:, j] = mu * psi[:, j + 1] + chi[:, j]
    Psum = psi[:, :k].sum(axis=1)
    Qsum = psi[:, k + 1:].sum(axis=1)
    w = chi[:, k] + mu * (psi[:, k - 1] + psi[:, k + 1])
    al, be, ga = f(P_["al"]), f(P_["be"]), f(P_["ga"])
    z0 = al * Psum + be * Qsum + ga * w
    zL = be * Psum + al * Qsum + ga * w
    E = f(P_["E"])
    z0n = np.concatenate([z0[1:], [0.0]])
    b = sep - E * (zL + z0n)
    s = Rsolve(b)
    sL = np.concatenate([[0.0], s[:-1]])
    sA, sB, lam = f(P_["sA"]), f(P_["sB"]), f(P_["lamv"])
    spL = sA * sL + sB * s - lam * z0
    spR = sA * s + sB * sL - lam * zL
    new = np.empty_like(chi)
    new[:, k] = kap_m * w + f(P_["Cm"]) * (spL + spR)
    g = P_["g"].astype(np.float64)
    for j in range(k - 1, -1, -1):
        t = psi[:, j] + g[j] * spL
        new[:, j] = kap * t + new[:, j + 1]
    for j in range(k + 1, m):
        t = psi[:, j] + g[m - 1 - j] * spR
        new[:, j] = kap * t + new[:, j - 1]
    return new, s

def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
    S = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
    Pn = int(sys.argv[3]) if len(sys.argv) > 3 else 64
    modes = 32 if N > 2000 else 8
    CH = 32
    assert N % CH == 0
    T = N // CH
    a_d, a_o, cc = H.heat1d_coeffs(N)
    dt = 1.0 / Pn / S
    tru = TruthTridiag1D(N, a_d, a_o, cc, 1.0 / Pn, S)
    D, E = tru.D, tru.E
    print("D,E", D, E)
    P_ = plan(D, E, CH)
    print("lam", float(P_["lam"]), "Cm", float(P_["Cm"]), "sA", float(P_["sA"]), "sB", float(P_["sB"]))
    m = CH - 1
    # Schur complement of separators (exact chunk inverses), solved densely-banded in fp64
    Kci = P_["Kci"]
    i00 = Kci[0, 0]; iLL = Kci[m - 1, m - 1]; i0L = Kci[0, m - 1]
    Dl, El = ld(D), ld(E)
    Rd = np.full(T, Dl - El * El * iLL - El * El * i00, dtype=ld)
    Rd[T - 1] = Dl - El * El * iLL  # last separator has no right chunk
    Ro = -El * El * i0L
    ab = np.zeros((3, T)); ab[1] = Rd.astype(np.float64); ab[0, 1:] = float(Ro); ab[2, :-1] = float(Ro)
    def Rsolve(b):
        return sl.solve_banded((1, 1), ab, b)
    u0 = H.sine_u0_1d(N, modes, seed=0)
    x = u0.reshape(T, CH).copy()
    rho = P_["rho"].astype(np.float64)
    chi = x[:, :m] / rho
    sep = x[:, m].copy()
    for _ in range(S):
        chi, sep = step(chi, sep, P_, Rsolve)
    out = np.concatenate([chi * rho, sep[:, None]], axis=1).reshape(-1)
    want = tru.apply(u0)
    print("rel-L2 vs long-double truth after", S, "steps:", np.linalg.norm(out - want) / np.linalg.norm(want))
    # plain fp64 LAPACK route for comparison
    ref = H.Tridiag1D(N, a_d, a_o, cc, 1.0 / Pn, S).apply(u0)
    print("fp64 LAPACK route:", np.linalg.norm(ref - want) / np.linalg.norm(want))

main()
