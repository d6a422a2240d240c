"""Test infrastructure: numpy emulation of one step of the 1-D partitioned
tridiagonal kernel (paper_2110_10762_b200/csrc/tri1d.cu, tri_step) driven by
the exact host plan exported through pint_tri1d_plan_host. Used on CPU to
check the plan (a step of the emulated algorithm must solve K x = d) and to
study rounding; it is not a product path."""
from __future__ import annotations

import ctypes

import numpy as np

from paper_2110_10762_b200 import _native


def export_plan(n, a_d, a_o, c_first, c_last, span, steps, rule="backward-euler"):
    lib = _native.load_library()
    d = _native.OpDesc()
    d.ndim = 1
    d.rule = {"backward-euler": 0, "trapezoidal": 1}[rule]
    d.dtype = _native.PINT_F64
    d.shape[0] = n
    d.span = span
    d.steps = steps
    d.a_diag, d.a_off, d.c_first, d.c_last = a_d, a_o, c_first, c_last
    dims = (ctypes.c_int32 * 6)()
    rc = lib.pint_tri1d_plan_host(ctypes.byref(d), dims, None, None, None)
    assert rc == 0, rc
    CH, T, nW, J, tb, NF = list(dims)
    fac = np.zeros(10 * CH)
    tab = np.zeros(NF * T)
    scal = np.zeros(8)
    rc = lib.pint_tri1d_plan_host(ctypes.byref(d), dims, fac.ctypes.data_as(ctypes.c_void_p),
                                  tab.ctypes.data_as(ctypes.c_void_p), scal.ctypes.data_as(ctypes.c_void_p))
    assert rc == 0
    ccst, ccfac = False, None
    if rule == "backward-euler":
        usable = ctypes.c_int32(0)
        ccfac = np.zeros(11 + 3 * (CH // 2))
        rc = lib.pint_tri1d_ccst_host(ctypes.byref(d), ctypes.byref(usable), ccfac.ctypes.data_as(ctypes.c_void_p))
        assert rc == 0
        ccst = bool(usable.value)
    return dict(CH=CH, T=T, nW=nW, J=J, tb=tb, NF=NF, fac=fac.reshape(2, 5, CH), tab=tab.reshape(NF, T),
                D=scal[0], E=scal[1], f_first=scal[2], f_last=scal[3], N=n, cn=(rule == "trapezoidal"),
                ccst=ccst, ccfac=ccfac)


def _fma(a, b, c):
    return (np.longdouble(a) * np.longdouble(b) + np.longdouble(c)).astype(np.float64)


def _shfl_up(v, d):
    w = v.reshape(-1, 32)
    out = w.copy()
    out[:, d:] = w[:, :-d]
    return out.reshape(-1)


def _shfl_xor(v, m):
    w = v.reshape(-1, 32)
    return w[:, np.arange(32) ^ m].reshape(-1)


def _shfl_down(v, d):
    w = v.reshape(-1, 32)
    out = w.copy()
    out[:, :-d] = w[:, d:]
    return out.reshape(-1)


def step(x_points: np.ndarray, P: dict) -> np.ndarray:
    """One implicit step (raw state in, raw state out) of a (N,) state."""
    CH, T, nW, J, tb, N = P["CH"], P["T"], P["nW"], P["J"], P["tb"], P["N"]
    E = P["E"]
    x = np.zeros(T * CH)
    x[:N] = x_points
    x = x.reshape(T, CH)
    cls = (np.arange(T) >= tb).astype(int)
    q, e, h, w, ws = (P["fac"][cls, k, :] for k in range(5))
    xo = x.copy()
    tab = P["tab"]
    cn = P["cn"]
    cc = P.get("ccst", False) and not cn
    if cc:
        # fast path (tri1d_device.cuh: ccst_scale / ccst_forward / ccst_back)
        m, k, h2 = CH - 1, (CH - 2) // 2, CH // 2
        f = P["ccfac"]
        mu, kap, kapm, al, be, ga, sAB, sB, nlam, CmAB, CmN = f[:11]
        g, rs, ro = f[11:11 + h2], f[11 + h2:11 + 2 * h2], f[11 + 2 * h2:11 + 3 * h2]
        for i in range(k):
            x[:, i] = x[:, i] * rs[i]
            x[:, m - 1 - i] = x[:, m - 1 - i] * rs[i]
    elif not cn:
        x[:, :CH - 1] = q[:, :CH - 1] * x[:, :CH - 1]
    if P["f_first"] != 0.0 or P["f_last"] != 0.0:
        raise NotImplementedError("emulator covers the zero-forcing case")
    d = x.copy()
    if cc:
        Ps, Qs = d[:, 0].copy(), d[:, m - 1].copy()
        for i in range(1, k):
            d[:, i] = _fma(mu, d[:, i - 1], d[:, i])
            d[:, m - 1 - i] = _fma(mu, d[:, m - i], d[:, m - 1 - i])
            Ps = Ps + d[:, i]
            Qs = Qs + d[:, m - 1 - i]
        wmid = _fma(mu, d[:, k - 1] + d[:, k + 1], d[:, k])
        gw = ga * wmid
        y0 = _fma(al, Ps, _fma(be, Qs, gw))
        zL = _fma(be, Ps, _fma(al, Qs, gw))
        d[:, k] = _fma(CmN, y0 + zL, kapm * wmid)
        d[:, CH - 2] = d[:, CH - 2]  # (ylast below is zL)
    elif cn:
        y0 = w[:, 0] * d[:, 0]
        d[:, 0] = q[:, 0] * d[:, 0]
        for j in range(1, CH - 1):
            y0 = _fma(w[:, j], x[:, j], y0)
            d[:, j] = _fma(e[:, j], d[:, j - 1], q[:, j] * x[:, j])
    else:
        y0 = ws[:, 0] * d[:, 0]
        for j in range(1, CH - 1):
            y0 = _fma(ws[:, j], d[:, j], y0)
            d[:, j] = _fma(e[:, j], d[:, j - 1], d[:, j])
    ylast = zL if cc else d[:, CH - 2]
    dsep = d[:, CH - 1]
    lane = np.arange(T) % 32
    y0n = _shfl_down(y0, 1)
    y0n[lane == 31] = 0.0
    b = tab[0] * (dsep - E * (ylast + y0n))
    for r in range(3):
        dd = 1 << r
        bm = _shfl_up(b, dd)
        bp = _shfl_down(b, dd)
        b = _fma(-tab[6 + r], bp, _fma(-tab[1 + r], bm, b))
    # dense closure of the eight 4-lane systems (C0, C8 in PCR_A slots 3, 4; C16, C24 in PCR_G slots 3, 4)
    y1 = _fma(tab[1 + 4], _shfl_xor(b, 8), tab[1 + 3] * b) + _fma(tab[6 + 4], _shfl_xor(b, 24), tab[6 + 3] * _shfl_xor(b, 16))
    y1w = y1.reshape(nW, 32)
    bw = b.reshape(nW, 32)
    pw = _fma(-tab[14].reshape(nW, 32)[:, 31], y1w[:, 30], bw[:, 31])
    # sender-side combination h_W = cq y1_0 + cz y0_0 (coefficients of column W - 1)
    hq = tab[15 + 2 * J].reshape(nW, 32)[:, 0]
    hz = tab[16 + 2 * J].reshape(nW, 32)[:, 0]
    Hh = np.append(_fma(hq, y1w[:, 0], hz * y0.reshape(nW, 32)[:, 0]), 0.0)
    sl = np.zeros(T)
    sr = np.zeros(T)
    # level-2 window (tri1d.cu): the plan zeroes the fields of columns j >= 1
    # when one 32-column window of R2^{-1} per warp suffices
    windowed = J > 1 and not tab[15 + 1:15 + J].any() and not tab[15 + J + 1:15 + 2 * J].any()
    if windowed:
        Wg = np.arange(T) // 32
        V = np.minimum(np.maximum(Wg - 16, 0), nW - 32) + lane
        B = pw[V] - Hh[V + 1]
        sl = tab[15] * B
        sr = tab[15 + J] * B
    else:
        for j in range(J):
            V = lane + 32 * j
            ok = V < nW
            Vc = np.minimum(V, nW - 1)
            B = np.where(ok, pw[Vc] - Hh[np.minimum(V + 1, nW)], 0.0)
            sl = sl + tab[15 + j] * B
            sr = sr + tab[15 + J + j] * B
    sl = sl.reshape(nW, 32).sum(axis=1).repeat(32)
    sr = sr.reshape(nW, 32).sum(axis=1).repeat(32)
    s = _fma(tab[13], sr, _fma(tab[12], sl, y1))
    s[lane == 31] = sr[lane == 31]
    s_left = _shfl_up(s, 1)
    s_left[lane == 0] = sl[lane == 0]
    out = d.copy()
    out[:, CH - 1] = s
    if cc:
        nlz0, nlzL = nlam * y0, nlam * zL
        dS = s - s_left
        spL = _fma(sAB, s_left, _fma(sB, dS, nlz0))
        spR = _fma(sAB, s, _fma(-sB, dS, nlzL))
        out[:, k] = _fma(CmAB, s_left + s, d[:, k])
        for i in range(k - 1, -1, -1):
            tT = _fma(g[i], spL, d[:, i])
            tB = _fma(g[i], spR, d[:, m - 1 - i])
            out[:, i] = _fma(kap, tT, out[:, i + 1])
            out[:, m - 1 - i] = _fma(kap, tB, out[:, m - 2 - i])
        for i in range(k):
            out[:, i] = out[:, i] * ro[i]
            out[:, m - 1 - i] = out[:, m - 1 - i] * ro[i]
        return out.reshape(-1)[:N]
    xn = s.copy()
    for j in range(CH - 2, -1, -1):
        xr = _fma(e[:, j], xn, _fma(h[:, j], s_left, d[:, j]))
        out[:, j] = xr
        xn = xr
    if cn:
        out = 2.0 * out - xo
    return out.reshape(-1)[:N]
