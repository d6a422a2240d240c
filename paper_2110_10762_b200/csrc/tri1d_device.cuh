// Device-side building blocks of the 1-D implicit propagators, shared by the
// batched/sweep kernels (tri1d.cu) and the asynchronous runtime (async_rt.cu).
// See tri1d.cu for the algorithm (three-level partitioned tridiagonal solve).
#pragma once
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstring>

#include "pint_internal.cuh"

namespace cg = cooperative_groups;

// ============================================================ device side

template <int CH>
struct Tri1DParams {
  ChunkFactors<CH> reg, tail;
  CcstFactors<CH> cc;   // backward-Euler fast path (no tail thread, no forcing)
  const double *table;  // [NF][T]
  int64_t N;
  int64_t steps;
  double E;
  double hq;  // fast path: coupling of a level-2 separator to its neighbour lane (= Ro)
  double f_first, f_last;
  int T, nW, tb;
  int t_last, l_last;
  int has_forcing;
  int l2win;  // level 2 through the 32-column window (one column per lane)
};

#define FULLMASK 0xffffffffu

__device__ __forceinline__ double shfl_up_d(double v, int d) { return __shfl_up_sync(FULLMASK, v, d); }
__device__ __forceinline__ double shfl_down_d(double v, int d) { return __shfl_down_sync(FULLMASK, v, d); }
__device__ __forceinline__ double shfl_d(double v, int l) { return __shfl_sync(FULLMASK, v, l); }

// Trapezoidal rule: raw state x, forward multiplies by q inline.
template <int CH>
__device__ __forceinline__ double chunk_forward_raw(double (&x)[CH], const ChunkFactors<CH> &F, int z) {
  double y0 = F.w[0 + z] * x[0];
  x[0] = F.q[0 + z] * x[0];
#pragma unroll
  for (int j = 1; j < CH - 1; ++j) {
    y0 = fma(F.w[j + z], x[j], y0);
    x[j] = fma(F.e[j + z], x[j - 1], F.q[j + z] * x[j]);
  }
  return y0;
}

template <int CH>
__device__ __forceinline__ void chunk_back_raw(double (&x)[CH], const ChunkFactors<CH> &F, double s_left, int z) {
#pragma unroll
  for (int j = CH - 2; j >= 0; --j) x[j] = fma(F.e[j + z], x[j + 1], fma(F.h[j + z], s_left, x[j]));
}

// Backward Euler: chunk slots carry the pivot-scaled state t_j = q_j x_j
// between steps (the scaling multiply is issued in the back-substitution,
// where it is off the critical path and needs no extra registers); the
// forward elimination is then d'_j = t_j + e_j d'_{j-1}, one FMA per point.
template <int CH>
__device__ __forceinline__ void chunk_scale(double (&x)[CH], const ChunkFactors<CH> &F, int z) {
#pragma unroll
  for (int j = 0; j < CH - 1; ++j) x[j] = F.q[j + z] * x[j];
}

template <int CH>
__device__ __forceinline__ double chunk_forward_scaled(double (&x)[CH], const ChunkFactors<CH> &F, int z) {
  double y0 = F.ws[0 + z] * x[0];
#pragma unroll
  for (int j = 1; j < CH - 1; ++j) {
    y0 = fma(F.ws[j + z], x[j], y0);
    x[j] = fma(F.e[j + z], x[j - 1], x[j]);
  }
  return y0;
}

template <int CH, bool OUT_RAW>
__device__ __forceinline__ void chunk_back_scaled(double (&x)[CH], const ChunkFactors<CH> &F, double s_left, int z) {
  double xn = x[CH - 1];
#pragma unroll
  for (int j = CH - 2; j >= 0; --j) {
    const double xr = fma(F.e[j + z], xn, fma(F.h[j + z], s_left, x[j]));
    x[j] = OUT_RAW ? xr : F.q[j + z] * xr;
    xn = xr;
  }
}

// ---- constant-coefficient twisted chunk solve (backward-Euler fast path) ----
// Chunk slots j = 0..m-1 (m = CH-1) hold chi_j = x_j / rho_j between steps.
template <int CH>
__device__ __forceinline__ void ccst_scale(double (&x)[CH], const double (&f)[CH / 2]) {
  constexpr int m = CH - 1, k = (m - 1) / 2;
#pragma unroll
  for (int i = 0; i < k; ++i) {
    x[i] *= f[i];
    x[m - 1 - i] *= f[i];
  }
}

// Elimination from both ends toward the middle (two independent chains) and
// the two functionals the separator system needs: z0 / zL = first / last
// component of the chunk solve with zero separators. On return x[j], j != k,
// holds the eliminated values psi_j and x[k] the zero-separator middle value.
template <int CH>
__device__ __forceinline__ void ccst_forward(double (&x)[CH], const CcstFactors<CH> &C, double &z0, double &zL) {
  constexpr int m = CH - 1, k = (m - 1) / 2;
  const double mu = C.mu;
  double P = x[0], Q = x[m - 1];
#pragma unroll
  for (int i = 1; i < k; ++i) {
    x[i] = fma(mu, x[i - 1], x[i]);
    x[m - 1 - i] = fma(mu, x[m - i], x[m - 1 - i]);
    P += x[i];
    Q += x[m - 1 - i];
  }
  const double w = fma(mu, x[k - 1] + x[k + 1], x[k]);
  const double gw = C.ga * w;
  z0 = fma(C.al, P, fma(C.be, Q, gw));
  zL = fma(C.be, P, fma(C.al, Q, gw));
  // the separator-independent part of the middle value
  x[k] = fma(C.CmN, z0 + zL, C.kapm * w);
}

// Substitution from the middle outward (two independent chains) once the
// separators on both sides are known; nlz0 / nlzL = nlam * z0 / zL.
template <int CH>
__device__ __forceinline__ void ccst_back(double (&x)[CH], const CcstFactors<CH> &C, double s_left, double s,
                                          double nlz0, double nlzL, int z) {
  constexpr int m = CH - 1, k = (m - 1) / 2;
  const double kap = C.kap;
  // effective boundary values sigma' = sigma - lam x_end, written so that the
  // near-cancellation sA + sB (~ 1 - lam) is formed on the host and the
  // separator difference on the device (both exact to a rounding)
  const double dS = s - s_left;
  const double spL = fma(C.sAB, s_left, fma(C.sB, dS, nlz0));
  const double spR = fma(C.sAB, s, fma(-C.sB, dS, nlzL));
  x[k] = fma(C.CmAB, s_left + s, x[k]);
#pragma unroll
  for (int i = k - 1; i >= 0; --i) {
    const double g = C.g[i + z];
    const double tT = fma(g, spL, x[i]);
    const double tB = fma(g, spR, x[m - 1 - i]);
    x[i] = fma(kap, tT, x[i + 1]);
    x[m - 1 - i] = fma(kap, tB, x[m - 2 - i]);
  }
}

// Per-thread PCR multipliers of the first rounds, held in registers
// for all steps of an application (the rest are re-read from shared memory
// every step: the register file holds the state).
// (all five slots on the fast path: three rounds' multipliers and the four
// closure coefficients plus the lane's two level-1 spikes, 128 registers, no
// spills; none where the general path's extra live values
// would otherwise spill under the two-CTAs-per-SM register cap)
template <bool GENERAL, bool CN>
struct HoistCount {
  static constexpr int value = GENERAL ? 0 : (CN ? 2 : 5);
};
struct Hoisted {
  double a[5], g[5];
  double w1, v1;  // level-1 spikes (fast path only)
};

struct StepCtx {
  uint32_t tab;   // shared address: this thread's table row (NF doubles)
  int TB;
  uint32_t gbuf;  // shared address: gather [2][4][nW+1] doubles
  uint32_t mbar;  // shared address: two mbarriers (one per gather parity)
  int nW;
  int t, lane, Wg;
  int CL;
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// Volatile shared loads: the per-thread tables are re-read every step instead
// of being hoisted into (spilled) registers across the step loop.
__device__ __forceinline__ double lds(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
// Non-volatile shared load: free to be scheduled (and CSE'd) within a step;
// its address comes from opaque() once per step so it is never hoisted out of
// the step loop into (spilled) registers.
__device__ __forceinline__ double lds_free(uint32_t a) {
  double v;
  asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t opaque(uint32_t x) {
  uint32_t y;
  asm volatile("mov.b32 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_async_f64(uint32_t raddr, double v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];"
               :: "r"(raddr), "l"(__double_as_longlong(v)), "r"(rbar) : "memory");
}
__device__ __forceinline__ void st_async_v2f64(uint32_t raddr, double v0, double v1, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];"
               :: "r"(raddr), "l"(__double_as_longlong(v0)), "l"(__double_as_longlong(v1)), "r"(rbar) : "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n}"
      :: "r"(bar), "r"(parity) : "memory");
}

// Publish this warp's level-2 values to every CTA of the cluster and wait for
// the whole slice's values of step `sc` (double buffered by sc & 1; the
// mbarrier of each buffer completes one phase per use). Lanes 0..CL-1 store the
// pair (gH, gP) of warp W at doubles [2W, 2W+1] of the target CTA's buffer with
// ONE 16-byte st.async: the receiving mbarrier absorbs its transaction-count
// updates serially, and halving them (64 instead of 128 per CTA and step)
// took the exchange of a lone slice from 542 to 407 cycles. With EXTRA the
// warp-uniform vX goes to row 2 (a max-reduction riding on the exchange).
template <bool EXTRA>
__device__ __forceinline__ void gather_publish(const StepCtx &c, uint32_t sc, double vH, double vP, double vX) {
  const uint32_t par = sc & 1u;
  const uint32_t stride = (uint32_t)(c.nW + 1);
  const uint32_t gb = c.gbuf + par * 4u * stride * 8u;
  const uint32_t bar = c.mbar + par * 8u;
  if (c.lane < c.CL) {
    const uint32_t rgb = mapa(gb, (uint32_t)c.lane);
    const uint32_t rbar = mapa(bar, (uint32_t)c.lane);
    // one 16-byte store per target CTA: half the transaction-count updates
    // the receiving mbarrier has to absorb per step
    st_async_v2f64(rgb + (uint32_t)c.Wg * 16u, vH, vP, rbar);
    if (EXTRA) st_async_f64(rgb + 2u * stride * 8u + (uint32_t)c.Wg * 8u, vX, rbar);
  }
  if (threadIdx.x == 0) mbar_arrive_expect_tx(bar, (uint32_t)c.nW * (EXTRA ? 3u : 2u) * 8u);
}
__device__ __forceinline__ uint32_t gather_wait(const StepCtx &c, uint32_t sc) {
  const uint32_t par = sc & 1u;
  mbar_wait_parity(c.mbar + par * 8u, (sc >> 1) & 1u);
  return c.gbuf + par * 4u * (uint32_t)(c.nW + 1) * 8u;
}
template <bool EXTRA>
__device__ __forceinline__ uint32_t gather_exchange(const StepCtx &c, uint32_t sc, double vH, double vP, double vX) {
  gather_publish<EXTRA>(c, sc, vH, vP, vX);
  return gather_wait(c, sc);
}

// Work a caller places between a step's publish and its wait (the exchange is
// in flight for several hundred cycles): the fused sweep drains the previous
// slice's results to global memory there.
struct NoShadow {
  __device__ __forceinline__ void operator()() const {}
};

#define TAB(f) lds_free(tab + (uint32_t)(f) * 8u)

#ifdef PINT_PHASE_TIMING
// debug build only (scripts/phase_timing.py): clock64 stamps of one step per warp
static __device__ long long *g_phase_buf;
static __device__ int g_phase_step;
#define PHASE(id)                                                                                         \
  if (g_phase_buf && sc == (uint32_t)g_phase_step && (c.lane == 0)) {                                    \
    g_phase_buf[((size_t)(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5))) * 8 + (id)] = clock64(); \
  }
#else
#define PHASE(id)
#endif

__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(uint32_t dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// One implicit step on the register-resident chunk. `extra_in` (warp-uniform)
// is published through the gather and its max over all warps of the slice is
// returned in *extra_out when WITH_EXTRA. Backward Euler: IN_RAW means the
// chunk slots hold the raw state (else the pivot-scaled one), OUT_RAW asks for
// a raw result (else scaled for the next step). The separator is always raw.
template <int CH, int J, bool CN, bool GENERAL, bool IN_RAW, bool OUT_RAW, bool WITH_EXTRA, typename Shadow = NoShadow>
__device__ __forceinline__ void tri_step(double (&x)[CH], const Tri1DParams<CH> &P, const StepCtx &c,
                                         const Hoisted &H, uint32_t sc, double extra_in, double *extra_out,
                                         const Shadow &shadow = Shadow()) {
  constexpr bool CC = !CN && !GENERAL;  // constant-coefficient twisted chunk solve
  const bool regular = !GENERAL || c.t < P.tb;
  const uint32_t tab = opaque(c.tab);
  // A uniform, step-variant zero (step counters stay below 2^31, checked on
  // the host): indexing the chunk factors with it keeps them in the constant
  // bank, loaded straight into uniform registers (LDCU) for each DFMA every
  // step, instead of being hoisted into general registers and moved back
  // (R2UR) before every use: -13 % per step at C2.
  const int z = (int)(sc >> 31);
  PHASE(0)
  double xo[CN ? CH : 1];
  if (CN) {
#pragma unroll
    for (int j = 0; j < CH; ++j) xo[j] = x[j];
  } else if (CC) {
    if (IN_RAW) ccst_scale<CH>(x, P.cc.rs);
  } else if (IN_RAW) {
    if (regular) chunk_scale<CH>(x, P.reg, z);
    else chunk_scale<CH>(x, P.tail, z);
  }
  if (GENERAL && P.has_forcing) {
    if (c.t == 0) x[0] += P.f_first;
    if (c.t == P.t_last) {
#pragma unroll
      for (int j = 0; j < CH; ++j)
        if (j == P.l_last) x[j] += P.f_last;
    }
  }
  double y0, ylast;
  if (CC) {
    ccst_forward<CH>(x, P.cc, y0, ylast);
  } else if (CN) {
    if (regular) y0 = chunk_forward_raw<CH>(x, P.reg, z);
    else y0 = chunk_forward_raw<CH>(x, P.tail, z);
    ylast = x[CH - 2];
  } else {
    if (regular) y0 = chunk_forward_scaled<CH>(x, P.reg, z);
    else y0 = chunk_forward_scaled<CH>(x, P.tail, z);
    ylast = x[CH - 2];
  }
  PHASE(1)
  const double dsep = x[CH - 1];
  // (fast path) the corner terms of the effective boundary values, formed
  // here, off the critical path that follows the exchange
  const double nlz0 = CC ? P.cc.nlam * y0 : 0.0;
  const double nlzL = CC ? P.cc.nlam * ylast : 0.0;
  double y0n = shfl_down_d(y0, 1);
  if (c.lane == 31) y0n = 0.0;
  double b = dsep - P.E * (ylast + y0n);
  if (GENERAL) b *= TAB(TF_MASK);  // virtual separators (all real on the fast path)
  constexpr int NH = HoistCount<GENERAL, CN>::value;
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const int d = 1 << r;
    const double bm = shfl_up_d(b, d);
    const double bp = shfl_down_d(b, d);
    const double ka = r < NH ? H.a[r] : TAB(TF_PCR_A + r);
    const double kg = r < NH ? H.g[r] : TAB(TF_PCR_G + r);
    b = fma(-kg, bp, fma(-ka, bm, b));
  }
  PHASE(2)
  // the eight 4-lane systems left by three rounds, closed by their dense
  // inverses (lane 31: all coefficients 0, its value is the level-2 unknown)
  const double c0 = 3 < NH ? H.a[3] : TAB(TF_PCR_A + 3);
  const double c16 = 3 < NH ? H.g[3] : TAB(TF_PCR_G + 3);
  const double b8 = __shfl_xor_sync(FULLMASK, b, 8);
  const double b16 = __shfl_xor_sync(FULLMASK, b, 16);
  const double b24 = __shfl_xor_sync(FULLMASK, b, 24);
  const double c8 = 4 < NH ? H.a[4] : TAB(TF_PCR_A + 4);
  const double c24 = 4 < NH ? H.g[4] : TAB(TF_PCR_G + 4);
  const double y1 = fma(c8, b8, c0 * b) + fma(c24, b24, c16 * b16);
  const double y1_30 = shfl_d(y1, 30);
  const double pw = fma(-TAB(TF_CP), y1_30, b);
  // what the previous warp's level-2 row needs from this warp, combined on the
  // sender: h = Ro y1_0 + E y0_0 (lane 0's values; coefficients of column W - 1)
  const double h0 = GENERAL ? fma(TAB(TF_HQ(J)), y1, TAB(TF_HZ(J)) * y0) : fma(P.hq, y1, P.E * y0);
  const double gP = shfl_d(pw, 31);
  const double gH = shfl_d(h0, 0);
  PHASE(3)
  gather_publish<WITH_EXTRA>(c, sc, gH, gP, extra_in);
  shadow();
  const uint32_t gb = opaque(gather_wait(c, sc));
  PHASE(4)
  const uint32_t stride8 = (uint32_t)(c.nW + 1) * 8u;
  double sl = 0.0, sr = 0.0, ex = 0.0;
  if (J > 1 && P.l2win) {
    // one column per lane: the 32-column window of R2^{-1} around the diagonal
    const int V = min(max(c.Wg - 16, 0), c.nW - 32) + c.lane;
    const uint32_t o = (uint32_t)V * 16u;  // pairs (gH_V, gP_V): B = gP_V - gH_{V+1}
    const double B = lds_free(gb + o + 8u) - lds_free(gb + o + 16u);
    sl = TAB(TF_R2) * B;
    sr = TAB(TF_R2 + J) * B;
    if (WITH_EXTRA) {
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const int Vx = c.lane + 32 * j;
        if (Vx < c.nW) ex = fmax(ex, lds_free(gb + 2u * stride8 + (uint32_t)Vx * 8u));
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const int V = c.lane + 32 * j;
      double B = 0.0;
      if (V < c.nW) {
        const uint32_t o = (uint32_t)V * 16u;
        B = lds_free(gb + o + 8u) - lds_free(gb + o + 16u);
        if (WITH_EXTRA) ex = fmax(ex, lds_free(gb + 2u * stride8 + (uint32_t)V * 8u));
      }
      sl = fma(TAB(TF_R2 + j), B, sl);
      sr = fma(TAB(TF_R2 + J + j), B, sr);
    }
  }
  // split butterfly: the lower half-warp reduces sl, the upper half sr
  {
    const bool lo = c.lane < 16;
    double keep = lo ? sl : sr;
    keep += __shfl_xor_sync(FULLMASK, lo ? sr : sl, 16);
#pragma unroll
    for (int o = 8; o >= 1; o >>= 1) keep += __shfl_xor_sync(FULLMASK, keep, o);
    // every lane of the lower half now holds sl, of the upper half sr
    const double other = __shfl_xor_sync(FULLMASK, keep, 16);
    sl = lo ? keep : other;
    sr = lo ? other : keep;
  }
  if (WITH_EXTRA) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) ex = fmax(ex, __shfl_xor_sync(FULLMASK, ex, o));
  }
  if (WITH_EXTRA) *extra_out = ex;
  // the tables of lane 31 (W1 = 0, V1 = 1, y1 = 0) make its value sr
  const double s = NH == 5 ? fma(H.v1, sr, fma(H.w1, sl, y1)) : fma(TAB(TF_V1), sr, fma(TAB(TF_W1), sl, y1));
  double s_left = shfl_up_d(s, 1);
  if (c.lane == 0) s_left = sl;
  PHASE(5)
  x[CH - 1] = s;
  if (CC) {
    ccst_back<CH>(x, P.cc, s_left, s, nlz0, nlzL, z);
    if (OUT_RAW) ccst_scale<CH>(x, P.cc.ro);
  } else if (CN) {
    if (regular) chunk_back_raw<CH>(x, P.reg, s_left, z);
    else chunk_back_raw<CH>(x, P.tail, s_left, z);
  } else {
    if (regular) chunk_back_scaled<CH, OUT_RAW>(x, P.reg, s_left, z);
    else chunk_back_scaled<CH, OUT_RAW>(x, P.tail, s_left, z);
  }
  if (CN) {
#pragma unroll
    for (int j = 0; j < CH; ++j) x[j] = fma(2.0, x[j], -xo[j]);
  }
  PHASE(6)
}

// Shared-memory setup common to all kernels. Ends with a cluster barrier so
// the mbarriers and zeroed gather buffers are initialised cluster-wide before
// any remote store.
template <int CH, int J>
__device__ __forceinline__ StepCtx setup_ctx(const Tri1DParams<CH> &P, double *smem, int rank) {
  StepCtx c;
  c.TB = blockDim.x;
  c.CL = P.T / c.TB;
  c.nW = P.nW;
  c.t = rank * c.TB + threadIdx.x;
  c.lane = threadIdx.x & 31;
  c.Wg = c.t >> 5;
  const int NF = TRI1D_NF(J);  // odd: the per-thread rows are bank-conflict free
  double *tab = smem;
  for (int f = 0; f < NF; ++f) tab[threadIdx.x * NF + f] = P.table[(size_t)f * P.T + c.t];
  c.tab = smem_u32(tab + threadIdx.x * NF);
  double *gbuf = smem + NF * c.TB;
  for (int i = threadIdx.x; i < 8 * (c.nW + 1); i += c.TB) gbuf[i] = 0.0;
  c.gbuf = smem_u32(gbuf);
  uint64_t *bars = reinterpret_cast<uint64_t *>(gbuf + 8 * (c.nW + 1));
  c.mbar = smem_u32(bars);
  if (threadIdx.x == 0) {
    mbar_init(c.mbar, 1);
    mbar_init(c.mbar + 8, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  cg::this_cluster().sync();
  return c;
}

// S implicit steps from a raw state to a raw state; the step counter `sc`
// drives the double-buffered exchange. With extra_out != nullptr the first
// step also reduces extra_in (max) over the slice.
template <int CH, int J, bool CN, bool GENERAL, typename Shadow = NoShadow>
__device__ __forceinline__ void run_steps(double (&x)[CH], const Tri1DParams<CH> &P, const StepCtx &c,
                                          uint32_t &sc, int64_t S, double extra_in, double *extra_out,
                                          const Shadow &shadow = Shadow()) {
  Hoisted H;
#pragma unroll
  for (int r = 0; r < HoistCount<GENERAL, CN>::value; ++r) {
    H.a[r] = lds(c.tab + (uint32_t)(TF_PCR_A + r) * 8u);
    H.g[r] = lds(c.tab + (uint32_t)(TF_PCR_G + r) * 8u);
  }
  if (HoistCount<GENERAL, CN>::value == 5) {
    H.w1 = lds(c.tab + (uint32_t)TF_W1 * 8u);
    H.v1 = lds(c.tab + (uint32_t)TF_V1 * 8u);
  }
  // `shadow` runs once, inside the first step's exchange
  if (S == 1) {
    if (extra_out) tri_step<CH, J, CN, GENERAL, true, true, true>(x, P, c, H, sc, extra_in, extra_out, shadow);
    else tri_step<CH, J, CN, GENERAL, true, true, false>(x, P, c, H, sc, 0.0, nullptr, shadow);
    ++sc;
    return;
  }
  if (extra_out) tri_step<CH, J, CN, GENERAL, true, false, true>(x, P, c, H, sc, extra_in, extra_out, shadow);
  else tri_step<CH, J, CN, GENERAL, true, false, false>(x, P, c, H, sc, 0.0, nullptr, shadow);
  ++sc;
  for (int64_t s = 1; s < S - 1; ++s, ++sc)
    tri_step<CH, J, CN, GENERAL, false, false, false>(x, P, c, H, sc, 0.0, nullptr);
  tri_step<CH, J, CN, GENERAL, false, true, false>(x, P, c, H, sc, 0.0, nullptr);
  ++sc;
}

template <int CH>
__device__ __forceinline__ void load_chunk(double (&x)[CH], const double *src, int64_t N, int t) {
  const int64_t base = (int64_t)t * CH;
  const double *p = src + base;
  if (base + CH <= N && ((reinterpret_cast<uintptr_t>(p) & 15) == 0)) {
#pragma unroll
    for (int j = 0; j < CH; j += 2) {
      double2 v = *reinterpret_cast<const double2 *>(p + j);
      x[j] = v.x;
      x[j + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int j = 0; j < CH; ++j) x[j] = (base + j < N) ? p[j] : 0.0;
  }
}

template <int CH>
__device__ __forceinline__ void store_chunk(const double (&x)[CH], double *dst, int64_t N, int t) {
  const int64_t base = (int64_t)t * CH;
  double *p = dst + base;
  if (base + CH <= N && ((reinterpret_cast<uintptr_t>(p) & 15) == 0)) {
#pragma unroll
    for (int j = 0; j < CH; j += 2) *reinterpret_cast<double2 *>(p + j) = make_double2(x[j], x[j + 1]);
  } else {
#pragma unroll
    for (int j = 0; j < CH; ++j)
      if (base + j < N) p[j] = x[j];
  }
}


__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v = fmax(v, __shfl_xor_sync(FULLMASK, v, o));
  return v;
}

// ============================================================== launchers

template <int CH>
static Tri1DParams<CH> make_params(const pint_op *op) {
  const Tri1DPlan &pl = op->plan;
  Tri1DParams<CH> P;
  memset(&P, 0, sizeof(P));
  for (int j = 0; j < CH; ++j) {
    P.reg.q[j] = pl.fac_reg[0 * CH + j];
    P.reg.e[j] = pl.fac_reg[1 * CH + j];
    P.reg.h[j] = pl.fac_reg[2 * CH + j];
    P.reg.w[j] = pl.fac_reg[3 * CH + j];
    P.tail.q[j] = pl.fac_tail[0 * CH + j];
    P.tail.e[j] = pl.fac_tail[1 * CH + j];
    P.tail.h[j] = pl.fac_tail[2 * CH + j];
    P.tail.w[j] = pl.fac_tail[3 * CH + j];
    P.reg.ws[j] = pl.fac_reg[4 * CH + j];
    P.tail.ws[j] = pl.fac_tail[4 * CH + j];
  }
  if (pl.ccst) {
    const double *f = pl.ccst_fac.data();
    P.cc.mu = f[0]; P.cc.kap = f[1]; P.cc.kapm = f[2];
    P.cc.al = f[3]; P.cc.be = f[4]; P.cc.ga = f[5];
    P.cc.sAB = f[6]; P.cc.sB = f[7]; P.cc.nlam = f[8]; P.cc.CmAB = f[9]; P.cc.CmN = f[10];
    for (int i = 0; i < CH / 2; ++i) {
      P.cc.g[i] = f[11 + i];
      P.cc.rs[i] = f[11 + CH / 2 + i];
      P.cc.ro[i] = f[11 + 2 * (CH / 2) + i];
    }
  }
  P.table = op->d_table;
  P.N = pl.N;
  P.steps = pl.steps;
  P.E = pl.E;
  P.hq = pl.hq;
  P.l2win = pl.l2win ? 1 : 0;
  P.f_first = pl.cn ? pl.f_first : pl.fq_first;
  P.f_last = pl.cn ? pl.f_last : pl.fq_last;
  P.T = pl.T;
  P.nW = pl.nW;
  P.tb = pl.tb;
  P.t_last = pl.t_last;
  P.l_last = pl.l_last;
  P.has_forcing = (pl.f_first != 0.0 || pl.f_last != 0.0) ? 1 : 0;
  return P;
}

template <typename Kern, typename... Args>
static void launch_cluster(Kern kern, int grid, int block, int cl, size_t smem, cudaStream_t s,
                           Args... args) {
  PINT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (cl > 8) PINT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(block, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (const char *pol = getenv("PINT_CLUSTER_POLICY")) {  // 1 = spread, 2 = load balancing (probe)
    attr[1].id = cudaLaunchAttributeClusterSchedulingPolicyPreference;
    attr[1].val.clusterSchedulingPolicyPreference =
        atoi(pol) == 1 ? cudaClusterSchedulingPolicySpread : cudaClusterSchedulingPolicyLoadBalancing;
    cfg.numAttrs = 2;
  }
  PINT_CUDA(cudaLaunchKernelEx(&cfg, kern, args...));
}

