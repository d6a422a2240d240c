// Batched implicit 1-D propagators (backward Euler / trapezoidal) for the
// symmetric constant-coefficient tridiagonal operators of heat1d_system and
// scalar_decay_system (reference: model.py:172-200, 209-243).
//
// The reference materialises the S-step map as a dense matrix
// (fine_from_onestep, model.py:147-154) and applies it as a matvec
// (AffinePropagator.apply, model.py:123-129). Here each application runs S
// implicit steps matrix-free with the slice state held in REGISTERS for all
// steps; HBM sees one read and one write of the state per application.
//
// Per step the system K x = d, K = tridiag(E, D, E) of size N, is solved
// exactly (no truncation) by a three-level partition:
//   level 0  each thread owns CH consecutive points: CH-1 "chunk" points and
//            one separator. Chunks are solved with zero-Dirichlet ends by a
//            Thomas sweep whose factors are uniform across threads (kernel
//            parameters -> constant-bank operands); the chunk's dependence on
//            the two adjacent separators is two precomputed spike vectors.
//   level 1  the separators form a symmetric tridiagonal Schur complement R.
//            Inside each warp, lanes 0..30 are solved by parallel cyclic
//            reduction over warp shuffles (5 rounds, precomputed multipliers).
//   level 2  lane 31 of every warp is a level-2 separator; the level-2 Schur
//            complement R2 (nW x nW, nW = warps per slice) is inverted on the
//            host and each warp forms the two values it needs by a dot product
//            of its two rows of R2^{-1} with the gathered right-hand side.
//            The gather crosses CTAs of the thread-block cluster through DSMEM
//            with st.async + mbarrier transaction counts (no cluster-wide
//            barrier or fence in the step loop; buffers double-buffered).
// Every multiplier is data independent and computed once per operator on the
// host in long double. The arithmetic per point does not depend on how the
// T threads of a slice are split into CTAs, so batch, single and fused-sweep
// launches give bitwise identical results (required by parareal.py:34-35
// caching/cancellation and the bitwise finite-termination tests,
// test_parareal.py:81-104).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "pint_internal.cuh"

namespace cg = cooperative_groups;
typedef long double ld;

// ================================================================ host plan

// Solve a general tridiagonal system (sub a, diag b, super c) in long double.
static void tri_solve_ld(int n, const ld *a, const ld *b, const ld *c, ld *rhs) {
  if (n <= 0) return;
  std::vector<ld> cp(n), dp(n);
  cp[0] = c[0] / b[0];
  dp[0] = rhs[0] / b[0];
  for (int i = 1; i < n; ++i) {
    ld m = b[i] - a[i] * cp[i - 1];
    cp[i] = c[i] / m;
    dp[i] = (rhs[i] - a[i] * dp[i - 1]) / m;
  }
  rhs[n - 1] = dp[n - 1];
  for (int i = n - 2; i >= 0; --i) rhs[i] = dp[i] - cp[i] * rhs[i + 1];
}

struct ChunkInv {
  ld i00 = 0, iLL = 0, i0L = 0;  // (K^{-1})_{00}, _{k-1,k-1}, _{0,k-1}
};

// Factors of the Toeplitz chunk with k real points (k <= CH-1); slots >= k zero.
static ChunkInv chunk_factors(int CH, int k, ld D, ld E, double *out) {
  ChunkInv inv;
  for (int j = 0; j < 5 * CH; ++j) out[j] = 0.0;
  if (k <= 0) return inv;
  std::vector<ld> piv(k), q(k), e(k), h(k);
  for (int j = 0; j < k; ++j) {
    piv[j] = (j == 0) ? D : D - E * E / piv[j - 1];
    q[j] = 1.0L / piv[j];
    e[j] = -E * q[j];
    h[j] = (j == 0) ? e[j] : e[j] * h[j - 1];
  }
  std::vector<ld> a(k, E), b(k, D), c(k, E), z0(k, 0.0L), zl(k, 0.0L);
  z0[0] = 1.0L;
  zl[k - 1] = 1.0L;
  tri_solve_ld(k, a.data(), b.data(), c.data(), z0.data());
  tri_solve_ld(k, a.data(), b.data(), c.data(), zl.data());
  for (int j = 0; j < k; ++j) {
    out[0 * CH + j] = (double)q[j];
    out[1 * CH + j] = (double)e[j];
    out[2 * CH + j] = (double)h[j];
    out[3 * CH + j] = (double)z0[j];  // symmetric: row 0 == column 0
    out[4 * CH + j] = (double)(z0[j] / q[j]);
  }
  inv.i00 = z0[0];
  inv.iLL = zl[k - 1];
  inv.i0L = zl[0];
  return inv;
}

Tri1DPlan tri1d_plan(int64_t N, int CH, double Dd, double Ed, double f_first,
                     double f_last, bool cn, int64_t steps) {
  Tri1DPlan P;
  P.N = N;
  P.CH = CH;
  P.D = Dd;
  P.E = Ed;
  P.cn = cn;
  P.steps = steps;
  P.f_first = f_first;
  P.f_last = (N > 1) ? f_last : 0.0;
  P.t_last = (int)((N - 1) / CH);
  P.l_last = (int)((N - 1) % CH);
  const int64_t threads_needed = (N + CH - 1) / CH;
  P.nW = (int)((threads_needed + 31) / 32);
  P.T = 32 * P.nW;
  P.J = (P.nW + 31) / 32;
  if (P.J == 3) P.J = 4;
  if (P.J > 4) pint_throw(PINT_EUNSUPPORTED, "1-D operator too large for the register-resident solver (N <= 4096*CH)");
  const ld D = Dd, E = Ed;
  const int m = CH - 1;
  const int T = P.T, nW = P.nW, J = P.J;

  // singularity check on the full system's pivots (linalg.py:241-266 analogue)
  {
    ld piv = D, mn = fabsl(D);
    for (int64_t j = 1; j < N; ++j) {
      piv = D - E * E / piv;
      mn = std::min(mn, fabsl(piv));
    }
    P.min_pivot = (double)mn;
    ld scale = std::max(fabsl(D), fabsl(E));
    if (scale == 0.0L || mn < 1e-14L * scale)
      pint_throw(PINT_ESINGULAR, "implicit step is singular (pivot " + std::to_string((double)mn) + ")", (double)mn);
  }

  P.tb = (int)std::min<int64_t>((N + 1) / CH, T);
  int ktail = (int)std::max<int64_t>(0, std::min<int64_t>(N - (int64_t)P.tb * CH, m));
  P.fac_reg.assign(5 * CH, 0.0);
  P.fac_tail.assign(5 * CH, 0.0);
  ChunkInv ireg = chunk_factors(CH, m, D, E, P.fac_reg.data());
  ChunkInv itail = chunk_factors(CH, ktail, D, E, P.fac_tail.data());
  // forcing expressed in the pivot-scaled state (backward Euler): t = q x
  {
    const double *f0 = (0 < P.tb) ? P.fac_reg.data() : P.fac_tail.data();
    P.fq_first = f0[0] * P.f_first;
    const double *fl = (P.t_last < P.tb) ? P.fac_reg.data() : P.fac_tail.data();
    P.fq_last = (P.l_last == CH - 1) ? P.f_last : fl[P.l_last] * P.f_last;
  }

  auto kclass = [&](int t) -> int { return t < P.tb ? m : (t == P.tb ? ktail : 0); };
  auto inv_of = [&](int t) -> ChunkInv {
    int k = kclass(t);
    if (t >= T || k == 0) return ChunkInv{};
    return k == m ? ireg : itail;
  };
  auto real = [&](int t) -> bool { return t >= 0 && t < T && (int64_t)t * CH + CH - 1 <= N - 1; };

  // level-1 reduced matrix R (T x T): diag Rd, coupling Ro[t] between t and t+1
  std::vector<ld> Rd(T), Ro(T + 1, 0.0L);
  for (int t = 0; t < T; ++t) {
    if (!real(t)) {
      Rd[t] = 1.0L;
      continue;
    }
    ChunkInv a = inv_of(t), b = inv_of(t + 1);
    Rd[t] = D + E * (-E * a.iLL) + E * (-E * b.i00);
    if (real(t + 1)) Ro[t] = -E * E * ireg.i0L;
  }
  auto RoAt = [&](int t) -> ld { return (t < 0 || t >= T) ? 0.0L : Ro[t]; };

  const int NF = tri1d_nfields(J);
  P.table.assign((size_t)NF * T, 0.0);
  auto TBL = [&](int f, int t) -> double & { return P.table[(size_t)f * T + t]; };

  // level 1 per warp
  std::vector<std::vector<ld>> w1(nW, std::vector<ld>(32, 0.0L)), v1(nW, std::vector<ld>(32, 0.0L));
  for (int W = 0; W < nW; ++W) {
    const int t0 = 32 * W;
    ld a[31], b[31], c[31];
    for (int l = 0; l < 31; ++l) {
      int t = t0 + l;
      a[l] = (l >= 1) ? RoAt(t - 1) : 0.0L;
      b[l] = Rd[t];
      c[l] = (l <= 29) ? RoAt(t) : 0.0L;
    }
    // PCR multipliers (data independent)
    ld pa[31], pb[31], pc[31];
    for (int l = 0; l < 31; ++l) { pa[l] = a[l]; pb[l] = b[l]; pc[l] = c[l]; }
    for (int r = 0; r < 5; ++r) {
      const int d = 1 << r;
      ld na[31], nb[31], nc[31];
      for (int l = 0; l < 31; ++l) {
        ld k1 = (l - d >= 0) ? pa[l] / pb[l - d] : 0.0L;
        ld k2 = (l + d <= 30) ? pc[l] / pb[l + d] : 0.0L;
        na[l] = (l - d >= 0) ? -k1 * pa[l - d] : 0.0L;
        nc[l] = (l + d <= 30) ? -k2 * pc[l + d] : 0.0L;
        nb[l] = pb[l] - ((l - d >= 0) ? k1 * pc[l - d] : 0.0L) - ((l + d <= 30) ? k2 * pa[l + d] : 0.0L);
        TBL(TF_PCR_A + r, t0 + l) = (double)k1;
        TBL(TF_PCR_G + r, t0 + l) = (double)k2;
      }
      for (int l = 0; l < 31; ++l) { pa[l] = na[l]; pb[l] = nb[l]; pc[l] = nc[l]; }
    }
    for (int l = 0; l < 31; ++l) TBL(TF_PCR_INV, t0 + l) = (double)(1.0L / pb[l]);
    TBL(TF_PCR_INV, t0 + 31) = 1.0;
    // spikes: R_CC^{-1} e_0 and e_30
    ld z0[31], z30[31];
    for (int l = 0; l < 31; ++l) { z0[l] = 0; z30[l] = 0; }
    z0[0] = 1;
    z30[30] = 1;
    ld sa[31], sc[31];
    for (int l = 0; l < 31; ++l) { sa[l] = a[l]; sc[l] = c[l]; }
    tri_solve_ld(31, sa, b, sc, z0);
    tri_solve_ld(31, sa, b, sc, z30);
    ld cl = RoAt(t0 - 1), cr = RoAt(t0 + 30);
    for (int l = 0; l < 31; ++l) {
      w1[W][l] = -cl * z0[l];
      v1[W][l] = -cr * z30[l];
      TBL(TF_W1, t0 + l) = (double)w1[W][l];
      TBL(TF_V1, t0 + l) = (double)v1[W][l];
    }
    TBL(TF_CP, t0 + 31) = (double)RoAt(t0 + 30);
    for (int l = 0; l < 32; ++l) TBL(TF_MASK, t0 + l) = real(t0 + l) ? 1.0 : 0.0;
  }

  // level 2: R2 (nW x nW) and its inverse
  std::vector<ld> r2a(nW, 0.0L), r2b(nW), r2c(nW, 0.0L);
  for (int W = 0; W < nW; ++W) {
    int t31 = 32 * W + 31;
    r2b[W] = Rd[t31] + RoAt(t31 - 1) * v1[W][30] + ((W + 1 < nW) ? RoAt(t31) * w1[W + 1][0] : 0.0L);
    r2a[W] = (W > 0) ? RoAt(t31 - 1) * w1[W][30] : 0.0L;
    r2c[W] = (W + 1 < nW) ? RoAt(t31) * v1[W + 1][0] : 0.0L;
  }
  std::vector<ld> R2inv((size_t)nW * nW);
  for (int col = 0; col < nW; ++col) {
    std::vector<ld> z(nW, 0.0L);
    z[col] = 1.0L;
    tri_solve_ld(nW, r2a.data(), r2b.data(), r2c.data(), z.data());
    for (int row = 0; row < nW; ++row) R2inv[(size_t)row * nW + col] = z[row];
  }
  for (int t = 0; t < T; ++t) {
    const int W = t / 32, lane = t % 32;
    for (int j = 0; j < J; ++j) {
      const int V = lane + 32 * j;
      double prevrow = 0.0, currow = 0.0, cz = 0.0, cq = 0.0;
      if (V < nW) {
        if (W >= 1) prevrow = (double)R2inv[(size_t)(W - 1) * nW + V];
        currow = (double)R2inv[(size_t)W * nW + V];
        const int t31 = 32 * V + 31;
        cz = real(t31) ? (double)E : 0.0;
        cq = (double)RoAt(t31);
      }
      TBL(TF_R2 + j, t) = prevrow;
      TBL(TF_R2 + J + j, t) = currow;
      TBL(TF_R2 + 2 * J + j, t) = cz;
      TBL(TF_R2 + 3 * J + j, t) = cq;
    }
  }
  return P;
}

// ============================================================ device side

template <int CH>
struct Tri1DParams {
  ChunkFactors<CH> reg, tail;
  const double *table;  // [NF][T]
  int64_t N;
  int64_t steps;
  double E;
  double f_first, f_last;
  int T, nW, tb;
  int t_last, l_last;
  int has_forcing;
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
// mbarrier of each buffer completes one phase per use).
template <int NV>
__device__ __forceinline__ uint32_t gather_exchange(const StepCtx &c, uint32_t sc, double v0, double v1, double v2,
                                                    double v3) {
  const uint32_t par = sc & 1u;
  const uint32_t stride = (uint32_t)(c.nW + 1);
  const uint32_t gb = c.gbuf + par * 4u * stride * 8u;
  const uint32_t bar = c.mbar + par * 8u;
  if (c.lane < c.CL) {
    const uint32_t rgb = mapa(gb, (uint32_t)c.lane);
    const uint32_t rbar = mapa(bar, (uint32_t)c.lane);
    const uint32_t o = (uint32_t)c.Wg * 8u;
    st_async_f64(rgb + o, v0, rbar);
    st_async_f64(rgb + stride * 8u + o, v1, rbar);
    st_async_f64(rgb + 2u * stride * 8u + o, v2, rbar);
    if (NV == 4) st_async_f64(rgb + 3u * stride * 8u + o, v3, rbar);
  }
  if (threadIdx.x == 0) mbar_arrive_expect_tx(bar, (uint32_t)c.nW * NV * 8u);
  mbar_wait_parity(bar, (sc >> 1) & 1u);
  return gb;
}

#define TAB(f) lds_free(tab + (uint32_t)(f) * 8u)

#ifdef PINT_PHASE_TIMING
// debug build only (scripts/phase_timing.py): clock64 stamps of one step per warp
__device__ long long *g_phase_buf;
__device__ int g_phase_step;
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
template <int CH, int J, bool CN, bool GENERAL, bool IN_RAW, bool OUT_RAW, bool WITH_EXTRA>
__device__ __forceinline__ void tri_step(double (&x)[CH], const Tri1DParams<CH> &P, const StepCtx &c,
                                         uint32_t sc, double extra_in, double *extra_out) {
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
  double y0;
  if (CN) {
    if (regular) y0 = chunk_forward_raw<CH>(x, P.reg, z);
    else y0 = chunk_forward_raw<CH>(x, P.tail, z);
  } else {
    if (regular) y0 = chunk_forward_scaled<CH>(x, P.reg, z);
    else y0 = chunk_forward_scaled<CH>(x, P.tail, z);
  }
  PHASE(1)
  const double ylast = x[CH - 2];
  const double dsep = x[CH - 1];
  double y0n = shfl_down_d(y0, 1);
  if (c.lane == 31) y0n = 0.0;
  double b = TAB(TF_MASK) * (dsep - P.E * (ylast + y0n));
#pragma unroll
  for (int r = 0; r < 5; ++r) {
    const int d = 1 << r;
    const double bm = shfl_up_d(b, d);
    const double bp = shfl_down_d(b, d);
    b = fma(-TAB(TF_PCR_G + r), bp, fma(-TAB(TF_PCR_A + r), bm, b));
  }
  PHASE(2)
  const double y1 = b * TAB(TF_PCR_INV);
  const double y1_30 = shfl_d(y1, 30);
  const double pw = fma(-TAB(TF_CP), y1_30, b);
  const double gP = shfl_d(pw, 31);
  const double gQ = shfl_d(y1, 0);
  const double gZ = shfl_d(y0, 0);
  PHASE(3)
  const uint32_t gb = opaque(gather_exchange<WITH_EXTRA ? 4 : 3>(c, sc, gP, gQ, gZ, extra_in));
  PHASE(4)
  const uint32_t stride8 = (uint32_t)(c.nW + 1) * 8u;
  double sl = 0.0, sr = 0.0, ex = 0.0;
#pragma unroll
  for (int j = 0; j < J; ++j) {
    const int V = c.lane + 32 * j;
    double B = 0.0;
    if (V < c.nW) {
      const uint32_t o = (uint32_t)V * 8u;
      B = fma(-TAB(TF_R2 + 3 * J + j), lds_free(gb + stride8 + o + 8u),
              fma(-TAB(TF_R2 + 2 * J + j), lds_free(gb + 2u * stride8 + o + 8u), lds_free(gb + o)));
      if (WITH_EXTRA) ex = fmax(ex, lds_free(gb + 3u * stride8 + o));
    }
    sl = fma(TAB(TF_R2 + j), B, sl);
    sr = fma(TAB(TF_R2 + J + j), B, sr);
  }
  // split butterfly: the lower half-warp reduces sl, the upper half sr
  {
    const bool lo = c.lane < 16;
    double keep = lo ? sl : sr;
    keep += __shfl_xor_sync(FULLMASK, lo ? sr : sl, 16);
#pragma unroll
    for (int o = 8; o >= 1; o >>= 1) keep += __shfl_xor_sync(FULLMASK, keep, o);
    sl = __shfl_sync(FULLMASK, keep, 0);
    sr = __shfl_sync(FULLMASK, keep, 16);
  }
  if (WITH_EXTRA) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) ex = fmax(ex, __shfl_xor_sync(FULLMASK, ex, o));
  }
  if (WITH_EXTRA) *extra_out = ex;
  double s = fma(TAB(TF_V1), sr, fma(TAB(TF_W1), sl, y1));
  if (c.lane == 31) s = sr;
  double s_left = shfl_up_d(s, 1);
  if (c.lane == 0) s_left = sl;
  PHASE(5)
  x[CH - 1] = s;
  if (CN) {
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
  const int NF = 15 + 4 * J;  // odd: the per-thread rows are bank-conflict free
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
template <int CH, int J, bool CN, bool GENERAL>
__device__ __forceinline__ void run_steps(double (&x)[CH], const Tri1DParams<CH> &P, const StepCtx &c,
                                          uint32_t &sc, int64_t S, double extra_in, double *extra_out) {
  if (S == 1) {
    if (extra_out) tri_step<CH, J, CN, GENERAL, true, true, true>(x, P, c, sc, extra_in, extra_out);
    else tri_step<CH, J, CN, GENERAL, true, true, false>(x, P, c, sc, 0.0, nullptr);
    ++sc;
    return;
  }
  if (extra_out) tri_step<CH, J, CN, GENERAL, true, false, true>(x, P, c, sc, extra_in, extra_out);
  else tri_step<CH, J, CN, GENERAL, true, false, false>(x, P, c, sc, 0.0, nullptr);
  ++sc;
  for (int64_t s = 1; s < S - 1; ++s, ++sc) tri_step<CH, J, CN, GENERAL, false, false, false>(x, P, c, sc, 0.0, nullptr);
  tri_step<CH, J, CN, GENERAL, false, true, false>(x, P, c, sc, 0.0, nullptr);
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

template <int CH, int J, bool CN, bool GENERAL, int MINB>
__global__ void __launch_bounds__(256, MINB)
tri1d_batch_kernel(const __grid_constant__ Tri1DParams<CH> P, const double *__restrict__ in,
                   double *__restrict__ out, int64_t stride) {
  extern __shared__ double smem[];
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int64_t slice = blockIdx.x / (P.T / blockDim.x);
  StepCtx c = setup_ctx<CH, J>(P, smem, rank);
  double x[CH];
  load_chunk<CH>(x, in + slice * stride, P.N, c.t);
  uint32_t sc = 0;
  run_steps<CH, J, CN, GENERAL>(x, P, c, sc, P.steps, 0.0, nullptr);
  store_chunk<CH>(x, out + slice * stride, P.N, c.t);
  cluster.sync();
}

// coarse_init: lam[i] = G(lam[i-1]), i = 1..p (parareal.py:54-63)
template <int CH, int J, bool CN, bool GENERAL>
__global__ void __launch_bounds__(256, 1)
tri1d_init_kernel(const __grid_constant__ Tri1DParams<CH> P, double *lam, double *gcache, int64_t p) {
  extern __shared__ double smem[];
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  StepCtx c = setup_ctx<CH, J>(P, smem, rank);
  double x[CH];
  load_chunk<CH>(x, lam, P.N, c.t);
  uint32_t sc = 0;
  for (int64_t i = 1; i <= p; ++i) {
    run_steps<CH, J, CN, GENERAL>(x, P, c, sc, P.steps, 0.0, nullptr);
    store_chunk<CH>(x, lam + i * P.N, P.N, c.t);
    if (gcache) store_chunk<CH>(x, gcache + i * P.N, P.N, c.t);
  }
  cluster.sync();
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v = fmax(v, __shfl_xor_sync(FULLMASK, v, o));
  return v;
}

// One synchronous sweep with the coarse chain fused with the correction
// (parareal.py:119-127): the running iterate next[i-1] never leaves the SMs.
template <int CH, int J, bool CN, bool GENERAL>
__global__ void __launch_bounds__(256, 1)
tri1d_sweep_kernel(const __grid_constant__ Tri1DParams<CH> P, const double *__restrict__ prev,
                   double *__restrict__ next, const double *__restrict__ fv, double *__restrict__ gcache,
                   int64_t k, int64_t p, double *deltas, int32_t *nonfinite, int chain_in) {
  extern __shared__ double smem[];
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  StepCtx c = setup_ctx<CH, J>(P, smem, rank);
  const int64_t N = P.N;
  double x[CH];
  // chain_in: next[k-1] / deltas[k-1] already hold this sweep's value of slice
  // k-1 (received from the previous GPU of the chain); else slice k-1 is the
  // frozen prefix (next[k-1] = prev[k-1], delta 0).
  const double delta_in = chain_in ? deltas[k - 1] : 0.0;
  if (chain_in) {
    load_chunk<CH>(x, next + (k - 1) * N, N, c.t);
  } else {
    load_chunk<CH>(x, prev + (k - 1) * N, N, c.t);
    store_chunk<CH>(x, next + (k - 1) * N, N, c.t);
  }
  __syncthreads();
  if (!chain_in && rank == 0 && threadIdx.x == 0) deltas[k - 1] = 0.0;
  uint32_t sc = 0;
  double dpart = 0.0;  // warp-uniform partial max of the previous slice
  bool bad = false;
  const int64_t base = (int64_t)c.t * CH;
  // Per-thread staging rows in shared memory, [F(old) | G(old) | prev] x CH
  // doubles + 16 B pad (stride 784 B: 16-byte accesses of 8 consecutive lanes
  // hit distinct banks). The warp fills them with coalesced cp.async while
  // the coarse step runs (lane l copies 16 B of the warp's contiguous
  // 32*CH-point segment into whichever row owns it), and writes the new
  // iterate and G(new) back the same way after the correction.
  const uint32_t RS = (uint32_t)(3 * CH + 2) * 8u;  // row stride in bytes
  const uint32_t row = smem_u32(smem + (15 + 4 * J) * c.TB + 8 * (c.nW + 1) + 2) + (uint32_t)threadIdx.x * RS;
  const uint32_t wrow0 = row - (uint32_t)c.lane * RS;  // lane 0's row
  const int64_t wbase = (int64_t)(c.t - c.lane) * CH;  // warp segment start (points)
  const bool even = (N & 1) == 0;
  double nanacc = 0.0;
  for (int64_t i = k; i <= p; ++i) {
    {
      const double *srcs[3] = {fv + i * N + wbase, gcache + i * N + wbase, prev + i * N + wbase};
      if (even) {
#pragma unroll
        for (int kk = 0; kk < CH / 2; ++kk) {
          const int e = kk * 64 + 2 * c.lane;
          const uint32_t d = wrow0 + (uint32_t)(e / CH) * RS + (uint32_t)(e % CH) * 8u;
          if (wbase + e < N) {
#pragma unroll
            for (int a = 0; a < 3; ++a) cp_async16(d + (uint32_t)(a * CH) * 8u, srcs[a] + e);
          }
        }
      } else {
#pragma unroll
        for (int kk = 0; kk < CH; ++kk) {
          const int e = kk * 32 + c.lane;
          const uint32_t d = wrow0 + (uint32_t)(e / CH) * RS + (uint32_t)(e % CH) * 8u;
          if (wbase + e < N) {
#pragma unroll
            for (int a = 0; a < 3; ++a) cp_async8(d + (uint32_t)(a * CH) * 8u, srcs[a] + e);
          }
        }
      }
      cp_async_commit();
    }
    double dprev = 0.0;
    run_steps<CH, J, CN, GENERAL>(x, P, c, sc, P.steps, dpart, &dprev);
    if (i > k && rank == 0 && threadIdx.x == 0) deltas[i - 1] = dprev;
    const bool fonly = (i == k) ? (delta_in == 0.0) : (dprev == 0.0);
    cp_async_wait_all();
    __syncwarp();
    const uint32_t r = opaque(row);
    double dm = 0.0;
    double gprev = 0.0, vprev = 0.0;
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      double v = 0.0;
      const double g = x[j];
      if (base + j < N) {
        const double fj = lds_free(r + (uint32_t)j * 8u);
        v = fonly ? fj : (g + fj) - lds_free(r + (uint32_t)(CH + j) * 8u);
        dm = fmax(dm, fabs(v - lds_free(r + (uint32_t)(2 * CH + j) * 8u)));
        nanacc += v - v;  // NaN iff v is not finite
      }
      x[j] = v;
      if (j & 1) {  // stage (new, G(new)) pairs into the F / G(old) slots of the own row
        asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(r + (uint32_t)(j - 1) * 8u), "d"(vprev), "d"(v)
                     : "memory");
        asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(r + (uint32_t)(CH + j - 1) * 8u), "d"(gprev),
                     "d"(g) : "memory");
      } else {
        vprev = v;
        gprev = g;
      }
    }
    __syncwarp();
    {
      double *dsts[2] = {next + i * N + wbase, gcache + i * N + wbase};
      if (even) {
#pragma unroll
        for (int kk = 0; kk < CH / 2; ++kk) {
          const int e = kk * 64 + 2 * c.lane;
          const uint32_t src = wrow0 + (uint32_t)(e / CH) * RS + (uint32_t)(e % CH) * 8u;
          if (wbase + e < N) {
#pragma unroll
            for (int a = 0; a < 2; ++a) {
              double2 v2;
              asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v2.x), "=d"(v2.y) : "r"(src + (uint32_t)(a * CH) * 8u));
              *reinterpret_cast<double2 *>(dsts[a] + e) = v2;
            }
          }
        }
      } else {
#pragma unroll
        for (int kk = 0; kk < CH; ++kk) {
          const int e = kk * 32 + c.lane;
          const uint32_t src = wrow0 + (uint32_t)(e / CH) * RS + (uint32_t)(e % CH) * 8u;
          if (wbase + e < N) {
#pragma unroll
            for (int a = 0; a < 2; ++a) dsts[a][e] = lds(src + (uint32_t)(a * CH) * 8u);
          }
        }
      }
    }
    __syncwarp();  // the rows are refilled by the next slice's cp.async
    dpart = warp_max(dm);
  }
  if (nanacc != nanacc) bad = true;
  // final reduction for slice p through one more gather round
  {
    const uint32_t gb = gather_exchange<4>(c, sc, 0.0, 0.0, 0.0, dpart);
    const uint32_t stride8 = (uint32_t)(c.nW + 1) * 8u;
    double ex = 0.0;
    for (int V = c.lane; V < c.nW; V += 32) ex = fmax(ex, lds(gb + 3u * stride8 + (uint32_t)V * 8u));
    ex = warp_max(ex);
    if (rank == 0 && threadIdx.x == 0) deltas[p] = ex;
  }
  if (bad) atomicExch(nonfinite, 1);
  cluster.sync();
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
  P.table = op->d_table;
  P.N = pl.N;
  P.steps = pl.steps;
  P.E = pl.E;
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
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  PINT_CUDA(cudaLaunchKernelEx(&cfg, kern, args...));
}

static size_t smem_bytes(const Tri1DPlan &pl, int TB) {
  return sizeof(double) * ((size_t)tri1d_nfields(pl.J) * TB + 8 * (size_t)(pl.nW + 1)) + 16;
}

enum class TriKind { Batch, Init, Sweep, WaveQuery };

// TriKind::WaveQuery result: clusters of the batch kernel that can be resident
// at once (cudaOccupancyMaxActiveClusters), i.e. slices per wave
static thread_local int g_wave_clusters = 0;

template <int CH, int J, bool CN, bool GENERAL>
static void run_kernel(TriKind kind, const pint_op *op, int grid_slices, int cl, cudaStream_t s,
                       const double *in, double *out, int64_t stride, double *lam, double *gcache,
                       int64_t p, const double *prev, double *next, const double *fv, int64_t k,
                       double *deltas, int32_t *nonfinite, int chain) {
  const Tri1DPlan &pl = op->plan;
  Tri1DParams<CH> P = make_params<CH>(op);
  const int TB = pl.T / cl;
  const size_t sm = smem_bytes(pl, TB);
  switch (kind) {
    case TriKind::Batch:
      if (op->batch_minb == 1)
        launch_cluster(tri1d_batch_kernel<CH, J, CN, GENERAL, 1>, grid_slices * cl, TB, cl, sm, s, P, in, out, stride);
      else
        launch_cluster(tri1d_batch_kernel<CH, J, CN, GENERAL, 2>, grid_slices * cl, TB, cl, sm, s, P, in, out, stride);
      break;
    case TriKind::Init:
      launch_cluster(tri1d_init_kernel<CH, J, CN, GENERAL>, cl, TB, cl, sm, s, P, lam, gcache, p);
      break;
    case TriKind::WaveQuery: {
      auto kern = op->batch_minb == 1 ? tri1d_batch_kernel<CH, J, CN, GENERAL, 1>
                                      : tri1d_batch_kernel<CH, J, CN, GENERAL, 2>;
      PINT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      if (cl > 8) PINT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      cudaLaunchConfig_t cfg;
      memset(&cfg, 0, sizeof(cfg));
      cfg.gridDim = dim3(cl * 1024, 1, 1);
      cfg.blockDim = dim3(TB, 1, 1);
      cfg.dynamicSmemBytes = sm;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = cl;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) {
        cudaGetLastError();
        n = 0;
      }
      g_wave_clusters = n;
      break;
    }
    case TriKind::Sweep:
      launch_cluster(tri1d_sweep_kernel<CH, J, CN, GENERAL>, cl, TB, cl,
                     sm + sizeof(double) * (size_t)TB * (3 * CH + 2), s, P, prev, next, fv, gcache, k, p,
                     deltas, nonfinite, chain);
      break;
  }
}

template <int CH, int J, bool CN>
static void run_kernel_t(TriKind kind, const pint_op *op, int grid_slices, int cl, cudaStream_t s,
                         const double *in, double *out, int64_t stride, double *lam, double *gcache,
                         int64_t p, const double *prev, double *next, const double *fv, int64_t k,
                         double *deltas, int32_t *nonfinite, int chain) {
  // GENERAL: a partially filled (tail) thread or boundary forcing; the fast path has neither
  if (op->plan.tb < op->plan.T || op->plan.f_first != 0.0 || op->plan.f_last != 0.0)
    run_kernel<CH, J, CN, true>(kind, op, grid_slices, cl, s, in, out, stride, lam, gcache, p, prev, next, fv, k,
                                deltas, nonfinite, chain);
  else
    run_kernel<CH, J, CN, false>(kind, op, grid_slices, cl, s, in, out, stride, lam, gcache, p, prev, next, fv, k,
                                 deltas, nonfinite, chain);
}

template <int CH, bool CN>
static void run_kernel_j(TriKind kind, const pint_op *op, int grid_slices, int cl, cudaStream_t s,
                         const double *in, double *out, int64_t stride, double *lam, double *gcache,
                         int64_t p, const double *prev, double *next, const double *fv, int64_t k,
                         double *deltas, int32_t *nonfinite, int chain) {
  switch (op->plan.J) {
    case 1:
      run_kernel_t<CH, 1, CN>(kind, op, grid_slices, cl, s, in, out, stride, lam, gcache, p, prev, next, fv, k,
                            deltas, nonfinite, chain);
      break;
    case 2:
      run_kernel_t<CH, 2, CN>(kind, op, grid_slices, cl, s, in, out, stride, lam, gcache, p, prev, next, fv, k,
                            deltas, nonfinite, chain);
      break;
    default:
      run_kernel_t<CH, 4, CN>(kind, op, grid_slices, cl, s, in, out, stride, lam, gcache, p, prev, next, fv, k,
                            deltas, nonfinite, chain);
      break;
  }
}

static void run_any(TriKind kind, const pint_op *op, int grid_slices, int cl, cudaStream_t s,
                    const double *in, double *out, int64_t stride, double *lam, double *gcache, int64_t p,
                    const double *prev, double *next, const double *fv, int64_t k, double *deltas,
                    int32_t *nonfinite, int chain = 0) {
  if (op->plan.cn) run_kernel_j<16, true>(kind, op, grid_slices, cl, s, in, out, stride, lam, gcache, p, prev, next, fv, k, deltas, nonfinite, chain);
  else if (op->plan.CH == 16) run_kernel_j<16, false>(kind, op, grid_slices, cl, s, in, out, stride, lam, gcache, p, prev, next, fv, k, deltas, nonfinite, chain);
  else run_kernel_j<32, false>(kind, op, grid_slices, cl, s, in, out, stride, lam, gcache, p, prev, next, fv, k, deltas, nonfinite, chain);
}

void tri1d_setup(pint_op *op) {
  const pint_op_desc &d = op->desc;
  const int64_t N = d.shape[0];
  const bool cn = d.rule == PINT_RULE_TRAPEZOIDAL;
  // backward Euler keeps 32 points per thread in registers; the trapezoidal
  // rule also keeps the previous state (x+ = 2 K^{-1}(x + dt/2 c) - x), so 16
  // (layout_ch = 16 is also accepted for backward Euler, so that a coarse
  //  operator can share the register layout of a trapezoidal fine operator)
  int CH = cn ? 16 : 32;
  if (d.layout_ch) {
    if (d.layout_ch == 16 || (d.layout_ch == 32 && !cn)) CH = d.layout_ch;
    else pint_throw(PINT_EARG, "layout_ch must be 32 or 16 (backward Euler) or 16 (trapezoidal)");
  }
  if (d.dtype != PINT_F64) pint_throw(PINT_EUNSUPPORTED, "1-D implicit propagators compute in float64");
  // coefficients formed like the reference's dense matrices:
  // eye - dt * a_mat (BE), half = 0.5 * dt * a_mat (trapezoidal)
  const double dt = d.span / (double)d.steps;
  const double th = cn ? 0.5 * dt : dt;
  const double D = 1.0 - th * d.a_diag;
  const double E = 0.0 - th * d.a_off;
  const double cf = cn ? 0.5 * (dt * d.c_first) : dt * d.c_first;
  const double cl = cn ? 0.5 * (dt * d.c_last) : dt * d.c_last;
  op->dt = dt;
  // kernels count steps in a uint32 whose bit 31 must stay clear (tri_step)
  if (d.steps >= (int64_t)1 << 30) pint_throw(PINT_EARG, "too many steps per application (limit 2^30)");
  op->plan = tri1d_plan(N, CH, D, E, cf, cl, cn, d.steps);
  const Tri1DPlan &pl = op->plan;
  PINT_CUDA(cudaMalloc(&op->d_table, pl.table.size() * sizeof(double)));
  PINT_CUDA(cudaMemcpy(op->d_table, pl.table.data(), pl.table.size() * sizeof(double), cudaMemcpyHostToDevice));
  // CTA split of the T threads of a slice (does not change the arithmetic)
  op->batch_cluster = std::max(1, pl.T / 256);
  op->sweep_cluster = std::min(16, std::max(1, pl.T / 128));
  if (const char *mb = getenv("PINT_TRI_MINB")) op->batch_minb = atoi(mb) == 1 ? 1 : 2;
  if (const char *bc = getenv("PINT_TRI_BATCH_CL")) {
    const int v = atoi(bc);
    if (v >= 1 && v <= 16 && pl.T % v == 0 && (pl.T / v) % 32 == 0 && pl.T / v <= 256) op->batch_cluster = v;
  }
  g_wave_clusters = 0;
  run_any(TriKind::WaveQuery, op, 1, op->batch_cluster, nullptr, nullptr, nullptr, 0, nullptr, nullptr, 0, nullptr,
          nullptr, nullptr, 0, nullptr, nullptr);
  op->batch_wave_slices = g_wave_clusters;
}

void tri1d_destroy(pint_op *op) {
  if (op->d_table) cudaFree(op->d_table);
  op->d_table = nullptr;
}

void tri1d_apply_batch(pint_op *op, const double *in, double *out, int64_t nbatch, int64_t stride,
                       cudaStream_t s) {
  if (nbatch <= 0) return;
  const int64_t maxgrid = 0x7fffffff / 16;
  for (int64_t b0 = 0; b0 < nbatch; b0 += maxgrid) {
    int64_t nb = std::min(maxgrid, nbatch - b0);
    run_any(TriKind::Batch, op, (int)nb, op->batch_cluster, s, in + b0 * stride, out + b0 * stride, stride,
            nullptr, nullptr, 0, nullptr, nullptr, nullptr, 0, nullptr, nullptr);
  }
}

void tri1d_coarse_init(pint_op *op, double *lam, int64_t p, double *gcache, cudaStream_t s) {
  if (p * op->plan.steps >= (int64_t)1 << 31) pint_throw(PINT_EARG, "p * steps must stay below 2^31");
  run_any(TriKind::Init, op, 1, op->sweep_cluster, s, nullptr, nullptr, 0, lam, gcache, p, nullptr, nullptr,
          nullptr, 0, nullptr, nullptr);
}

void tri1d_sweep(pint_op *op, const double *prev, double *next, const double *fv, double *gcache, int64_t k,
                 int64_t p, double *deltas, int32_t *nonfinite, cudaStream_t s, int chain) {
  if (p * op->plan.steps >= (int64_t)1 << 31) pint_throw(PINT_EARG, "p * steps must stay below 2^31");
  run_any(TriKind::Sweep, op, 1, op->sweep_cluster, s, nullptr, nullptr, 0, nullptr, gcache, p, prev, next, fv,
          k, deltas, nonfinite, chain);
}

#ifdef PINT_PHASE_TIMING
extern "C" int pint_debug_phase_timing(long long *dev_buf, int step) {
  cudaMemcpyToSymbol(g_phase_buf, &dev_buf, sizeof(dev_buf));
  cudaMemcpyToSymbol(g_phase_step, &step, sizeof(step));
  return (int)cudaGetLastError();
}
#endif

// Host-only plan export (include/pint_abi.h: pint_tri1d_plan_host).
extern "C" int pint_tri1d_plan_host(const pint_op_desc *d, int32_t *dims_out, double *fac_out, double *table_out,
                                    double *scal_out) {
  if (!d || !dims_out) return PINT_EARG;
  try {
    if (d->ndim != 1 || d->rule == PINT_RULE_FORWARD_EULER || d->steps < 1 || !(d->span > 0.0)) return PINT_EARG;
    const bool cn = d->rule == PINT_RULE_TRAPEZOIDAL;
    const int CH = cn ? 16 : 32;
    const double dt = d->span / (double)d->steps;
    const double th = cn ? 0.5 * dt : dt;
    const double D = 1.0 - th * d->a_diag;
    const double E = 0.0 - th * d->a_off;
    const double cf = cn ? 0.5 * (dt * d->c_first) : dt * d->c_first;
    const double cl = cn ? 0.5 * (dt * d->c_last) : dt * d->c_last;
    Tri1DPlan pl = tri1d_plan(d->shape[0], CH, D, E, cf, cl, cn, d->steps);
    const int NF = tri1d_nfields(pl.J);
    dims_out[0] = pl.CH;
    dims_out[1] = pl.T;
    dims_out[2] = pl.nW;
    dims_out[3] = pl.J;
    dims_out[4] = pl.tb;
    dims_out[5] = NF;
    if (fac_out) {
      memcpy(fac_out, pl.fac_reg.data(), sizeof(double) * 5 * CH);
      memcpy(fac_out + 5 * CH, pl.fac_tail.data(), sizeof(double) * 5 * CH);
    }
    if (table_out) memcpy(table_out, pl.table.data(), sizeof(double) * pl.table.size());
    if (scal_out) {
      scal_out[0] = pl.D;
      scal_out[1] = pl.E;
      scal_out[2] = pl.f_first;
      scal_out[3] = pl.f_last;
      scal_out[4] = pl.fq_first;
      scal_out[5] = pl.fq_last;
      scal_out[6] = pl.t_last;
      scal_out[7] = pl.l_last;
    }
    return PINT_OK;
  } catch (const PintError &e) {
    return e.code;
  }
}

// ======================================================= asynchronous runtime
//
// Asynchronous Parareal with real concurrency (reference semantics:
// async_parareal.py:24-84, Algorithm 2): one persistent launch whose
// thread-block clusters repeatedly claim a slice activation from an atomic
// ticket queue (round-robin order, per-slice try-lock), run
//     F(remembered) -> read the freshest published predecessor -> G(fresh)
//     -> new = F-only ? F(rem) : (G(fresh) + F(rem)) - G(rem) -> publish
// and never wait on another cluster: predecessor states are read from a
// ring of R version-stamped buffers with a seqlock check (retry if the
// writer lapped the slot), so no co-residency is required and staleness is
// whatever the hardware schedule produces. G(rem) is the previous
// activation's G(fresh) (cached per slice). Termination (checked by the
// cluster that just published): every slice drained (consumed the newest
// predecessor version) and every last change < eps, or, with eps < 0, exact
// quiescence (every slice's last activation was F-only on the newest
// predecessor version).

struct AsyncArgs {
  double *ring;            // (P+1) x R x N  published versions
  double *remb;            // (P+1) x N      remembered predecessor reading
  double *gremb;           // (P+1) x N      G(remembered)
  double *scratch;         // nclusters x 2 x N (F result, fresh reading)
  long long *ver;          // (P+1) newest published version per slice
  long long *vrem;         // (P+1) version of the remembered reading
  long long *consumed;     // (P+1) predecessor version consumed at the last activation
  int *busy;               // (P+1) try-lock
  int *stable;             // (P+1) last activation was F-only
  long long *counts;       // (P+1) activations per slice
  double *last_delta;      // (P+1)
  unsigned long long *ticket;
  int *stop;               // 1 = converged, 2 = max_events reached
  int *nonfinite;
  long long *events;
  long long *retries;
  int64_t P, N;
  int R;
  double eps;              // < 0: exact quiescence
  int64_t max_events;
  double delay_frac;       // injected delay per activation: U(0, delay_frac) * t_F
  unsigned long long seed;
  long long *trace;        // optional: ASYNC_TRACE_FIELDS int64 per published activation, in publish order
  long long trace_cap;
};

// trace record: slice, fresh predecessor version read, remembered version,
// F-only flag, delta (bits), globaltimer at F start / at publish, cluster
constexpr int ASYNC_TRACE_FIELDS = 8;

__device__ __forceinline__ long long ld_acquire_s64(const long long *p) {
  long long v;
  asm volatile("ld.acquire.gpu.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_s64(long long *p, long long v) {
  asm volatile("st.release.gpu.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// Stop test (async_parareal.py:52-58 / quiescence): every slice drained and
// every last change < eps (eps >= 0), or every slice stable (eps < 0).
__device__ bool async_done(const AsyncArgs &A) {
  for (long long s = 1; s <= A.P; ++s) {
    const long long vp = (s - 1 == 0) ? 0 : ld_acquire_s64(A.ver + s - 1);
    if (*(volatile long long *)(A.consumed + s) != vp) return false;
    if (A.eps >= 0.0 ? !(*(volatile double *)(A.last_delta + s) < A.eps) : !*(volatile int *)(A.stable + s))
      return false;
  }
  return true;
}

template <int CH>
__device__ __forceinline__ void load_chunk_cg(double (&x)[CH], const double *src, int64_t N, int t) {
  const int64_t base = (int64_t)t * CH;
#pragma unroll
  for (int j = 0; j < CH; ++j) x[j] = (base + j < N) ? __ldcg(src + base + j) : 0.0;
}

// broadcast a few int64 control words from rank 0 / thread 0 to every CTA
__device__ __forceinline__ void ctl_broadcast(long long *ctl, int CL, int n) {
  cg::cluster_group cluster = cg::this_cluster();
  for (int r = 0; r < CL; ++r) {
    long long *dst = cluster.map_shared_rank(ctl, r);
    for (int q = 0; q < n; ++q) dst[q] = ctl[q];
  }
}

template <int CH, int J, bool CNF, bool CNG, bool GENERAL>
__global__ void __launch_bounds__(256, 1)
tri1d_async_kernel(const __grid_constant__ Tri1DParams<CH> PF, const __grid_constant__ Tri1DParams<CH> PG,
                   const AsyncArgs A) {
  extern __shared__ double smem[];
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int TB = blockDim.x;
  const int NF = 15 + 4 * J;
  const int nW = PF.nW;
  // layout: [tabF][tabG][gather 8(nW+1)][2 mbarriers][ctl 8 x int64][red 32]
  double *tabF = smem;
  double *tabG = smem + NF * TB;
  double *gbuf = tabG + NF * TB;
  uint64_t *bars = reinterpret_cast<uint64_t *>(gbuf + 8 * (nW + 1));
  long long *ctl = reinterpret_cast<long long *>(bars + 2);
  double *red = reinterpret_cast<double *>(ctl + 8);
  StepCtx cF, cG;
  cF.TB = cG.TB = TB;
  cF.CL = cG.CL = PF.T / TB;
  cF.nW = cG.nW = nW;
  cF.t = cG.t = rank * TB + threadIdx.x;
  cF.lane = cG.lane = threadIdx.x & 31;
  cF.Wg = cG.Wg = cF.t >> 5;
  for (int f = 0; f < NF; ++f) {
    tabF[threadIdx.x * NF + f] = PF.table[(size_t)f * PF.T + cF.t];
    tabG[threadIdx.x * NF + f] = PG.table[(size_t)f * PG.T + cF.t];
  }
  cF.tab = smem_u32(tabF + threadIdx.x * NF);
  cG.tab = smem_u32(tabG + threadIdx.x * NF);
  for (int i = threadIdx.x; i < 8 * (nW + 1); i += TB) gbuf[i] = 0.0;
  cF.gbuf = cG.gbuf = smem_u32(gbuf);
  cF.mbar = cG.mbar = smem_u32(bars);
  if (threadIdx.x == 0) {
    mbar_init(cF.mbar, 1);
    mbar_init(cF.mbar + 8, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  cluster.sync();

  const int64_t N = A.N, P = A.P;
  const int CL = cF.CL;
  const int64_t cid = blockIdx.x / CL;
  double *sF = A.scratch + (size_t)cid * 2 * N;
  double *sFresh = sF + N;
  const int64_t base = (int64_t)cF.t * CH;
  uint32_t sc = 0;
  double x[CH];
  bool bad = false;
  for (;;) {
    // ---- claim an activation (rank 0, thread 0), broadcast to the cluster
    if (rank == 0 && threadIdx.x == 0) {
      long long slice = -1;
      unsigned backoff = 32;
      for (;;) {
        if (*(volatile int *)A.stop) break;
        const unsigned long long tk = atomicAdd(A.ticket, 1ull);
        if (tk >= (unsigned long long)A.max_events * 64ull) {  // livelock guard
          atomicCAS(A.stop, 0, 2);
          break;
        }
        const long long i = 1 + (long long)(tk % (unsigned long long)P);
        if (atomicCAS(A.busy + i, 0, 1) != 0) continue;
        const long long vp = (i - 1 == 0) ? 0 : ld_acquire_s64(A.ver + i - 1);
        if (*(volatile int *)(A.stable + i) && *(volatile long long *)(A.consumed + i) == vp) {
          // nothing new to consume: an activation would reproduce the same
          // value, i.e. a zero change; record it as such without publishing
          *(volatile double *)(A.last_delta + i) = 0.0;
          __threadfence();
          atomicExch(A.busy + i, 0);
          if (async_done(A)) atomicExch(A.stop, 1);
          __nanosleep(backoff);
          backoff = min(backoff * 2, 4096u);
          continue;
        }
        slice = i;
        break;
      }
      ctl[0] = slice;
      ctl_broadcast(ctl, CL, 1);
    }
    cluster.sync();
    const long long i = ctl[0];
    if (i < 0) break;

    // ---- F(remembered)
    const unsigned long long tf0 = globaltimer();
    load_chunk_cg<CH>(x, A.remb + i * N, N, cF.t);
    run_steps<CH, J, CNF, GENERAL>(x, PF, cF, sc, PF.steps, 0.0, nullptr);
    store_chunk<CH>(x, sF, N, cF.t);
    if (A.delay_frac > 0.0 && rank == 0 && threadIdx.x == 0) {
      const unsigned long long tF = globaltimer() - tf0;
      const unsigned long long h = mix64(A.seed ^ ((unsigned long long)i << 32) ^ (unsigned long long)A.counts[i]);
      const double u = (double)(h >> 11) * (1.0 / 9007199254740992.0);
      const unsigned long long until = globaltimer() + (unsigned long long)(u * A.delay_frac * (double)tF);
      while (globaltimer() < until) __nanosleep(1000);
    }

    // ---- freshest predecessor (seqlock read of the ring)
    long long v = 0;
    for (int attempt = 0;; ++attempt) {
      if (rank == 0 && threadIdx.x == 0) {
        ctl[1] = (i - 1 == 0) ? 0 : ld_acquire_s64(A.ver + i - 1);
        ctl_broadcast(ctl + 1, CL, 1);
      }
      cluster.sync();
      v = ctl[1];
      load_chunk_cg<CH>(x, A.ring + ((size_t)(i - 1) * A.R + (size_t)(v % A.R)) * N, N, cF.t);
      __syncthreads();
      if (rank == 0 && threadIdx.x == 0) {
        const long long v2 = (i - 1 == 0) ? 0 : ld_acquire_s64(A.ver + i - 1);
        ctl[2] = (v2 <= v + A.R - 2) ? 1 : 0;
        if (!ctl[2]) atomicAdd((unsigned long long *)A.retries, 1ull);
        ctl_broadcast(ctl + 2, CL, 1);
      }
      cluster.sync();
      if (ctl[2]) break;
    }
    const long long vr = A.vrem[i];
    // bitwise comparison with the remembered reading (array_equal semantics)
    double mism = 0.0;
#pragma unroll
    for (int j = 0; j < CH; ++j)
      if (base + j < N && !(x[j] == __ldcg(A.remb + i * N + base + j))) mism = 1.0;
    mism = warp_max(mism);
    store_chunk<CH>(x, sFresh, N, cF.t);

    // ---- G(fresh), with the mismatch flag reduced over the slice on the way
    double anymism = 0.0;
    run_steps<CH, J, CNG, GENERAL>(x, PG, cG, sc, PG.steps, mism, &anymism);
    const bool fonly = (v == vr) || (anymism == 0.0);

    // ---- correction, delta, publish into the next ring slot
    const long long vi = A.ver[i];
    const double *cur = A.ring + ((size_t)i * A.R + (size_t)(vi % A.R)) * N + base;
    double *dst = A.ring + ((size_t)i * A.R + (size_t)((vi + 1) % A.R)) * N + base;
    double *gw = A.gremb + i * N + base;
    double *rw = A.remb + i * N + base;
    double dm = 0.0;
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      if (base + j < N) {
        const double g = x[j];
        const double f = __ldcg(sF + base + j);
        const double nv = fonly ? f : (g + f) - __ldcg(gw + j);
        dm = fmax(dm, fabs(nv - __ldcg(cur + j)));
        bad |= !isfinite(nv);
        dst[j] = nv;
        gw[j] = g;
        rw[j] = __ldcg(sFresh + base + j);
      }
    }
    dm = warp_max(dm);
    __threadfence();
    if ((threadIdx.x & 31) == 0) cluster.map_shared_rank(red, 0)[cF.Wg] = dm;
    cluster.sync();
    if (rank == 0 && threadIdx.x == 0) {
      double d = 0.0;
      for (int w = 0; w < nW; ++w) d = fmax(d, red[w]);
      A.last_delta[i] = d;
      A.vrem[i] = v;
      A.consumed[i] = v;
      A.stable[i] = fonly ? 1 : 0;
      A.counts[i] += 1;
      const long long ev = (long long)atomicAdd((unsigned long long *)A.events, 1ull) + 1;
      if (A.trace && ev - 1 < A.trace_cap) {
        long long *r = A.trace + (ev - 1) * ASYNC_TRACE_FIELDS;
        r[0] = i;
        r[1] = v;
        r[2] = vr;
        r[3] = fonly ? 1 : 0;
        r[4] = __double_as_longlong(d);
        r[5] = (long long)tf0;
        r[6] = (long long)globaltimer();
        r[7] = cid;
      }
      __threadfence();
      st_release_s64(A.ver + i, vi + 1);
      atomicExch(A.busy + i, 0);
      if (async_done(A)) atomicExch(A.stop, 1);
      else if (ev >= A.max_events) atomicCAS(A.stop, 0, 2);
    }
  }
  if (bad) atomicExch(A.nonfinite, 1);
  cluster.sync();
}

extern "C" int pint_async_run_traced(pint_op *fine, pint_op *coarse, const void *lam0, int64_t p, double epsilon,
                                     int64_t max_events, double delay_frac, uint64_t seed, void *final_out,
                                     int64_t *counts_out, int64_t *info_out, int64_t *trace_out, int64_t trace_cap,
                                     void *stream) {
  if (!fine || !coarse) return PINT_EARG;
  pint_ctx *ctx = fine->ctx;
  try {
    if (fine->desc.ndim != 1 || coarse->desc.ndim != 1 || fine->desc.rule == PINT_RULE_FORWARD_EULER ||
        coarse->desc.rule == PINT_RULE_FORWARD_EULER)
      pint_throw(PINT_EUNSUPPORTED, "the device async runtime supports 1-D implicit fine and coarse operators");
    const Tri1DPlan &pf = fine->plan, &pg = coarse->plan;
    if (pf.N != pg.N || pf.CH != pg.CH || pf.T != pg.T)
      pint_throw(PINT_EUNSUPPORTED, "fine and coarse operators must share the register layout (same rule family)");
    if (p < 1 || !lam0 || !final_out) pint_throw(PINT_EARG, "bad arguments");
    if (trace_cap < 0 || (trace_cap > 0 && !trace_out)) pint_throw(PINT_EARG, "trace buffer missing");
    if ((max_events > 0 ? max_events : 20000) * (pf.steps + pg.steps) >= (int64_t)1 << 31)
      pint_throw(PINT_EARG, "max_events * (fine + coarse steps) must stay below 2^31");
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t N = pf.N;
    const int R = 3;
    const int CL = fine->batch_cluster;
    const int TB = pf.T / CL;
    int dev_sms = ctx->num_sms;
    const int64_t ncl = std::max<int64_t>(1, std::min<int64_t>(p, dev_sms / CL));
    // device workspace
    size_t bytes = 0;
    auto take = [&](size_t n) { size_t o = bytes; bytes += (n + 255) / 256 * 256; return o; };
    const size_t o_ring = take(sizeof(double) * (p + 1) * R * N), o_remb = take(sizeof(double) * (p + 1) * N),
                 o_gremb = take(sizeof(double) * (p + 1) * N), o_scr = take(sizeof(double) * ncl * 2 * N),
                 o_ver = take(8 * (p + 1)), o_vrem = take(8 * (p + 1)), o_cons = take(8 * (p + 1)),
                 o_busy = take(4 * (p + 1)), o_stab = take(4 * (p + 1)), o_cnt = take(8 * (p + 1)),
                 o_ld = take(8 * (p + 1)), o_misc = take(64),
                 o_trace = take(sizeof(long long) * ASYNC_TRACE_FIELDS * (size_t)trace_cap);
    char *w = nullptr;
    PINT_CUDA(cudaMallocAsync((void **)&w, bytes, s));
    PINT_CUDA(cudaMemsetAsync(w + o_ver, 0, o_misc + 64 - o_ver, s));
    AsyncArgs A;
    A.ring = (double *)(w + o_ring);
    A.remb = (double *)(w + o_remb);
    A.gremb = (double *)(w + o_gremb);
    A.scratch = (double *)(w + o_scr);
    A.ver = (long long *)(w + o_ver);
    A.vrem = (long long *)(w + o_vrem);
    A.consumed = (long long *)(w + o_cons);
    A.busy = (int *)(w + o_busy);
    A.stable = (int *)(w + o_stab);
    A.counts = (long long *)(w + o_cnt);
    A.last_delta = (double *)(w + o_ld);
    A.ticket = (unsigned long long *)(w + o_misc);
    A.stop = (int *)(w + o_misc + 8);
    A.nonfinite = (int *)(w + o_misc + 12);
    A.events = (long long *)(w + o_misc + 16);
    A.retries = (long long *)(w + o_misc + 24);
    A.P = p;
    A.N = N;
    A.R = R;
    A.eps = epsilon;
    A.max_events = max_events > 0 ? max_events : 20000;
    A.delay_frac = delay_frac;
    A.seed = seed;
    A.trace = trace_cap > 0 ? (long long *)(w + o_trace) : nullptr;
    A.trace_cap = trace_cap;
    // initial versions: ring[i][0] = lam0[i]; remembered = lam0[i-1] (version 0);
    // G(remembered) = G(lam0[i-1]) = lam0[i] (coarse initial iterate)
    const double *L = (const double *)lam0;
    for (int64_t i = 0; i <= p; ++i)
      PINT_CUDA(cudaMemcpyAsync(A.ring + (size_t)i * R * N, L + i * N, sizeof(double) * N, cudaMemcpyDeviceToDevice, s));
    PINT_CUDA(cudaMemcpyAsync(A.remb + N, L, sizeof(double) * p * N, cudaMemcpyDeviceToDevice, s));
    PINT_CUDA(cudaMemcpyAsync(A.gremb + N, L + N, sizeof(double) * p * N, cudaMemcpyDeviceToDevice, s));
    {
      std::vector<double> inf(p + 1, INFINITY);
      inf[0] = 0.0;
      std::vector<long long> minus1(p + 1, -1);
      PINT_CUDA(cudaMemcpyAsync(A.last_delta, inf.data(), 8 * (p + 1), cudaMemcpyHostToDevice, s));
      PINT_CUDA(cudaMemcpyAsync(A.consumed, minus1.data(), 8 * (p + 1), cudaMemcpyHostToDevice, s));
      PINT_CUDA(cudaStreamSynchronize(s));
    }
    const size_t sm = sizeof(double) * (2 * (size_t)tri1d_nfields(pf.J) * TB + 8 * (size_t)(pf.nW + 1)) + 16 +
                      64 + 32 * 8 * 4;
    const bool general = pf.tb < pf.T || pf.f_first != 0.0 || pf.f_last != 0.0 || pg.f_first != 0.0 ||
                         pg.f_last != 0.0;
#define PINT_ASYNC_LAUNCH(CHV, JV, CNF, CNG, GV)                                                        \
  launch_cluster(tri1d_async_kernel<CHV, JV, CNF, CNG, GV>, (int)(ncl * CL), TB, CL, sm, s,              \
                 make_params<CHV>(fine), make_params<CHV>(coarse), A)
#define PINT_ASYNC_J(CHV, CNF, CNG, GV)                      \
  switch (pf.J) {                                            \
    case 1: PINT_ASYNC_LAUNCH(CHV, 1, CNF, CNG, GV); break;  \
    case 2: PINT_ASYNC_LAUNCH(CHV, 2, CNF, CNG, GV); break;  \
    default: PINT_ASYNC_LAUNCH(CHV, 4, CNF, CNG, GV); break; \
  }
    if (pf.CH == 16) {
      if (pf.cn && pg.cn) {
        if (general) { PINT_ASYNC_J(16, true, true, true) } else { PINT_ASYNC_J(16, true, true, false) }
      } else if (pf.cn) {
        if (general) { PINT_ASYNC_J(16, true, false, true) } else { PINT_ASYNC_J(16, true, false, false) }
      } else if (!pg.cn) {
        if (general) { PINT_ASYNC_J(16, false, false, true) } else { PINT_ASYNC_J(16, false, false, false) }
      } else {
        pint_throw(PINT_EUNSUPPORTED, "backward-Euler fine with trapezoidal coarse is not fused in the device runtime");
      }
    } else {
      if (general) { PINT_ASYNC_J(32, false, false, true) } else { PINT_ASYNC_J(32, false, false, false) }
    }
#undef PINT_ASYNC_J
#undef PINT_ASYNC_LAUNCH
    // gather the newest published version of every slice
    std::vector<long long> ver(p + 1), cnt(p + 1);
    long long misc[4];
    int flags[2];
    PINT_CUDA(cudaMemcpyAsync(ver.data(), A.ver, 8 * (p + 1), cudaMemcpyDeviceToHost, s));
    PINT_CUDA(cudaMemcpyAsync(cnt.data(), A.counts, 8 * (p + 1), cudaMemcpyDeviceToHost, s));
    PINT_CUDA(cudaMemcpyAsync(flags, A.stop, 8, cudaMemcpyDeviceToHost, s));
    PINT_CUDA(cudaMemcpyAsync(misc, A.events, 16, cudaMemcpyDeviceToHost, s));
    PINT_CUDA(cudaStreamSynchronize(s));
    if (trace_cap > 0) {
      const size_t nrec = (size_t)std::min<long long>(misc[0], trace_cap);
      PINT_CUDA(cudaMemcpyAsync(trace_out, A.trace, sizeof(long long) * ASYNC_TRACE_FIELDS * nrec,
                                cudaMemcpyDeviceToHost, s));
    }
    for (int64_t i = 0; i <= p; ++i)
      PINT_CUDA(cudaMemcpyAsync((double *)final_out + i * N, A.ring + ((size_t)i * R + (size_t)(ver[i] % R)) * N,
                                sizeof(double) * N, cudaMemcpyDeviceToDevice, s));
    PINT_CUDA(cudaFreeAsync(w, s));
    PINT_CUDA(cudaStreamSynchronize(s));
    if (counts_out)
      for (int64_t i = 0; i <= p; ++i) counts_out[i] = cnt[i];
    if (info_out) {
      info_out[0] = misc[0];   // events (activations)
      info_out[1] = flags[0];  // 1 converged, 2 max_events
      info_out[2] = flags[1];  // non-finite
      info_out[3] = misc[1];   // seqlock retries
      info_out[4] = ncl;       // concurrent clusters
    }
    return PINT_OK;
  } catch (const PintError &e) {
    ctx->last_error = e.msg;
    ctx->last_value = e.value;
    return e.code;
  }
}

extern "C" int pint_async_run(pint_op *fine, pint_op *coarse, const void *lam0, int64_t p, double epsilon,
                              int64_t max_events, double delay_frac, uint64_t seed, void *final_out,
                              int64_t *counts_out, int64_t *info_out, void *stream) {
  return pint_async_run_traced(fine, coarse, lam0, p, epsilon, max_events, delay_frac, seed, final_out, counts_out,
                               info_out, nullptr, 0, stream);
}
