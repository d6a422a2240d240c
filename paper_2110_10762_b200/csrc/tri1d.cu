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
#include "tri1d_device.cuh"

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
  // Pad with virtual warps (all-zero chunks, masked separators: decoupled
  // unknowns) so that every cluster split is whole warps: the batch kernel
  // splits a slice into nW/8 CTAs of 256 threads, the fused sweep into
  // min(16, nW/4) CTAs (multiples of 32 threads need nW % 16 == 0 above 64).
  if (P.nW > 8) P.nW = (P.nW + 7) / 8 * 8;
  if (P.nW > 64) P.nW = (P.nW + 15) / 16 * 16;
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

  // Constant-coefficient twisted chunk solve (backward Euler, every thread
  // regular, no forcing): K = c (I - lam S)(I - lam S^T) away from the chunk
  // ends, c the larger root of c^2 - D c + E^2 = 0, lam = -E / c. Eliminating
  // with these limit factors from both chunk ends solves Kt = K_c - delta
  // (e_0 e_0^T + e_L e_L^T), delta = D - c, exactly; since K_c x = b is
  // Kt x = b - delta (x_0 e_0 + x_L e_L), the defect acts like a change of the
  // adjacent separator values (sigma' = sigma - lam x_end) and folds into
  // data-independent scalars. In the scaled variables chi_j = x_j / lam^|j-k|
  // both sweeps have position-independent multipliers (mu = lam^2 and 1/c).
  P.ccst = false;
  P.ccst_fac.assign(ccst_nscalars(CH), 0.0);
  if (!cn && m >= 3 && (m & 1) && E != 0.0L && D * D > 4.0L * E * E) {
    // every factor in closed form in lam (the chunk's Green's function is a
    // combination of lam^j and lam^-j); 1 - mu = (c - E)(c + E) / c^2 is formed
    // without cancellation so the factors keep full relative accuracy as
    // lam -> 1 (large dt / h^2)
    const int k = (m - 1) / 2, n = m + 1;  // n = 2k + 2: distance between the two separators
    const ld sd = D >= 0 ? 1.0L : -1.0L;
    const ld disc = sd * sqrtl((D - 2.0L * E) * (D + 2.0L * E));
    const ld c = (D + disc) / 2.0L;
    const ld lam = -E / c;
    const ld om = ((D - 2.0L * E + disc) / 2.0L) * ((D + 2.0L * E + disc) / 2.0L) / (c * c);  // 1 - mu
    const ld mu = lam * lam;
    const ld lk = powl(lam, k);
    // (not used when the step matrix is E-dominated beyond any grid scale,
    //  |E| / (|D| - 2|E|) > 100 N^2, i.e. dt >> the slowest mode's time scale:
    //  the nearly free chunk ends then cost accuracy, measured in
    //  tests/test_host_logic.py; the exact-pivot path serves those)
    const bool stiff_ok = fabsl(E) <= 100.0L * (ld)N * (ld)N * (fabsl(D) - 2.0L * fabsl(E));
    if (fabsl(lk) > 1e-100L && om > 0.0L && stiff_ok) {
      ld geo = 0.0L, t = 1.0L;  // (1 - lam^(2n)) / (1 - mu)
      for (int i = 0; i < n; ++i) {
        geo += t;
        t *= mu;
      }
      const ld ln = powl(lam, n), lk1 = lk * lam;
      double *f = P.ccst_fac.data();
      f[0] = (double)mu;
      f[1] = (double)(1.0L / c);
      f[2] = (double)(1.0L / (c * om));
      f[3] = (double)(lk1 / (-E * geo));                       // al
      f[4] = (double)(-powl(lam, 3 * k + 3) / (-E * geo));     // be
      f[5] = (double)(lk1 / (-E * (1.0L + ln)));               // ga
      f[6] = (double)(om / (1.0L + ln));                       // sAB = 1 - lam (vL_0 + vR_0)
      f[7] = (double)(-ln / geo);                              // sB = -lam vR_0
      f[8] = (double)(-lam);
      f[9] = (double)(lk1 / (1.0L + ln));                      // CmAB
      f[10] = (double)(-lk1 * lam / om);                       // CmN
      for (int i = 0; i < k; ++i) {
        f[11 + i] = (double)(-E * powl(lam, 2 * i - k));
        const ld rho = powl(lam, k - i);
        f[11 + CH / 2 + i] = (double)(1.0L / rho);
        f[11 + 2 * (CH / 2) + i] = (double)rho;
      }
      bool fin = true;
      for (int i = 0; i < ccst_nscalars(CH); ++i) fin = fin && std::isfinite(f[i]);
      P.ccst = fin;
    }
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
  P.hq = (double)(-E * E * ireg.i0L);

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
    // three PCR rounds (distances 1, 2, 4) leave eight independent systems
    // over the lanes {l, l+8, l+16, l+24} (those <= 30); each is closed by its
    // dense inverse: y1_l = C0 b_l + C8 b_{l^8} + C16 b_{l^16} + C24 b_{l^24}
    // (three independent xor shuffles instead of two more dependent rounds).
    // Table slots: rounds 0..2 in TF_PCR_A/G + r; C0, C8 in TF_PCR_A + 3, + 4;
    // C16, C24 in TF_PCR_G + 3, + 4 (lane 31: all zero, its value is the
    // level-2 unknown).
    for (int r = 0; r < 3; ++r) {
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
    for (int g = 0; g < 8; ++g) {
      int mem[4], nq = 0;
      for (int q = 0; q < 4; ++q)
        if (g + 8 * q <= 30) mem[nq++] = g + 8 * q;
      ld ga[4], gb2[4], gc[4], ginv[4][4];
      for (int q = 0; q < nq; ++q) {
        ga[q] = (q > 0) ? pa[mem[q]] : 0.0L;
        gb2[q] = pb[mem[q]];
        gc[q] = (q + 1 < nq) ? pc[mem[q]] : 0.0L;
      }
      for (int col = 0; col < nq; ++col) {
        ld e[4] = {0.0L, 0.0L, 0.0L, 0.0L};
        e[col] = 1.0L;
        tri_solve_ld(nq, ga, gb2, gc, e);
        for (int row = 0; row < nq; ++row) ginv[row][col] = e[row];
      }
      for (int q = 0; q < nq; ++q) {
        const int l = mem[q];
        auto coef = [&](int x) -> double {  // partner l ^ (8 x) = member q ^ x
          const int qp = q ^ x;
          return (qp < nq) ? (double)ginv[q][qp] : 0.0;
        };
        TBL(TF_PCR_A + 3, t0 + l) = coef(0);
        TBL(TF_PCR_A + 4, t0 + l) = coef(1);
        TBL(TF_PCR_G + 3, t0 + l) = coef(2);
        TBL(TF_PCR_G + 4, t0 + l) = coef(3);
      }
    }
    TBL(TF_PCR_INV, t0 + 31) = 0.0;  // (slot unused by the kernels)
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
    TBL(TF_W1, t0 + 31) = 0.0;
    TBL(TF_V1, t0 + 31) = 1.0;
    TBL(TF_CP, t0 + 31) = (double)RoAt(t0 + 30);
    // level-2 right-hand side of warp W - 1: B = gP_{W-1} - h_W, h_W = cq y1_0 + cz y0_0
    // with the coefficients of column W - 1 (lane 31 of the previous warp)
    {
      const int t31p = t0 - 1;
      const double cz = (W >= 1 && real(t31p)) ? (double)E : 0.0;
      const double cq = (W >= 1) ? (double)RoAt(t31p) : 0.0;
      for (int l = 0; l < 32; ++l) {
        TBL(TF_HQ(J), t0 + l) = cq;
        TBL(TF_HZ(J), t0 + l) = cz;
      }
    }
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
  // Level-2 window: R2 is strongly diagonally dominant (its couplings are the
  // chunk Green's function over a whole warp, lam^1024), so its inverse decays
  // geometrically away from the diagonal. When every entry outside the 32
  // columns [c0(W), c0(W) + 32), c0(W) = clamp(W - 16, 0, nW - 32), of rows
  // W - 1 and W is below 2^-64 of the row's largest entry, the dropped terms
  // cannot change an fp64 dot product, and each lane handles one column
  // instead of J.
  P.l2win = false;
  if (nW > 32) {
    bool ok = true;
    for (int W = 0; W < nW && ok; ++W) {
      const int c0 = std::min(std::max(W - 16, 0), nW - 32);
      for (int row = std::max(W - 1, 0); row <= W && ok; ++row) {
        ld mx = 0.0L, out = 0.0L;
        for (int V = 0; V < nW; ++V) {
          const ld a = fabsl(R2inv[(size_t)row * nW + V]);
          mx = std::max(mx, a);
          if (V < c0 || V >= c0 + 32) out = std::max(out, a);
        }
        if (!(out <= mx * 5.4e-20L)) ok = false;
      }
    }
    P.l2win = ok;
    if (const char *e = getenv("PINT_L2WIN")) P.l2win = P.l2win && atoi(e) != 0;  // 0: full rows (A/B switch)
  }
  for (int t = 0; t < T; ++t) {
    const int W = t / 32, lane = t % 32;
    const int c0 = P.l2win ? std::min(std::max(W - 16, 0), nW - 32) : 0;
    for (int j = 0; j < J; ++j) {
      const int V = c0 + lane + 32 * j;
      double prevrow = 0.0, currow = 0.0;
      if (V < nW && !(P.l2win && j > 0)) {
        if (W >= 1) prevrow = (double)R2inv[(size_t)(W - 1) * nW + V];
        currow = (double)R2inv[(size_t)W * nW + V];
      }
      TBL(TF_R2 + j, t) = prevrow;
      TBL(TF_R2 + J + j, t) = currow;
    }
  }
  return P;
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


// One synchronous sweep with the coarse chain fused with the correction
// (parareal.py:119-127): the running iterate next[i-1] never leaves the SMs.
template <int CH, int J, bool CN, bool GENERAL>
__global__ void __launch_bounds__(256, 1)
tri1d_sweep_kernel(const __grid_constant__ Tri1DParams<CH> P, const double *__restrict__ prev,
                   double *__restrict__ next, const double *__restrict__ fv, double *__restrict__ gcache,
                   int64_t k, int64_t p, double *deltas, int32_t *nonfinite, int chain_in, int defer) {
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
  const uint32_t row = smem_u32(smem + TRI1D_NF(J) * c.TB + 8 * (c.nW + 1) + 2) + (uint32_t)threadIdx.x * RS;
  const uint32_t wrow0 = row - (uint32_t)c.lane * RS;  // lane 0's row
  const int64_t wbase = (int64_t)(c.t - c.lane) * CH;  // warp segment start (points)
  // Fast path: when they fit (`defer`), the results (new | G(new)) are staged
  // in rows of their own (2 CH doubles + 16 B pad) and drained to global
  // memory one slice later, inside the next coarse step's cluster exchange
  // (tri_step's shadow hook); otherwise they go through the F / G(old) slots
  // of the input rows and are drained right after the correction.
  const uint32_t OS = (defer & 1) ? (uint32_t)(2 * CH + 2) * 8u : RS;
  const uint32_t orow = (defer & 1) ? smem_u32(smem + TRI1D_NF(J) * c.TB + 8 * (c.nW + 1) + 2 +
                                         (size_t)c.TB * (3 * CH + 2)) + (uint32_t)threadIdx.x * OS
                              : row;
  const uint32_t worow0 = orow - (uint32_t)c.lane * OS;
  auto drain = [&](int64_t islice) {
    double *dsts[2] = {next + islice * N + wbase, gcache + islice * N + wbase};
#pragma unroll
    for (int kk = 0; kk < CH / 2; ++kk) {
      const int e = kk * 64 + 2 * c.lane;
      const uint32_t src = worow0 + (uint32_t)(e / CH) * OS + (uint32_t)(e % CH) * 8u;
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        double2 v2;
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v2.x), "=d"(v2.y) : "r"(src + (uint32_t)(a * CH) * 8u));
        *reinterpret_cast<double2 *>(dsts[a] + e) = v2;
      }
    }
    __syncwarp();  // the rows are rewritten by the next correction
  };
  const bool even = !GENERAL || (N & 1) == 0;  // fast path: N is a multiple of CH
  double nanacc = 0.0;
  // operands of slice i -> the staging rows (coalesced cp.async, lane l copies
  // 16 B of the warp's contiguous segment into whichever row owns it)
  auto prefetch = [&](int64_t i) {
    const double *srcs[3] = {fv + i * N + wbase, gcache + i * N + wbase, prev + i * N + wbase};
    if (even) {
#pragma unroll
      for (int kk = 0; kk < CH / 2; ++kk) {
        const int e = kk * 64 + 2 * c.lane;
        const uint32_t d = wrow0 + (uint32_t)(e / CH) * RS + (uint32_t)(e % CH) * 8u;
        if (!GENERAL || wbase + e < N) {  // fast path: N is a multiple of CH, every point real
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
  };
  // PINT_SWEEP_PREFETCH_SHADOW (launcher): issue the prefetch inside the coarse
  // step's exchange as well (fast path)
  const bool pf_shadow = !GENERAL && (defer & 2);
  for (int64_t i = k; i <= p; ++i) {
    if (!pf_shadow) prefetch(i);
    double dprev = 0.0;
    if (!GENERAL) {
      auto shadow = [&]() {
        if (pf_shadow) prefetch(i);
        if ((defer & 1) && i > k) drain(i - 1);
      };
      run_steps<CH, J, CN, GENERAL, decltype(shadow)>(x, P, c, sc, P.steps, dpart, &dprev, shadow);
    } else {
      run_steps<CH, J, CN, GENERAL>(x, P, c, sc, P.steps, dpart, &dprev);
    }
    if (i > k && rank == 0 && threadIdx.x == 0) deltas[i - 1] = dprev;
    const bool fonly = (i == k) ? (delta_in == 0.0) : (dprev == 0.0);
    cp_async_wait_all();
    __syncwarp();
    const uint32_t r = opaque(row);
    double dm = 0.0;
    if (!GENERAL) {
      // fast path: every point of every thread is real (N a multiple of CH);
      // the F-only choice (warp-uniform) is hoisted out of the point loop.
      // Same per-point expressions as the general loop below.
      const uint32_t ro = opaque(orow);
      if (fonly) {
#pragma unroll
        for (int j = 0; j < CH; j += 2) {
          const double g0 = x[j], g1 = x[j + 1];
          const double v0 = lds_free(r + (uint32_t)j * 8u), v1 = lds_free(r + (uint32_t)(j + 1) * 8u);
          dm = fmax(dm, fabs(v0 - lds_free(r + (uint32_t)(2 * CH + j) * 8u)));
          dm = fmax(dm, fabs(v1 - lds_free(r + (uint32_t)(2 * CH + j + 1) * 8u)));
          nanacc += v0 - v0;
          nanacc += v1 - v1;
          x[j] = v0;
          x[j + 1] = v1;
          asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(ro + (uint32_t)j * 8u), "d"(v0), "d"(v1) : "memory");
          asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(ro + (uint32_t)(CH + j) * 8u), "d"(g0), "d"(g1)
                       : "memory");
        }
      } else {
#pragma unroll
        for (int j = 0; j < CH; j += 2) {
          const double g0 = x[j], g1 = x[j + 1];
          const double v0 = (g0 + lds_free(r + (uint32_t)j * 8u)) - lds_free(r + (uint32_t)(CH + j) * 8u);
          const double v1 = (g1 + lds_free(r + (uint32_t)(j + 1) * 8u)) - lds_free(r + (uint32_t)(CH + j + 1) * 8u);
          dm = fmax(dm, fabs(v0 - lds_free(r + (uint32_t)(2 * CH + j) * 8u)));
          dm = fmax(dm, fabs(v1 - lds_free(r + (uint32_t)(2 * CH + j + 1) * 8u)));
          nanacc += v0 - v0;
          nanacc += v1 - v1;
          x[j] = v0;
          x[j + 1] = v1;
          asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(ro + (uint32_t)j * 8u), "d"(v0), "d"(v1) : "memory");
          asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(ro + (uint32_t)(CH + j) * 8u), "d"(g0), "d"(g1)
                       : "memory");
        }
      }
    } else {
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
    }
    __syncwarp();
    if (!GENERAL && !(defer & 1)) drain(i);
    if (GENERAL) {
      double *dsts[2] = {next + i * N + wbase, gcache + i * N + wbase};
      if (even) {
#pragma unroll
        for (int kk = 0; kk < CH / 2; ++kk) {
          const int e = kk * 64 + 2 * c.lane;
          const uint32_t src = wrow0 + (uint32_t)(e / CH) * RS + (uint32_t)(e % CH) * 8u;
          if (!GENERAL || wbase + e < N) {
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
  if (!GENERAL && (defer & 1)) drain(p);  // the last slice's results
  if (nanacc != nanacc) bad = true;
  // final reduction for slice p through one more gather round
  {
    const uint32_t gb = gather_exchange<true>(c, sc, 0.0, 0.0, dpart);
    const uint32_t stride8 = (uint32_t)(c.nW + 1) * 8u;
    double ex = 0.0;
    for (int V = c.lane; V < c.nW; V += 32) ex = fmax(ex, lds(gb + 2u * stride8 + (uint32_t)V * 8u));
    ex = warp_max(ex);
    if (rank == 0 && threadIdx.x == 0) deltas[p] = ex;
  }
  if (bad) atomicExch(nonfinite, 1);
  cluster.sync();
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
                     sm + sizeof(double) * (size_t)TB * ((3 * CH + 2) + (!GENERAL && op->sweep_defer ? 2 * CH + 2 : 0)),
                     s, P, prev, next, fv, gcache, k, p,
                     deltas, nonfinite, chain,
                     (!GENERAL && op->sweep_defer) ? (getenv("PINT_SWEEP_PREFETCH_SHADOW") ? 3 : 1) : 0);
      break;
  }
}

template <int CH, int J, bool CN>
static void run_kernel_t(TriKind kind, const pint_op *op, int grid_slices, int cl, cudaStream_t s,
                         const double *in, double *out, int64_t stride, double *lam, double *gcache,
                         int64_t p, const double *prev, double *next, const double *fv, int64_t k,
                         double *deltas, int32_t *nonfinite, int chain) {
  // GENERAL: a partially filled (tail) thread or boundary forcing; the fast path has neither
  // (backward Euler: the fast path is the constant-coefficient twisted chunk solve); see tri1d_setup
  if (op->tri_general)
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
  {
    // fused sweep: factor table + gather buffers + a staging row of 3 CH + 2
    // doubles per thread (tri1d_sweep_kernel); beyond ~100k points it no
    // longer fits and the sync engine uses the generic (per-slice) sweep
    const int TBs = pl.T / op->sweep_cluster;
    const size_t need = smem_bytes(pl, TBs) + sizeof(double) * (size_t)TBs * (3 * pl.CH + 2);
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) optin = 232448;
    op->fused_sweep = need <= (size_t)optin;
    // result rows of their own (deferred drain, fast kernels only) when they fit too
    op->sweep_defer = need + sizeof(double) * (size_t)TBs * (2 * pl.CH + 2) <= (size_t)optin;
  }
  // the fast kernels need every thread regular, every separator a real unknown
  // (N a multiple of CH), no boundary forcing and, for backward Euler, a
  // usable constant-coefficient chunk solve; PINT_TRI_FORCE_GENERAL=1 selects
  // the exact-pivot kernels regardless (A/B tests)
  op->tri_general = pl.tb < pl.T || pl.N % pl.CH != 0 || pl.f_first != 0.0 || pl.f_last != 0.0 ||
                    (!pl.cn && !pl.ccst);
  if (const char *fg = getenv("PINT_TRI_FORCE_GENERAL")) op->tri_general = op->tri_general || atoi(fg) != 0;
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
  if (!op->fused_sweep) pint_throw(PINT_EUNSUPPORTED, "the fused coarse sweep does not fit this grid (use the generic sweep)");
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


// Host-only export of the backward-Euler fast-path factors (include/pint_abi.h:
// pint_tri1d_ccst_host).
extern "C" int pint_tri1d_ccst_host(const pint_op_desc *d, int32_t *usable_out, double *fac_out) {
  if (!d || !usable_out) return PINT_EARG;
  try {
    if (d->ndim != 1 || d->rule != PINT_RULE_BACKWARD_EULER || d->steps < 1 || !(d->span > 0.0)) return PINT_EARG;
    const int CH = d->layout_ch == 16 ? 16 : 32;
    const double dt = d->span / (double)d->steps;
    Tri1DPlan pl = tri1d_plan(d->shape[0], CH, 1.0 - dt * d->a_diag, 0.0 - dt * d->a_off, dt * d->c_first,
                              dt * d->c_last, false, d->steps);
    const bool fast = pl.ccst && pl.tb >= pl.T && pl.N % CH == 0 && pl.f_first == 0.0 && pl.f_last == 0.0;
    *usable_out = fast ? 1 : 0;
    if (fac_out) memcpy(fac_out, pl.ccst_fac.data(), sizeof(double) * pl.ccst_fac.size());
    return PINT_OK;
  } catch (const PintError &e) {
    return e.code;
  }
}
