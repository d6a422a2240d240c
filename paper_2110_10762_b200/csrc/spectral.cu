// Direct coarse solve for the 2-D/3-D backward-Euler heat step
//   (I - dT * Laplacian_h) x = b,   zero Dirichlet, n points per axis,
// the B200 replacement of the reference's dense LU solve of the same system
// (model.py:157-184 via linalg.py:241-266).
//
// Matrix decomposition method: the orthonormal sine transform
//   Q[j][k] = sqrt(2/(n+1)) sin(pi (j+1)(k+1) / (n+1))      (Q = Q^T = Q^-1)
// diagonalises the 1-D Dirichlet Laplacian (eigenvalues -mu_k / h^2,
// mu_k = 4 sin^2(pi (k+1) / (2(n+1)))). Transforming every axis but the
// slowest one leaves independent constant-coefficient tridiagonal systems
// along the slowest axis, one per transverse mode:
//   2-D [y][x]:    W = B Q ;  tridiag_y(1 + 2c + c mu_kx, -c) ;  X = W Q
//   3-D [z][y][x]: W = B Q ;  W_z = Q W_z ;  tridiag_z(1 + 2c + c (mu_kx + mu_ky), -c) ;
//                  W_z = Q W_z ;  X = W Q
// with c = dT / h^2. The transforms are dense GEMMs, halved by the parity
// symmetry of Q (n FLOP per point per transformed axis). fp32 with n a
// multiple of 256 runs them on the tensor cores in 3xTF32 split precision
// (tc_xform.cu: tcgen05.mma, TMEM accumulators, the constant Q pre-split on
// the host); fp64 and other shapes use register-tiled SIMT tiles below (no
// FP64 tensor-core mode worth using on sm_100). The tridiagonal sweeps are one
// thread per mode (coalesced across modes). Exact to rounding: no iteration,
// no tolerance, a pure function of the input bits, stream ordered with no
// host sync.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "pint_internal.cuh"

bool tc_xform_supported(int n);
std::vector<uint32_t> tc_split_q(int n, const long double *q);
void tc_xform_last(const float *src, float *dst, const uint32_t *qs, int n, int64_t rows, cudaStream_t s);
void tc_xform_mid(const float *src, float *dst, const uint32_t *qs, int n, int planes, cudaStream_t s);

namespace {

// C = A B, row-major, batched (z -> (z / inner, z % inner) with per-operand
// strides). FOLD applies the parity symmetry of the sine transform,
// Q[n-1-i][j] = (-1)^j Q[i][j], to halve the K extent: z = 2*batch + par and
//   FOLD 1 (transform along A's columns): A'[m][k] = A[m][k] +- A[m][n-1-k],
//          B = half[par] (K' x N_par), output column 2 q + par;
//   FOLD 2 (transform along B's rows):    B'[k][x] = B[k][x] +- B[n-1-k][x],
//          A = half[par] (M_par x K'), output row 2 q + par;
// with K' = ceil(n/2) and the sign + for even, - for odd output indices.
// byte offset of the fp64 modal-sweep scratch inside an fp32 op's work area
static size_t spectral_g64_offset(int64_t dim) { return ((size_t)3 * dim * 4 + 255) / 256 * 256; }

template <typename T>
struct GemmArgs {
  const T *A;
  const T *B;
  T *C;
  int M, N, K;
  int lda, ldb, ldc;
  int inner;
  int64_t a_outer, a_inner, b_outer, b_inner, c_outer, c_inner;
  const T *half[2];
  int mn[2];
  int ldh[2];
  int nfold;
};

__device__ __forceinline__ void ld2(const float *p, float *d) {
  const float2 v = *reinterpret_cast<const float2 *>(p);
  d[0] = v.x;
  d[1] = v.y;
}
__device__ __forceinline__ void ld4(const float *p, float *d) {
  const float4 v = *reinterpret_cast<const float4 *>(p);
  d[0] = v.x;
  d[1] = v.y;
  d[2] = v.z;
  d[3] = v.w;
}
__device__ __forceinline__ void ld2(const double *p, double *d) {
  const double2 v = *reinterpret_cast<const double2 *>(p);
  d[0] = v.x;
  d[1] = v.y;
}
__device__ __forceinline__ void ld4(const double *p, double *d) {
  ld2(p, d);
  ld2(p + 2, d + 2);
}
template <int NV, typename T>
__device__ __forceinline__ void ldv(const T *p, T *d) {
  if constexpr (NV == 2) ld2(p, d);
  else ld4(p, d);
}

// 256 threads as 16 x 16; each thread owns a TM x TN register tile split in
// two halves per axis (rows ty*HM.. and BM/2 + ty*HM..), so its shared-memory
// operand reads are 2 vector loads per axis. K staged 8 at a time, double
// buffered through registers. Acc is the accumulation (and fold) type: fp32
// operands accumulate in fp64 (DFMA), so an fp32 solve carries only the
// rounding of its stored operands, not a sqrt(K)-growing accumulation error
// (C3 fp32: the coarse chain of 32 solves moved 1.4e-5 off the exact solve
// with fp32 accumulation, tests/test_gpu_config_parity.py).
template <typename T, int BM, int BN, int FOLD, int MINB, typename Acc = T>
__global__ void __launch_bounds__(256, MINB) gemm_nn(const GemmArgs<T> g) {
  constexpr int BK = 8, TM = BM / 16, TN = BN / 16, HM = TM / 2, HN = TN / 2;
  constexpr int LA = BM * BK / 256, LB = BN * BK / 256;
  __shared__ __align__(16) Acc As[2][BK][BM];
  __shared__ __align__(16) Acc Bs[2][BK][BN];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  int z = blockIdx.z, par = 0;
  if (FOLD) {
    par = z & 1;
    z >>= 1;
  }
  const int bo = z / g.inner, bi = z % g.inner;
  const T *A = FOLD == 2 ? g.half[par] : g.A + bo * g.a_outer + bi * g.a_inner;
  const T *B = FOLD == 1 ? g.half[par] : g.B + bo * g.b_outer + bi * g.b_inner;
  const int lda = FOLD == 2 ? g.ldh[par] : g.lda;
  const int ldb = FOLD == 1 ? g.ldh[par] : g.ldb;
  const int M = FOLD == 2 ? g.mn[par] : g.M;
  const int N = FOLD == 1 ? g.mn[par] : g.N;
  const int K = g.K;
  T *C = g.C + bo * g.c_outer + bi * g.c_inner;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  if (m0 >= M || n0 >= N) return;
  const int a_row = tid / (BK / LA), a_k = (tid % (BK / LA)) * LA;
  const int b_row = tid / (BN / LB), b_n = (tid % (BN / LB)) * LB;
  Acc ra[LA], rb[LB];
  auto load = [&](int k0) {
#pragma unroll
    for (int i = 0; i < LA; ++i) {
      const int m = m0 + a_row, k = k0 + a_k + i;
      Acc v = Acc(0);
      if (m < M && k < K) {
        v = (Acc)A[(int64_t)m * lda + k];
        if (FOLD == 1) {
          const int k2 = g.nfold - 1 - k;
          if (k2 > k) v = par ? v - (Acc)A[(int64_t)m * lda + k2] : v + (Acc)A[(int64_t)m * lda + k2];
        }
      }
      ra[i] = v;
    }
#pragma unroll
    for (int i = 0; i < LB; ++i) {
      const int k = k0 + b_row, n = n0 + b_n + i;
      Acc v = Acc(0);
      if (k < K && n < N) {
        v = (Acc)B[(int64_t)k * ldb + n];
        if (FOLD == 2) {
          const int k2 = g.nfold - 1 - k;
          if (k2 > k) v = par ? v - (Acc)B[(int64_t)k2 * ldb + n] : v + (Acc)B[(int64_t)k2 * ldb + n];
        }
      }
      rb[i] = v;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int i = 0; i < LA; ++i) As[buf][a_k + i][a_row] = ra[i];
#pragma unroll
    for (int i = 0; i < LB; ++i) Bs[buf][b_row][b_n + i] = rb[i];
  };
  Acc acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = Acc(0);
  load(0);
  store(0);
  __syncthreads();
  const int nk = (K + BK - 1) / BK;
  for (int t = 0; t < nk; ++t) {
    const int buf = t & 1;
    if (t + 1 < nk) load((t + 1) * BK);
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      Acc a[TM], b[TN];
      ldv<HM>(&As[buf][k][ty * HM], a);
      ldv<HM>(&As[buf][k][BM / 2 + ty * HM], a + HM);
      ldv<HN>(&Bs[buf][k][tx * HN], b);
      ldv<HN>(&Bs[buf][k][BN / 2 + tx * HN], b + HN);
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    if (t + 1 < nk) store(buf ^ 1);
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int m = m0 + (i < HM ? ty * HM + i : BM / 2 + ty * HM + (i - HM));
    if (m >= M) continue;
    const int64_t row = FOLD == 2 ? 2 * m + par : m;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int n = n0 + (j < HN ? tx * HN + j : BN / 2 + tx * HN + (j - HN));
      if (n < N) C[row * g.ldc + (FOLD == 1 ? 2 * n + par : n)] = (T)acc[i][j];
    }
  }
}

template <typename T, int FOLD>
void gemm(const GemmArgs<T> &g, int batch, cudaStream_t s) {
  const int M = FOLD == 2 ? g.mn[0] : g.M, N = FOLD == 1 ? g.mn[0] : g.N;  // parity 0 is the larger half
  const int zs = batch * (FOLD ? 2 : 1);
  auto tiles = [&](int bm, int bn) { return (int64_t)((M + bm - 1) / bm) * ((N + bn - 1) / bn) * zs; };
  (void)tiles;
  // 4x4 per thread keeps the DFMA pipe ahead of shared memory; fp32 operands
  // are staged and accumulated in fp64 (see gemm_nn)
  dim3 grid((unsigned)((N + 63) / 64), (unsigned)((M + 63) / 64), (unsigned)zs);
  gemm_nn<T, 64, 64, FOLD, 1, double><<<grid, 256, 0, s>>>(g);
  PINT_CUDA(cudaGetLastError());
}

// Few transverse modes (2-D grids: n systems of length n) leave the
// one-thread-per-mode sweep on a handful of SMs (C3: 1024 threads = 8 SMs,
// 169 us). Here each system is split into MC chunks: warp-of-chunks x
// system-lane threads (lanes = consecutive systems, so every row access is
// coalesced), each thread composes its chunk's affine map of the first-order
// recurrences (forward g_j = (c g_{j-1} + d_j) p_j^-1; backward
// x_j = g_j + c p_j^-1 x_{j+1}), the chunk entry values are chained through
// shared memory, and every chunk is recomputed from its exact entry value
// with the sequential formula. Same operator, rounding-level differences
// only (the recurrences contract: c p_j^-1 < 1).
template <typename T, int MC, int SYS>
__global__ void __launch_bounds__(MC * SYS)
modal_tridiag_chunked(T *__restrict__ u, const double *__restrict__ ipt, double *__restrict__ g64, int J, int n,
                      int64_t nsys, double c, int64_t steps) {
  // forward intermediates g_j: kept in fp64 (g64) for fp32 states — rounding
  // them to fp32 before the back substitution (x_j = g_j + e_j x_{j+1},
  // e_j -> 1 for strongly coupled modes) cost 8.7e-7 per C3 solve
  auto gst = [&](int64_t idx, double v) {
    if constexpr (sizeof(T) == 4) g64[idx] = v;
    else u[idx] = (T)v;
  };
  auto gld = [&](int64_t idx) -> double {
    if constexpr (sizeof(T) == 4) return g64[idx];
    else return (double)u[idx];
  };
  __shared__ double cmp[2][MC][SYS];  // chunk maps (A, B)
  __shared__ double entry[MC + 1][SYS];
  const int w = threadIdx.x / SYS, sl = threadIdx.x % SYS;
  const int64_t i = (int64_t)blockIdx.x * SYS + sl;
  const bool live = i < nsys;
  const int L = (n + MC - 1) / MC, j0 = w * L, j1 = min(n, j0 + L);  // chunk [j0, j1)
  const double ipinf = live ? (double)ipt[(int64_t)(J - 1) * nsys + i] : 0.0;
  auto ipat = [&](int j) { return j < J ? (double)ipt[(int64_t)j * nsys + i] : ipinf; };
  for (int64_t s = 0; s < steps; ++s) {
    // ---- forward: g_end = A g_in + B over the chunk
    double A = 1.0, B = 0.0;
    if (live)
      for (int j = j0; j < j1; ++j) {
        const double ip = ipat(j);
        A = (c * ip) * A;
        B = fma(c, B, (double)u[(int64_t)j * nsys + i]) * ip;
      }
    cmp[0][w][sl] = A;
    cmp[1][w][sl] = B;
    __syncthreads();
    if (w == 0) {
      double g = 0.0;
      for (int q = 0; q < MC; ++q) {
        entry[q][sl] = g;
        g = fma(cmp[0][q][sl], g, cmp[1][q][sl]);
      }
    }
    __syncthreads();
    double g = entry[w][sl];
    if (live)
      for (int j = j0; j < j1; ++j) {
        g = fma(c, g, (double)u[(int64_t)j * nsys + i]) * ipat(j);
        gst((int64_t)j * nsys + i, g);
      }
    __syncthreads();
    // ---- backward: x_j = g_j + e_j x_{j+1}, e_j = c / p_j (e_{n-1} = 0)
    double C = 1.0, D = 0.0;
    if (live)
      for (int j = j1 - 1; j >= j0; --j) {
        const double e = j == n - 1 ? 0.0 : c * ipat(j);
        C = e * C;
        D = fma(e, D, gld((int64_t)j * nsys + i));
      }
    cmp[0][w][sl] = C;
    cmp[1][w][sl] = D;
    __syncthreads();
    if (w == 0) {
      double x = 0.0;
      for (int q = MC - 1; q >= 0; --q) {
        entry[q][sl] = x;
        x = fma(cmp[0][q][sl], x, cmp[1][q][sl]);
      }
    }
    __syncthreads();
    double x = entry[w][sl];
    if (live)
      for (int j = j1 - 1; j >= j0; --j) {
        const double e = j == n - 1 ? 0.0 : c * ipat(j);
        x = fma(e, x, gld((int64_t)j * nsys + i));
        u[(int64_t)j * nsys + i] = (T)x;
      }
    __syncthreads();
  }
}

// One thread per transverse mode: `steps` backward-Euler solves along the
// slowest axis (n points, `nsys` modes interleaved: point j of mode i at
// u[j * nsys + i]). The reciprocal pivots 1/p_j (p_0 = d, p_j = d - c^2 /
// p_{j-1}) do not depend on the right-hand side and converge geometrically
// in j, so they come from a host-built table ipt[j][mode] (long double,
// rows j < J; row J-1 is the converged value used for every j >= J-1). The
// dependent chain is then one FMA and one multiply per point; loads are
// issued a block of U points ahead of it.
template <typename T>
__global__ void __launch_bounds__(128)
modal_tridiag(T *__restrict__ u, const double *__restrict__ ipt, double *__restrict__ g64, int J, int n, int64_t nsys,
              double c, int64_t steps) {
  constexpr int U = 8;
  // forward intermediates in fp64 for fp32 states (see modal_tridiag_chunked)
  auto gst = [&](int64_t idx, double v) {
    if constexpr (sizeof(T) == 4) g64[idx] = v;
    else u[idx] = (T)v;
  };
  auto gld = [&](int64_t idx) -> double {
    if constexpr (sizeof(T) == 4) return g64[idx];
    else return (double)u[idx];
  };
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nsys) return;
  const double ipinf = (double)ipt[(int64_t)(J - 1) * nsys + i];
  auto ipat = [&](int j) { return j < J ? (double)ipt[(int64_t)j * nsys + i] : ipinf; };
  for (int64_t s = 0; s < steps; ++s) {
    double g = 0.0;
    T cur[U], nxt[U];
    double cip[U], nip[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      cur[q] = q < n ? u[(int64_t)q * nsys + i] : T(0);
      cip[q] = ipat(q);
    }
    for (int j0 = 0; j0 < n; j0 += U) {
#pragma unroll
      for (int q = 0; q < U; ++q) {
        nxt[q] = j0 + U + q < n ? u[(int64_t)(j0 + U + q) * nsys + i] : T(0);
        nip[q] = ipat(j0 + U + q);
      }
#pragma unroll
      for (int q = 0; q < U; ++q) {
        if (j0 + q < n) {
          g = fma(c, g, (double)cur[q]) * cip[q];
          gst((int64_t)(j0 + q) * nsys + i, g);
        }
      }
#pragma unroll
      for (int q = 0; q < U; ++q) {
        cur[q] = nxt[q];
        cip[q] = nip[q];
      }
    }
    // back substitution x_j = g_j + (c / p_j) x_{j+1}, blocks of U from the top
    double x = g;
    if constexpr (sizeof(T) == 4) u[(int64_t)(n - 1) * nsys + i] = (T)x;  // x_{n-1} = g_{n-1}
    double cg[U], ng[U];
    auto fetch = [&](int top, double *gg, double *pp) {
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const int jj = top - q;
        gg[q] = jj >= 0 ? gld((int64_t)jj * nsys + i) : 0.0;
        pp[q] = jj >= 0 ? ipat(jj) : 0.0;
      }
    };
    fetch(n - 2, cg, cip);
    for (int top = n - 2; top >= 0; top -= U) {
      fetch(top - U, ng, nip);
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const int jj = top - q;
        if (jj >= 0) {
          x = fma(c * cip[q], x, cg[q]);
          u[(int64_t)jj * nsys + i] = (T)x;
        }
      }
#pragma unroll
      for (int q = 0; q < U; ++q) {
        cg[q] = ng[q];
        cip[q] = nip[q];
      }
    }
  }
}

template <typename T>
void spectral_solve(pint_op *op, const T *b, T *x, cudaStream_t s) {
  const int n = (int)op->nx;
  const int64_t n2 = (int64_t)n * n;
  const int kh = (n + 1) / 2, n0 = (n + 1) / 2, n1 = n / 2;  // folded K; output counts per parity
  T *w1 = reinterpret_cast<T *>(op->cg_work);
  T *w2 = w1 + op->dim;
  // fp64 forward intermediates of the modal sweep (fp32 states only)
  double *g64 = sizeof(T) == 4 ? reinterpret_cast<double *>(reinterpret_cast<char *>(op->cg_work) +
                                                             spectral_g64_offset(op->dim))
                               : nullptr;
  const T *Q = reinterpret_cast<const T *>(op->spec_q);
  // host layout of spec_q: Qh[0] (kh x n0), Qh[1] (kh x n1), QhT[0] (n0 x kh), QhT[1] (n1 x kh)
  const T *qh0 = Q, *qh1 = qh0 + (size_t)kh * n0, *qt0 = qh1 + (size_t)kh * n1, *qt1 = qt0 + (size_t)n0 * kh;
  const double c = op->dt / (op->desc.h * op->desc.h);
  // fp32 on the tensor cores (3xTF32, tc_xform.cu) where the shape allows;
  // PINT_TC_XFORM=0 keeps the SIMT GEMMs (measurement)
  bool tc = false;
  if constexpr (sizeof(T) == 4) {
    const char *e = getenv("PINT_TC_XFORM");
    // 3-D only: a 2-D transform (n rows) is too small a grid for the tensor-core tiles
    // (1024^2: 0.376 vs 0.349 ms SIMT, scripts/tc_xform_probe.py)
    tc = op->spec_tcq != nullptr && op->desc.ndim == 3 && !(e && atoi(e) == 0);
  }
  auto xform_last = [&](const T *src, T *dst, int rows) {  // dst = src Q (rows x n)
    if constexpr (sizeof(T) == 4) {
      if (tc) {
        tc_xform_last(src, dst, reinterpret_cast<const uint32_t *>(op->spec_tcq), n, rows, s);
        return;
      }
    }
    GemmArgs<T> g{};
    g.A = src;
    g.C = dst;
    g.M = rows;
    g.K = kh;
    g.lda = n;
    g.ldc = n;
    g.inner = 1;
    g.half[0] = qh0;
    g.half[1] = qh1;
    g.mn[0] = n0;
    g.mn[1] = n1;
    g.ldh[0] = n0;
    g.ldh[1] = n1 > 0 ? n1 : 1;
    g.nfold = n;
    gemm<T, 1>(g, 1, s);
  };
  auto xform_mid = [&](const T *src, T *dst) {  // dst_z = Q src_z for every z plane
    if constexpr (sizeof(T) == 4) {
      if (tc) {
        tc_xform_mid(src, dst, reinterpret_cast<const uint32_t *>(op->spec_tcq), n, n, s);
        return;
      }
    }
    GemmArgs<T> g{};
    g.B = src;
    g.C = dst;
    g.N = n;
    g.K = kh;
    g.ldb = n;
    g.ldc = n;
    g.inner = n;
    g.b_inner = n2;
    g.c_inner = n2;
    g.half[0] = qt0;
    g.half[1] = qt1;
    g.mn[0] = n0;
    g.mn[1] = n1;
    g.ldh[0] = kh;
    g.ldh[1] = kh;
    g.nfold = n;
    gemm<T, 2>(g, n, s);
  };
  const unsigned threads = 128;
  if (op->desc.ndim == 2) {
    xform_last(b, w1, n);
    const char *mc = getenv("PINT_MODAL_CHUNKED");
    if (n >= 256 && !(mc && atoi(mc) == 0)) {
      constexpr int MC = 64, SYS = 16;
      modal_tridiag_chunked<T, MC, SYS><<<(unsigned)((n + SYS - 1) / SYS), MC * SYS, 0, s>>>(
          w1, reinterpret_cast<const double *>(op->spec_ip), g64, op->spec_J, n, n, c, op->desc.steps);
    } else {
      modal_tridiag<T><<<(unsigned)((n + threads - 1) / threads), threads, 0, s>>>(
          w1, reinterpret_cast<const double *>(op->spec_ip), g64, op->spec_J, n, n, c, op->desc.steps);
    }
    PINT_CUDA(cudaGetLastError());
    xform_last(w1, x, n);
  } else {
    xform_last(b, w1, (int)n2);
    xform_mid(w1, w2);
    // (the chunked sweep measured slower here: 3-D grids have n^2 modes, 0.510 vs 0.480 ms at C4)
    modal_tridiag<T><<<(unsigned)((n2 + threads - 1) / threads), threads, 0, s>>>(
        w2, reinterpret_cast<const double *>(op->spec_ip), g64, op->spec_J, n, n2, c, op->desc.steps);
    PINT_CUDA(cudaGetLastError());
    xform_mid(w2, w1);
    xform_last(w1, x, (int)n2);
  }
}

}  // namespace

void spectral_setup(pint_op *op) {
  op->dt = op->desc.span / (double)op->desc.steps;
  const int64_t n = op->nx;
  if (op->ny != n || (op->desc.ndim == 3 && op->nz != n))
    pint_throw(PINT_EDIM, "direct solve needs the same point count on every axis");
  if (n * n > 0x7fffffffLL) pint_throw(PINT_EDIM, "grid too large");
  const size_t esz = op->desc.dtype == PINT_F64 ? 8 : 4;
  op->cg_work_bytes = esz == 8 ? (size_t)3 * op->dim * esz : spectral_g64_offset(op->dim) + (size_t)op->dim * 8;
  PINT_CUDA(cudaMalloc(&op->cg_work, op->cg_work_bytes));
  std::vector<long double> mu(n);
  std::vector<long double> q((size_t)n * n);
  const long double pi = 3.141592653589793238462643383279502884L;
  const long double scale = sqrtl(2.0L / (long double)(n + 1));
  for (int64_t k = 0; k < n; ++k) {
    const long double sk = sinl(pi * (long double)(k + 1) / (2.0L * (long double)(n + 1)));
    mu[k] = 4.0L * sk * sk;
  }
  for (int64_t j = 0; j < n; ++j)
    for (int64_t k = 0; k < n; ++k) {
      // reduce (j+1)(k+1) mod 2(n+1) before the sine: exact integer argument
      const int64_t a = ((j + 1) * (k + 1)) % (2 * (n + 1));
      const long double v = scale * sinl(pi * (long double)a / (long double)(n + 1));
      q[(size_t)j * n + k] = v;
    }
  // parity-folded halves (see GemmArgs): Qh[par][k][t] = Q[k][2t+par],
  // QhT[par][t][k] = Q[2t+par][k], k < ceil(n/2)
  const int64_t kh = (n + 1) / 2, cnt[2] = {(n + 1) / 2, n / 2};
  std::vector<long double> packed;
  for (int par = 0; par < 2; ++par)
    for (int64_t k = 0; k < kh; ++k)
      for (int64_t t = 0; t < cnt[par]; ++t) packed.push_back(q[(size_t)k * n + 2 * t + par]);
  for (int par = 0; par < 2; ++par)
    for (int64_t t = 0; t < cnt[par]; ++t)
      for (int64_t k = 0; k < kh; ++k) packed.push_back(q[(size_t)(2 * t + par) * n + k]);
  std::vector<double> qd(packed.size());
  std::vector<float> qf(esz == 4 ? packed.size() : 0);
  for (size_t e = 0; e < packed.size(); ++e) {
    qd[e] = (double)packed[e];
    if (esz == 4) qf[e] = (float)packed[e];
  }
  // reciprocal pivots per transverse mode, rows until every mode has
  // converged (|p_j - p_{j-1}| <= 2^-64 p_j), capped at n
  const long double cl = (long double)op->dt / ((long double)op->desc.h * (long double)op->desc.h);
  const int64_t nsys = op->desc.ndim == 2 ? n : n * n;
  std::vector<long double> dmode(nsys);
  for (int64_t m = 0; m < nsys; ++m) {
    const long double mus = op->desc.ndim == 2 ? mu[m] : mu[m % n] + mu[m / n];
    dmode[m] = 1.0L + 2.0L * cl + cl * mus;
  }
  int64_t J = 1;
  {
    // the slowest-converging mode is the one with the smallest diagonal
    long double dmin = dmode[0];
    for (int64_t m = 1; m < nsys; ++m) dmin = std::min(dmin, dmode[m]);
    long double pv = dmin;
    for (J = 1; J < n; ++J) {
      const long double pn = dmin - cl * cl / pv;
      if (fabsl(pn - pv) <= ldexpl(pn, -64)) break;
      pv = pn;
    }
    J = std::min<int64_t>(J + 1, n);
  }
  // fp64 for both state types: the pivots of strongly coupled modes are
  // where fp32 rounding would be amplified
  std::vector<double> ipd((size_t)J * nsys);
  for (int64_t m = 0; m < nsys; ++m) {
    long double pv = dmode[m];
    for (int64_t jj = 0; jj < J; ++jj) {
      if (jj > 0) pv = dmode[m] - cl * cl / pv;
      ipd[(size_t)jj * nsys + m] = (double)(1.0L / pv);
    }
  }
  op->spec_J = (int)J;
  PINT_CUDA(cudaMalloc(&op->spec_ip, 8 * ipd.size()));
  PINT_CUDA(cudaMemcpy(op->spec_ip, ipd.data(), 8 * ipd.size(), cudaMemcpyHostToDevice));
  if (esz == 4 && op->desc.ndim == 3 && tc_xform_supported((int)n)) {
    const std::vector<uint32_t> tcq = tc_split_q((int)n, q.data());
    PINT_CUDA(cudaMalloc(&op->spec_tcq, 4 * tcq.size()));
    PINT_CUDA(cudaMemcpy(op->spec_tcq, tcq.data(), 4 * tcq.size(), cudaMemcpyHostToDevice));
  }
  PINT_CUDA(cudaMalloc(&op->spec_q, esz * qd.size()));
  PINT_CUDA(cudaMemcpy(op->spec_q, esz == 8 ? (const void *)qd.data() : (const void *)qf.data(), esz * qd.size(),
                       cudaMemcpyHostToDevice));
}

void spectral_apply_batch(pint_op *op, const void *in, void *out, int64_t nbatch, int64_t stride, cudaStream_t s) {
  const size_t esz = op->desc.dtype == PINT_F64 ? 8 : 4;
  for (int64_t b = 0; b < nbatch; ++b) {
    const char *src = (const char *)in + (size_t)b * stride * esz;
    char *dst = (char *)out + (size_t)b * stride * esz;
    if (op->desc.dtype == PINT_F64) spectral_solve<double>(op, (const double *)src, (double *)dst, s);
    else spectral_solve<float>(op, (const float *)src, (float *)dst, s);
  }
}

void spectral_destroy(pint_op *op) {
  if (op->spec_q) cudaFree(op->spec_q);
  if (op->spec_ip) cudaFree(op->spec_ip);
  if (op->spec_tcq) cudaFree(op->spec_tcq);
  op->spec_tcq = nullptr;
  op->spec_q = nullptr;
  op->spec_ip = nullptr;
}
