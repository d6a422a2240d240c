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
// with c = dT / h^2. The transforms are dense GEMMs with an n x n operand
// (2 n FLOP per point per transformed axis, FP64/FP32 SIMT tiles; the
// tensor cores have no FP64 mode worth using on sm_100 and TF32 would not
// hold the fp32 tolerance), the tridiagonal sweeps are one thread per mode
// (coalesced across modes). Exact to rounding: no iteration, no tolerance,
// a pure function of the input bits, stream ordered with no host sync.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "pint_internal.cuh"

namespace {

template <typename T>
struct GemmArgs {
  const T *A;
  const T *B;
  T *C;
  int M, N, K;
  int lda, ldb, ldc;
  int inner;  // batch index z -> (z / inner, z % inner)
  int64_t a_outer, a_inner, b_outer, b_inner, c_outer, c_inner;
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

// C = A B (row-major, batched). 256 threads as 16 x 16; each thread owns a
// TM x TN register tile split in two halves per axis (rows ty*HM.. and
// BM/2 + ty*HM..), so its shared-memory operand reads are 2 vector loads per
// axis. K staged 8 at a time, double buffered through registers.
template <typename T, int BM, int BN>
__global__ void __launch_bounds__(256) gemm_nn(const GemmArgs<T> g) {
  constexpr int BK = 8, TM = BM / 16, TN = BN / 16, HM = TM / 2, HN = TN / 2;
  constexpr int LA = BM * BK / 256, LB = BN * BK / 256;
  __shared__ __align__(16) T As[2][BK][BM];
  __shared__ __align__(16) T Bs[2][BK][BN];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int bo = blockIdx.z / g.inner, bi = blockIdx.z % g.inner;
  const T *A = g.A + bo * g.a_outer + bi * g.a_inner;
  const T *B = g.B + bo * g.b_outer + bi * g.b_inner;
  T *C = g.C + bo * g.c_outer + bi * g.c_inner;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int a_row = tid / (BK / LA), a_k = (tid % (BK / LA)) * LA;
  const int b_row = tid / (BN / LB), b_n = (tid % (BN / LB)) * LB;
  T ra[LA], rb[LB];
  auto load = [&](int k0) {
#pragma unroll
    for (int i = 0; i < LA; ++i) {
      const int m = m0 + a_row, k = k0 + a_k + i;
      ra[i] = (m < g.M && k < g.K) ? A[(int64_t)m * g.lda + k] : T(0);
    }
#pragma unroll
    for (int i = 0; i < LB; ++i) {
      const int k = k0 + b_row, n = n0 + b_n + i;
      rb[i] = (k < g.K && n < g.N) ? B[(int64_t)k * g.ldb + n] : T(0);
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int i = 0; i < LA; ++i) As[buf][a_k + i][a_row] = ra[i];
#pragma unroll
    for (int i = 0; i < LB; ++i) Bs[buf][b_row][b_n + i] = rb[i];
  };
  T acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = T(0);
  load(0);
  store(0);
  __syncthreads();
  const int nk = (g.K + BK - 1) / BK;
  for (int t = 0; t < nk; ++t) {
    const int buf = t & 1;
    if (t + 1 < nk) load((t + 1) * BK);
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      T a[TM], b[TN];
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
    if (m >= g.M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int n = n0 + (j < HN ? tx * HN + j : BN / 2 + tx * HN + (j - HN));
      if (n < g.N) C[(int64_t)m * g.ldc + n] = acc[i][j];
    }
  }
}

template <typename T>
void gemm(const GemmArgs<T> &g, int batch, cudaStream_t s) {
  auto tiles = [&](int bm, int bn) {
    return (int64_t)((g.M + bm - 1) / bm) * ((g.N + bn - 1) / bn) * batch;
  };
  // FP64: 4x4 per thread already keeps the DFMA pipe ahead of shared memory.
  // FP32: 8x8 per thread when that still fills two waves of 148 SMs.
  const bool big = sizeof(T) == 4 && tiles(128, 128) >= 2 * 148;
  if (big) {
    dim3 grid((unsigned)((g.N + 127) / 128), (unsigned)((g.M + 127) / 128), (unsigned)batch);
    gemm_nn<T, 128, 128><<<grid, 256, 0, s>>>(g);
  } else {
    dim3 grid((unsigned)((g.N + 63) / 64), (unsigned)((g.M + 63) / 64), (unsigned)batch);
    gemm_nn<T, 64, 64><<<grid, 256, 0, s>>>(g);
  }
  PINT_CUDA(cudaGetLastError());
}

// One thread per transverse mode: `steps` backward-Euler solves along the
// slowest axis (n points, `nsys` modes interleaved: point j of mode i at
// u[j * nsys + i]). Pivots in FP64, recomputed per step (c/p_j kept in
// `ratio` for the back substitution).
template <typename T>
__global__ void __launch_bounds__(256)
modal_tridiag(T *__restrict__ u, T *__restrict__ ratio, const double *__restrict__ mu, int n, int64_t nsys,
              int two_axes, double c, int64_t steps) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nsys) return;
  double m = mu[i % n];
  if (two_axes) m += mu[i / n];
  const double d = 1.0 + 2.0 * c + c * m;
  for (int64_t s = 0; s < steps; ++s) {
    double ip = 1.0 / d;
    double g = (double)u[i] * ip;
    double r = c * ip;
    u[i] = (T)g;
    ratio[i] = (T)r;
    for (int j = 1; j < n; ++j) {
      const int64_t o = (int64_t)j * nsys + i;
      ip = 1.0 / (d - c * r);
      g = ((double)u[o] + c * g) * ip;
      r = c * ip;
      u[o] = (T)g;
      ratio[o] = (T)r;
    }
    double x = g;
    for (int j = n - 2; j >= 0; --j) {
      const int64_t o = (int64_t)j * nsys + i;
      x = (double)u[o] + (double)ratio[o] * x;
      u[o] = (T)x;
    }
  }
}

template <typename T>
void spectral_solve(pint_op *op, const T *b, T *x, cudaStream_t s) {
  const int n = (int)op->nx;
  const int64_t n2 = (int64_t)n * n;
  T *w1 = reinterpret_cast<T *>(op->cg_work);
  T *w2 = w1 + op->dim;
  T *rat = w2 + op->dim;
  const T *Q = reinterpret_cast<const T *>(op->spec_q);
  const double c = op->dt / (op->desc.h * op->desc.h);
  auto xform_last = [&](const T *src, T *dst, int rows) {  // dst = src Q (rows x n)
    GemmArgs<T> g{src, Q, dst, rows, n, n, n, n, n, 1, 0, 0, 0, 0, 0, 0};
    gemm<T>(g, 1, s);
  };
  auto xform_mid = [&](const T *src, T *dst) {  // dst_z = Q src_z for every z plane
    GemmArgs<T> g{Q, src, dst, n, n, n, n, n, n, n, 0, 0, 0, n2, 0, n2};
    gemm<T>(g, n, s);
  };
  const unsigned threads = 256;
  if (op->desc.ndim == 2) {
    xform_last(b, w1, n);
    modal_tridiag<T><<<(unsigned)((n + threads - 1) / threads), threads, 0, s>>>(w1, rat, op->spec_mu, n, n, 0, c,
                                                                               op->desc.steps);
    PINT_CUDA(cudaGetLastError());
    xform_last(w1, x, n);
  } else {
    xform_last(b, w1, (int)n2);
    xform_mid(w1, w2);
    modal_tridiag<T><<<(unsigned)((n2 + threads - 1) / threads), threads, 0, s>>>(w2, rat, op->spec_mu, n, n2, 1,
                                                                                c, op->desc.steps);
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
  op->cg_work_bytes = (size_t)3 * op->dim * esz;
  PINT_CUDA(cudaMalloc(&op->cg_work, op->cg_work_bytes));
  std::vector<double> mu(n);
  std::vector<double> qd((size_t)n * n);
  std::vector<float> qf(esz == 4 ? (size_t)n * n : 0);
  const long double pi = 3.141592653589793238462643383279502884L;
  const long double scale = sqrtl(2.0L / (long double)(n + 1));
  for (int64_t k = 0; k < n; ++k) {
    const long double sk = sinl(pi * (long double)(k + 1) / (2.0L * (long double)(n + 1)));
    mu[k] = (double)(4.0L * sk * sk);
  }
  for (int64_t j = 0; j < n; ++j)
    for (int64_t k = 0; k < n; ++k) {
      // reduce (j+1)(k+1) mod 2(n+1) before the sine: exact integer argument
      const int64_t a = ((j + 1) * (k + 1)) % (2 * (n + 1));
      const long double v = scale * sinl(pi * (long double)a / (long double)(n + 1));
      qd[(size_t)j * n + k] = (double)v;
      if (esz == 4) qf[(size_t)j * n + k] = (float)v;
    }
  PINT_CUDA(cudaMalloc(&op->spec_mu, sizeof(double) * n));
  PINT_CUDA(cudaMemcpy(op->spec_mu, mu.data(), sizeof(double) * n, cudaMemcpyHostToDevice));
  PINT_CUDA(cudaMalloc(&op->spec_q, esz * n * n));
  PINT_CUDA(cudaMemcpy(op->spec_q, esz == 8 ? (const void *)qd.data() : (const void *)qf.data(), esz * n * n,
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
  if (op->spec_mu) cudaFree(op->spec_mu);
  op->spec_q = nullptr;
  op->spec_mu = nullptr;
}
