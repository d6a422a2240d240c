// Coarse implicit-Euler propagator for the 2-D/3-D zero-Dirichlet heat
// operator: solve (I - dT * Laplacian_h) x = b by conjugate gradients
// (reference analogue: backward_euler_propagator's dense LU solve,
// model.py:157-184; here matrix-free).
//
// Deterministic by construction: every reduction is a fixed-shape per-block
// partial sum followed by a single-block fixed-order sum, so G is a pure
// function of its input bits (required by the cached-G(old) cancellation of
// parareal.py:34-36 and the bitwise finite-termination property).
// The stencil apply is fused with the p.Ap partial dot; the x/r update is
// fused with the r.r partial dot. Iterations are launched in groups and a
// device-side "converged" flag turns the remaining kernels of a group into
// no-ops, so the host synchronises once per group, not per iteration.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "pint_internal.cuh"

namespace {

constexpr int CG_THREADS = 256;
constexpr int CG_BLOCKS = 148 * 4;
constexpr int CG_GROUP = 8;

struct CGState {
  double rr, rr_new, pap, bb, alpha, beta, stop;
  int done;
  int iters;
};

template <typename T>
__device__ __forceinline__ T lap_apply(const T *p, int64_t i, int nx, int ny, int nz, int x, int y, int z) {
  T nb = T(0);
  if (x > 0) nb += p[i - 1];
  if (x < nx - 1) nb += p[i + 1];
  if (y > 0) nb += p[i - nx];
  if (y < ny - 1) nb += p[i + nx];
  if (nz > 1) {
    if (z > 0) nb += p[i - (int64_t)nx * ny];
    if (z < nz - 1) nb += p[i + (int64_t)nx * ny];
  }
  return nb;
}

template <typename T>
__device__ __forceinline__ double block_sum(double v, double *red) {
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < CG_THREADS / 32; ++w) s += red[w];
  return s;
}

// init: x = 0, r = b, p = b, partial(b.b)
template <typename T>
__global__ void __launch_bounds__(CG_THREADS) cg_init(const T *b, T *x, T *r, T *p, int64_t n, double *part) {
  __shared__ double red[CG_THREADS / 32];
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * CG_THREADS + threadIdx.x; i < n; i += (int64_t)gridDim.x * CG_THREADS) {
    const T v = b[i];
    x[i] = T(0);
    r[i] = v;
    p[i] = v;
    acc += (double)v * (double)v;
  }
  double s = block_sum<T>(acc, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void cg_finish_init(const double *part, int nb, CGState *st, double rtol2) {
  __shared__ double red[CG_THREADS / 32];
  double acc = 0.0;
  for (int i = threadIdx.x; i < nb; i += CG_THREADS) acc += part[i];
  double s = block_sum<double>(acc, red);
  if (threadIdx.x == 0) {
    st->bb = s;
    st->rr = s;
    st->stop = rtol2 * s;
    st->done = (s <= st->stop) ? 1 : 0;
    st->iters = 0;
  }
}

// ap = (I - c Lap) p with c = dT/h^2 (per point: (1 + 2 d c) p - c * sum nb); partial p.ap
template <typename T>
__global__ void __launch_bounds__(CG_THREADS) cg_spmv(const T *p, T *ap, int nx, int ny, int nz, T cdiag, T coff,
                                                      double *part, const CGState *st) {
  if (st->done) return;
  __shared__ double red[CG_THREADS / 32];
  const int64_t n = (int64_t)nx * ny * nz;
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * CG_THREADS + threadIdx.x; i < n; i += (int64_t)gridDim.x * CG_THREADS) {
    const int x = (int)(i % nx);
    const int y = (int)((i / nx) % ny);
    const int z = (int)(i / ((int64_t)nx * ny));
    const T pv = p[i];
    const T v = cdiag * pv - coff * lap_apply<T>(p, i, nx, ny, nz, x, y, z);
    ap[i] = v;
    acc += (double)pv * (double)v;
  }
  double s = block_sum<T>(acc, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void cg_alpha(const double *part, int nb, CGState *st) {
  if (st->done) return;
  __shared__ double red[CG_THREADS / 32];
  double acc = 0.0;
  for (int i = threadIdx.x; i < nb; i += CG_THREADS) acc += part[i];
  double s = block_sum<double>(acc, red);
  if (threadIdx.x == 0) {
    st->pap = s;
    st->alpha = st->rr / s;
  }
}

// x += alpha p ; r -= alpha ap ; partial r.r
template <typename T>
__global__ void __launch_bounds__(CG_THREADS) cg_update(T *x, T *r, const T *p, const T *ap, int64_t n, double *part,
                                                        const CGState *st) {
  if (st->done) return;
  __shared__ double red[CG_THREADS / 32];
  const T alpha = (T)st->alpha;
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * CG_THREADS + threadIdx.x; i < n; i += (int64_t)gridDim.x * CG_THREADS) {
    x[i] = x[i] + alpha * p[i];
    const T rv = r[i] - alpha * ap[i];
    r[i] = rv;
    acc += (double)rv * (double)rv;
  }
  double s = block_sum<T>(acc, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void cg_beta(const double *part, int nb, CGState *st, int64_t maxit) {
  if (st->done) return;
  __shared__ double red[CG_THREADS / 32];
  double acc = 0.0;
  for (int i = threadIdx.x; i < nb; i += CG_THREADS) acc += part[i];
  double s = block_sum<double>(acc, red);
  if (threadIdx.x == 0) {
    st->rr_new = s;
    st->beta = s / st->rr;
    st->rr = s;
    st->iters += 1;
    if (s <= st->stop) st->done = 1;
    else if (st->iters >= maxit) st->done = 2;
  }
}

// p = r + beta p
template <typename T>
__global__ void __launch_bounds__(CG_THREADS) cg_pupdate(T *p, const T *r, int64_t n, const CGState *st) {
  if (st->done) return;
  const T beta = (T)st->beta;
  for (int64_t i = (int64_t)blockIdx.x * CG_THREADS + threadIdx.x; i < n; i += (int64_t)gridDim.x * CG_THREADS)
    p[i] = r[i] + beta * p[i];
}

template <typename T>
void cg_solve(pint_op *op, const T *b, T *x, cudaStream_t s) {
  const int64_t n = op->dim;
  T *r = reinterpret_cast<T *>(op->cg_work);
  T *p = r + n;
  T *ap = p + n;
  CGState *st = reinterpret_cast<CGState *>(op->cg_partials + CG_BLOCKS);
  const double c = op->dt / (op->desc.h * op->desc.h);
  const T coff = (T)c;
  const T cdiag = (T)(1.0 + 2.0 * op->desc.ndim * c);
  const int nb = (int)std::min<int64_t>(CG_BLOCKS, (n + CG_THREADS - 1) / CG_THREADS);
  const double rtol2 = op->desc.cg_rtol * op->desc.cg_rtol;
  const int64_t maxit = op->desc.cg_maxit > 0 ? op->desc.cg_maxit : 10000;
  cg_init<T><<<nb, CG_THREADS, 0, s>>>(b, x, r, p, n, op->cg_partials);
  cg_finish_init<<<1, CG_THREADS, 0, s>>>(op->cg_partials, nb, st, rtol2);
  PINT_CUDA(cudaGetLastError());
  CGState host;
  for (int64_t it = 0;; it += CG_GROUP) {
    for (int g = 0; g < CG_GROUP; ++g) {
      cg_spmv<T><<<nb, CG_THREADS, 0, s>>>(p, ap, (int)op->nx, (int)op->ny, (int)op->nz, cdiag, coff,
                                           op->cg_partials, st);
      cg_alpha<<<1, CG_THREADS, 0, s>>>(op->cg_partials, nb, st);
      cg_update<T><<<nb, CG_THREADS, 0, s>>>(x, r, p, ap, n, op->cg_partials, st);
      cg_beta<<<1, CG_THREADS, 0, s>>>(op->cg_partials, nb, st, maxit);
      cg_pupdate<T><<<nb, CG_THREADS, 0, s>>>(p, r, n, st);
    }
    PINT_CUDA(cudaGetLastError());
    PINT_CUDA(cudaMemcpyAsync(&host, st, sizeof(CGState), cudaMemcpyDeviceToHost, s));
    PINT_CUDA(cudaStreamSynchronize(s));
    if (host.done) break;
  }
  op->cg_last_iters = host.iters;
  if (host.done == 2)
    pint_throw(PINT_ENOCONV, "conjugate gradients did not reach the requested tolerance", std::sqrt(host.rr / host.bb));
}

}  // namespace

void cg_setup(pint_op *op) {
  op->dt = op->desc.span / (double)op->desc.steps;
  if (op->desc.steps != 1) {
    // several implicit steps per application: solve them one after another
  }
  if (!(op->desc.cg_rtol > 0.0)) pint_throw(PINT_EARG, "cg_rtol must be positive");
  const size_t esz = op->desc.dtype == PINT_F64 ? 8 : 4;
  op->cg_work_bytes = (size_t)3 * op->dim * esz;
  PINT_CUDA(cudaMalloc(&op->cg_work, op->cg_work_bytes));
  PINT_CUDA(cudaMalloc(&op->cg_partials, sizeof(double) * CG_BLOCKS + sizeof(CGState) + 64));
}

void cg_apply_batch(pint_op *op, const void *in, void *out, int64_t nbatch, int64_t stride, cudaStream_t s) {
  const size_t esz = op->desc.dtype == PINT_F64 ? 8 : 4;
  for (int64_t b = 0; b < nbatch; ++b) {
    const char *src = (const char *)in + (size_t)b * stride * esz;
    char *dst = (char *)out + (size_t)b * stride * esz;
    for (int64_t k = 0; k < op->desc.steps; ++k) {
      // step k solves into dst from the previous step's result (in place is
      // safe: the solver copies b into r/p before writing x)
      const void *bb = (k == 0) ? (const void *)src : (const void *)dst;
      if (op->desc.dtype == PINT_F64) cg_solve<double>(op, (const double *)bb, (double *)dst, s);
      else cg_solve<float>(op, (const float *)bb, (float *)dst, s);
    }
  }
}

void nd_implicit_apply_batch(pint_op *op, const void *in, void *out, int64_t nbatch, int64_t stride,
                             cudaStream_t s) {
  if (op->desc.nd_solver == PINT_ND_CG) cg_apply_batch(op, in, out, nbatch, stride, s);
  else spectral_apply_batch(op, in, out, nbatch, stride, s);
}

void nd_destroy(pint_op *op) {
  spectral_destroy(op);
  if (op->cg_work) cudaFree(op->cg_work);
  if (op->cg_partials) cudaFree(op->cg_partials);
  op->cg_work = nullptr;
  op->cg_partials = nullptr;
}
