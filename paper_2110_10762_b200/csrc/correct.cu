// Predictor-corrector update with fused convergence norm (reference:
// parareal_update parareal.py:25-36, delta parareal.py:126 / linalg.py:113-117,
// finiteness linalg.py:74-75). Used by the asynchronous driver and by any
// propagator pair that is not fused into pint_sync_sweep.
//
// One CTA row of the grid per state (blockIdx.y), 16-byte vector accesses,
// per-state max through a fixed-shape block reduction + one atomicMax on the
// order-preserving integer image of a nonnegative double (max is exact, so the
// result is independent of the order CTAs finish).
#include <cuda_runtime.h>

#include "pint_internal.cuh"

template <typename T>
struct Vec2;
template <>
struct Vec2<double> { typedef double2 type; };
template <>
struct Vec2<float> { typedef float4 type; };

__device__ __forceinline__ void atomic_max_nonneg(double *addr, double v) {
  // nonnegative doubles order like their bit patterns as signed 64-bit ints
  atomicMax(reinterpret_cast<unsigned long long *>(addr), (unsigned long long)__double_as_longlong(v));
}

template <typename T>
__device__ __forceinline__ T corr(bool fo, T g, T f, T o) {
  return fo ? f : (g + f) - o;
}

template <typename T>
__global__ void __launch_bounds__(256)
correct_kernel(int64_t dim, const T *__restrict__ gnew, const T *__restrict__ f, const T *__restrict__ gold,
               const T *__restrict__ prev, T *__restrict__ out, const uint8_t *__restrict__ f_only,
               double *__restrict__ delta, int32_t *nonfinite) {
  const int64_t b = blockIdx.y;
  const bool fo = f_only ? (f_only[b] != 0) : false;
  const size_t off = (size_t)b * dim;
  double dm = 0.0;
  bool bad = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < dim; i += (int64_t)gridDim.x * blockDim.x) {
    const T v = corr<T>(fo, fo ? T(0) : gnew[off + i], f[off + i], fo ? T(0) : gold[off + i]);
    out[off + i] = v;
    bad |= !isfinite((double)v);
    if (prev) dm = fmax(dm, fabs((double)v - (double)prev[off + i]));
  }
  __shared__ double red[8];
  __shared__ int bads[8];
  for (int o = 16; o >= 1; o >>= 1) dm = fmax(dm, __shfl_xor_sync(0xffffffffu, dm, o));
  int anybad = __any_sync(0xffffffffu, bad);
  if ((threadIdx.x & 31) == 0) {
    red[threadIdx.x >> 5] = dm;
    bads[threadIdx.x >> 5] = anybad;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    int ab = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      m = fmax(m, red[w]);
      ab |= bads[w];
    }
    if (prev && delta) atomic_max_nonneg(delta + b, m);
    if (ab && nonfinite) atomicExch(nonfinite, 1);
  }
}

__global__ void zero_kernel(double *d, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    d[i] = 0.0;
}

void correct_launch(int dtype, int64_t dim, int64_t nbatch, const void *gnew, const void *f, const void *gold,
                    const void *prev, void *out, const uint8_t *f_only, double *delta, int32_t *nonfinite,
                    cudaStream_t s) {
  if (nbatch <= 0) return;
  if (delta && prev) zero_kernel<<<(unsigned)((nbatch + 255) / 256), 256, 0, s>>>(delta, nbatch);
  int64_t per = (dim + 255) / 256;
  unsigned gx = (unsigned)(per < 148 * 4 ? (per > 0 ? per : 1) : 148 * 4);
  dim3 grid(gx, (unsigned)nbatch);
  if (dtype == PINT_F64)
    correct_kernel<double><<<grid, 256, 0, s>>>(dim, (const double *)gnew, (const double *)f, (const double *)gold,
                                                (const double *)prev, (double *)out, f_only, delta, nonfinite);
  else
    correct_kernel<float><<<grid, 256, 0, s>>>(dim, (const float *)gnew, (const float *)f, (const float *)gold,
                                               (const float *)prev, (float *)out, f_only, delta, nonfinite);
  PINT_CUDA(cudaGetLastError());
}

__global__ void max_reduce_kernel(const double *d, int64_t lo, int64_t hi, double *out) {
  double m = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) m = fmax(m, d[i]);
  for (int o = 16; o >= 1; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ double red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r = fmax(r, red[w]);
    *out = r;
  }
}

void max_reduce_launch(const double *d, int64_t lo, int64_t hi, double *out, cudaStream_t s) {
  max_reduce_kernel<<<1, 256, 0, s>>>(d, lo, hi, out);
  PINT_CUDA(cudaGetLastError());
}

template <typename T>
__global__ void equal_kernel(int64_t dim, const T *__restrict__ a, const T *__restrict__ b, uint8_t *eq) {
  bool ne = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < dim; i += (int64_t)gridDim.x * blockDim.x)
    ne |= !(a[i] == b[i]);
  if (__any_sync(0xffffffffu, ne) && (threadIdx.x & 31) == 0) *eq = 0;
}

__global__ void set_u8(uint8_t *p, uint8_t v) { *p = v; }

void equal_launch(int dtype, int64_t dim, const void *a, const void *b, uint8_t *eq, cudaStream_t s) {
  set_u8<<<1, 1, 0, s>>>(eq, 1);
  int64_t per = (dim + 255) / 256;
  unsigned gx = (unsigned)(per < 148 * 4 ? (per > 0 ? per : 1) : 148 * 4);
  if (dtype == PINT_F64) equal_kernel<double><<<gx, 256, 0, s>>>(dim, (const double *)a, (const double *)b, eq);
  else equal_kernel<float><<<gx, 256, 0, s>>>(dim, (const float *)a, (const float *)b, eq);
  PINT_CUDA(cudaGetLastError());
}
