// Predictor-corrector update with fused convergence norm (reference:
// parareal_update parareal.py:25-36, delta parareal.py:126 / linalg.py:113-117,
// finiteness linalg.py:74-75). Used by the asynchronous driver and by any
// propagator pair that is not fused into pint_sync_sweep.
//
// One CTA row of the grid per state (blockIdx.y); 16-byte vector accesses
// (double2 / float4) when the rows are 16-byte aligned and dim is a multiple
// of the vector width, scalar otherwise; per-state max through a fixed-shape
// block reduction + one atomicMax on the order-preserving integer image of a
// nonnegative double (max is exact, so the result is independent of the
// order CTAs finish).
//
// pint_correct_chain is the per-slice step of the serial coarse chain of the
// generic (non-fused) sweep: the F-only branch is decided on the device from
// the predecessor slice's delta of this sweep (array_equal(fresh, old) <=>
// max|fresh - old| == 0), the G(old) cache row is overwritten in place with
// G(new) (each element is read before it is written, by the same thread),
// and the delta accumulates into a slot the caller zeroed once per sweep —
// one launch per slice instead of four (eq, zero, correct, cache copy).
#include <cuda_runtime.h>

#include "pint_internal.cuh"

__device__ __forceinline__ void atomic_max_nonneg(double *addr, double v) {
  // nonnegative doubles order like their bit patterns as signed 64-bit ints
  atomicMax(reinterpret_cast<unsigned long long *>(addr), (unsigned long long)__double_as_longlong(v));
}

template <typename T>
struct VecOf;
template <>
struct VecOf<double> {
  typedef double2 V;
  static constexpr int W = 2;
};
template <>
struct VecOf<float> {
  typedef float4 V;
  static constexpr int W = 4;
};

template <typename V, typename T, int W>
__device__ __forceinline__ void unpack(const V &v, T (&a)[W]) {
  const T *p = reinterpret_cast<const T *>(&v);
#pragma unroll
  for (int j = 0; j < W; ++j) a[j] = p[j];
}
template <typename V, typename T, int W>
__device__ __forceinline__ V pack(const T (&a)[W]) {
  V v;
  T *p = reinterpret_cast<T *>(&v);
#pragma unroll
  for (int j = 0; j < W; ++j) p[j] = a[j];
  return v;
}

struct CorrArgs {
  int64_t dim;
  const void *gnew, *f, *gold, *prev;
  void *out;
  void *gcache_out;              // chain mode: G(new) written over gold
  const uint8_t *f_only;         // per-state mask (or null)
  const double *fonly_delta;     // chain mode: F-only iff *fonly_delta == 0 (or null)
  double *delta;                 // per-state max |out - prev| (or null)
  int32_t *nonfinite;
  bool zero_delta_first;         // pint_correct: delta slots zeroed by a preceding launch
};

template <typename T, bool VEC>
__global__ void __launch_bounds__(256) correct_kernel(CorrArgs a) {
  using VT = VecOf<T>;
  constexpr int W = VEC ? VT::W : 1;
  const int64_t b = blockIdx.y;
  bool fo = a.f_only ? (a.f_only[b] != 0) : false;
  if (a.fonly_delta) fo = fo || (*a.fonly_delta == 0.0);
  const size_t off = (size_t)b * a.dim;
  const T *gn = (const T *)a.gnew + off, *ff = (const T *)a.f + off, *go = (const T *)a.gold + off;
  const T *pv = a.prev ? (const T *)a.prev + off : nullptr;
  T *out = (T *)a.out + off;
  T *gc = a.gcache_out ? (T *)a.gcache_out + off : nullptr;
  double dm = 0.0;
  bool bad = false;
  const int64_t nv = a.dim / W;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nv; q += (int64_t)gridDim.x * blockDim.x) {
    T g[W], f[W], o[W], v[W], p[W];
    if constexpr (VEC) {
      using V = typename VT::V;
      unpack<V, T, W>(reinterpret_cast<const V *>(ff)[q], f);
      if (!fo || gc) unpack<V, T, W>(reinterpret_cast<const V *>(gn)[q], g);
      if (!fo) unpack<V, T, W>(reinterpret_cast<const V *>(go)[q], o);
      if (pv) unpack<V, T, W>(reinterpret_cast<const V *>(pv)[q], p);
    } else {
      f[0] = ff[q];
      if (!fo || gc) g[0] = gn[q];
      if (!fo) o[0] = go[q];
      if (pv) p[0] = pv[q];
    }
#pragma unroll
    for (int j = 0; j < W; ++j) {
      v[j] = fo ? f[j] : (g[j] + f[j]) - o[j];  // left-to-right order of parareal.py:36
      bad |= !isfinite((double)v[j]);
      if (pv) dm = fmax(dm, fabs((double)v[j] - (double)p[j]));
    }
    if constexpr (VEC) {
      using V = typename VT::V;
      reinterpret_cast<V *>(out)[q] = pack<V, T, W>(v);
      if (gc) reinterpret_cast<V *>(gc)[q] = pack<V, T, W>(g);
    } else {
      out[q] = v[0];
      if (gc) gc[q] = g[0];
    }
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
    if (pv && a.delta) atomic_max_nonneg(a.delta + b, m);
    if (ab && a.nonfinite) atomicExch(a.nonfinite, 1);
  }
}

__global__ void zero_kernel(double *d, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    d[i] = 0.0;
}

namespace {

bool aligned16(const void *p) { return p == nullptr || ((uintptr_t)p & 15u) == 0; }

template <typename T>
void launch_correct(const CorrArgs &a, int64_t nbatch, cudaStream_t s) {
  constexpr int W = VecOf<T>::W;
  const bool vec = a.dim % W == 0 && aligned16(a.gnew) && aligned16(a.f) && aligned16(a.gold) &&
                   aligned16(a.prev) && aligned16(a.out) && aligned16(a.gcache_out);
  const int64_t items = vec ? a.dim / W : a.dim;
  int64_t per = (items + 255) / 256;
  unsigned gx = (unsigned)(per < 148 * 4 ? (per > 0 ? per : 1) : 148 * 4);
  dim3 grid(gx, (unsigned)nbatch);
  if (vec) correct_kernel<T, true><<<grid, 256, 0, s>>>(a);
  else correct_kernel<T, false><<<grid, 256, 0, s>>>(a);
}

}  // namespace

void correct_launch(int dtype, int64_t dim, int64_t nbatch, const void *gnew, const void *f, const void *gold,
                    const void *prev, void *out, const uint8_t *f_only, double *delta, int32_t *nonfinite,
                    cudaStream_t s) {
  if (nbatch <= 0) return;
  if (delta && prev) zero_kernel<<<(unsigned)((nbatch + 255) / 256), 256, 0, s>>>(delta, nbatch);
  CorrArgs a{dim, gnew, f, gold, prev, out, nullptr, f_only, nullptr, delta, nonfinite, true};
  if (dtype == PINT_F64) launch_correct<double>(a, nbatch, s);
  else launch_correct<float>(a, nbatch, s);
  PINT_CUDA(cudaGetLastError());
}

void correct_chain_launch(int dtype, int64_t dim, const void *gnew, const void *f, void *gcache, const void *prev,
                          void *out, const uint8_t *f_only, const double *fonly_delta, double *delta,
                          int32_t *nonfinite, cudaStream_t s) {
  CorrArgs a{dim, gnew, f, gcache, prev, out, gcache, f_only, fonly_delta, delta, nonfinite, false};
  if (dtype == PINT_F64) launch_correct<double>(a, 1, s);
  else launch_correct<float>(a, 1, s);
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
