// Explicit (forward-Euler) fine propagator for the zero-Dirichlet heat
// operator on 1/2/3-D grids: u+ = u + r * (sum of 2*d neighbours - 2 d u),
// r = dt / h^2, applied `steps` times per slice (reference route:
// fine_from_onestep(AffinePropagator(I + dt A, dt c, 1), S), model.py:147-154;
// the dense (I + dt A) is never formed here).
//
// Temporal blocking: one CTA loads a box of the slice plus a halo of `s`
// cells into shared memory, advances it `s` steps there (the valid region
// shrinks by one cell per step), and writes back the interior box. HBM
// traffic per fused pass is one read and one write of the state, so the
// traffic per grid-point update is 2*sizeof(T)/s. Points outside the domain
// are the Dirichlet zeros and stay zero.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "pint_internal.cuh"

namespace {

template <typename T>
struct StencilArgs {
  const T *in;
  T *out;
  int64_t stride;  // elements between slices
  int nx, ny, nz;  // nz = 1 in 2-D, ny = nz = 1 in 1-D
  T r;
  int s;           // fused steps in this pass
};

// Box sizes (output cells per CTA) per dimension.
template <int DIM>
struct Box;
template <>
struct Box<1> { static constexpr int X = 1024, Y = 1, Z = 1; };
template <>
struct Box<2> { static constexpr int X = 64, Y = 32, Z = 1; };
template <>
struct Box<3> { static constexpr int X = 32, Y = 16, Z = 8; };

template <typename T, int DIM>
__global__ void __launch_bounds__(512)
fe_block_kernel(const StencilArgs<T> a) {
  extern __shared__ unsigned char smem_raw[];
  T *buf0 = reinterpret_cast<T *>(smem_raw);
  const int s = a.s;
  const int hx = s, hy = DIM >= 2 ? s : 0, hz = DIM >= 3 ? s : 0;
  const int LX = Box<DIM>::X + 2 * hx, LY = Box<DIM>::Y + 2 * hy, LZ = Box<DIM>::Z + 2 * hz;
  const int L = LX * LY * LZ;
  T *buf1 = buf0 + L;
  const int tiles_x = (a.nx + Box<DIM>::X - 1) / Box<DIM>::X;
  const int tiles_y = (a.ny + Box<DIM>::Y - 1) / Box<DIM>::Y;
  const int tile = blockIdx.x;
  const int bx = tile % tiles_x;
  const int by = (tile / tiles_x) % tiles_y;
  const int bz = tile / (tiles_x * tiles_y);
  const int64_t slice = blockIdx.y;
  const T *in = a.in + slice * a.stride;
  T *out = a.out + slice * a.stride;
  const int x0 = bx * Box<DIM>::X - hx, y0 = by * Box<DIM>::Y - hy, z0 = bz * Box<DIM>::Z - hz;
  for (int i = threadIdx.x; i < L; i += blockDim.x) {
    const int lx = i % LX, ly = (i / LX) % LY, lz = i / (LX * LY);
    const int gx = x0 + lx, gy = y0 + ly, gz = z0 + lz;
    T v = T(0);
    if (gx >= 0 && gx < a.nx && gy >= 0 && gy < a.ny && gz >= 0 && gz < a.nz)
      v = in[((int64_t)gz * a.ny + gy) * a.nx + gx];
    buf0[i] = v;
  }
  __syncthreads();
  const T c = T(2 * DIM);
  T *src = buf0, *dst = buf1;
  for (int step = 0; step < s; ++step) {
    for (int i = threadIdx.x; i < L; i += blockDim.x) {
      const int lx = i % LX, ly = (i / LX) % LY, lz = i / (LX * LY);
      const int gx = x0 + lx, gy = y0 + ly, gz = z0 + lz;
      const bool inside = gx >= 0 && gx < a.nx && gy >= 0 && gy < a.ny && gz >= 0 && gz < a.nz;
      const bool interior = lx > 0 && lx < LX - 1 && (DIM < 2 || (ly > 0 && ly < LY - 1)) &&
                            (DIM < 3 || (lz > 0 && lz < LZ - 1));
      T v = T(0);
      if (inside && interior) {
        const T u = src[i];
        T nb = src[i - 1] + src[i + 1];
        if (DIM >= 2) nb += src[i - LX] + src[i + LX];
        if (DIM >= 3) nb += src[i - LX * LY] + src[i + LX * LY];
        v = fma(a.r, fma(-c, u, nb), u);  // pinned expression (oracle/stencil_nd.c)
      }
      dst[i] = v;
    }
    __syncthreads();
    T *t = src;
    src = dst;
    dst = t;
  }
  for (int i = threadIdx.x; i < Box<DIM>::X * Box<DIM>::Y * Box<DIM>::Z; i += blockDim.x) {
    const int ox = i % Box<DIM>::X, oy = (i / Box<DIM>::X) % Box<DIM>::Y, oz = i / (Box<DIM>::X * Box<DIM>::Y);
    const int gx = bx * Box<DIM>::X + ox, gy = by * Box<DIM>::Y + oy, gz = bz * Box<DIM>::Z + oz;
    if (gx < a.nx && gy < a.ny && gz < a.nz) {
      const int li = ((oz + hz) * LY + (oy + hy)) * LX + (ox + hx);
      out[((int64_t)gz * a.ny + gy) * a.nx + gx] = src[li];
    }
  }
}

template <int DIM>
int fused_steps(int esz) {
  // halo width per pass, bounded by shared memory (two buffers)
  const int cap = 200 * 1024;
  int best = 1;
  for (int s = 1; s <= 16; ++s) {
    const int LX = Box<DIM>::X + 2 * s;
    const int LY = Box<DIM>::Y + (DIM >= 2 ? 2 * s : 0);
    const int LZ = Box<DIM>::Z + (DIM >= 3 ? 2 * s : 0);
    if ((int64_t)2 * LX * LY * LZ * esz <= cap) best = s;
  }
  const int maxs = DIM == 1 ? 16 : (DIM == 2 ? 8 : 2);
  return std::min(best, maxs);
}

template <typename T, int DIM>
void fe_launch(const pint_op *op, const T *in, T *out, T *scratch, int64_t nbatch, int64_t stride,
               cudaStream_t st) {
  const int64_t S = op->desc.steps;
  const int sblk = fused_steps<DIM>((int)sizeof(T));
  const int64_t npass = (S + sblk - 1) / sblk;
  StencilArgs<T> a;
  a.stride = stride;
  a.nx = (int)op->nx;
  a.ny = (int)op->ny;
  a.nz = (int)op->nz;
  const double h = op->desc.ndim == 1 ? 0.0 : op->desc.h;
  (void)h;
  a.r = (T)(op->dt / (op->desc.h * op->desc.h));
  const int tiles = ((a.nx + Box<DIM>::X - 1) / Box<DIM>::X) * ((a.ny + Box<DIM>::Y - 1) / Box<DIM>::Y) *
                    ((a.nz + Box<DIM>::Z - 1) / Box<DIM>::Z);
  auto kern = fe_block_kernel<T, DIM>;
  int64_t done = 0;
  for (int64_t pass = 0; pass < npass; ++pass) {
    const int s = (int)std::min<int64_t>(sblk, S - done);
    const T *src = pass == 0 ? in : (((npass - pass) % 2 == 0) ? out : scratch);
    T *dst = ((npass - 1 - pass) % 2 == 0) ? out : scratch;
    a.in = src;
    a.out = dst;
    a.s = s;
    const int LX = Box<DIM>::X + 2 * s, LY = Box<DIM>::Y + (DIM >= 2 ? 2 * s : 0),
              LZ = Box<DIM>::Z + (DIM >= 3 ? 2 * s : 0);
    const size_t smem = (size_t)2 * LX * LY * LZ * sizeof(T);
    PINT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    for (int64_t b0 = 0; b0 < nbatch; b0 += 65535) {
      const int64_t nb = std::min<int64_t>(65535, nbatch - b0);
      StencilArgs<T> ab = a;
      ab.in = src + b0 * stride;
      ab.out = dst + b0 * stride;
      kern<<<dim3((unsigned)tiles, (unsigned)nb), 512, smem, st>>>(ab);
      PINT_CUDA(cudaGetLastError());
    }
    done += s;
  }
}

}  // namespace

void stencil_setup(pint_op *op) {
  const pint_op_desc &d = op->desc;
  if (d.ndim == 1) {
    // 1-D explicit Euler on the zero-Dirichlet Laplacian needs h
    if (!(d.h > 0.0)) pint_throw(PINT_EARG, "grid spacing must be positive");
    op->nx = d.shape[0];
    op->ny = op->nz = 1;
  }
  op->dt = d.span / (double)d.steps;
  const int64_t maxint = 0x7fffffff;
  if (op->nx > maxint || op->ny > maxint || op->nz > maxint) pint_throw(PINT_EDIM, "grid too large");
}

template <typename T>
void fe2d_wave_apply(const pint_op *op, const T *in, T *out, T *scratch, int64_t nb, int64_t stride, cudaStream_t st);
template <typename T>
void fe3d_wave_apply(const pint_op *op, const T *in, T *out, T *scratch, int64_t nb, int64_t stride, cudaStream_t st);
template <typename T>
bool fe3d_tile_apply(int variant, const pint_op *op, const T *in, T *out, T *scratch, int64_t nb, int64_t stride,
                     cudaStream_t st);
int fe3d_tile_default(int esz);

void stencil_apply_batch(pint_op *op, const void *in, void *out, int64_t nbatch, int64_t stride, cudaStream_t s) {
  const int64_t S = op->desc.steps;
  const int nd = op->desc.ndim;
  const int esz = op->desc.dtype == PINT_F64 ? 8 : 4;
  int sblk = nd == 1 ? fused_steps<1>(esz) : (nd == 2 ? fused_steps<2>(esz) : fused_steps<3>(esz));
  const bool v1 = getenv("PINT_STENCIL_V1") && atoi(getenv("PINT_STENCIL_V1"));
  const bool wave2 = nd == 2 && !v1, wave3 = nd == 3 && !v1;
  if (wave2) sblk = 8;
  int v3 = 0;
  if (wave3) {
    // 3-D tiling variant (stencil3d.cu); PINT_FE3D_VARIANT overrides for measurement, 0 = fe3d_wave
    v3 = fe3d_tile_default(esz);
    if (const char *e = getenv("PINT_FE3D_VARIANT")) v3 = atoi(e);
    sblk = v3 > 0 ? 1 : 4;
  }
  void *scratch = nullptr;
  if (S > sblk) {
    const size_t need = (size_t)nbatch * stride * esz;
    if (op->cg_work_bytes < need) {
      if (op->cg_work) cudaFree(op->cg_work);
      op->cg_work = nullptr;
      op->cg_work_bytes = 0;
      PINT_CUDA(cudaMalloc(&op->cg_work, need));
      op->cg_work_bytes = need;
    }
    scratch = op->cg_work;
  }
  if (wave3 && v3 > 0) {
    const bool ok = op->desc.dtype == PINT_F64
                        ? fe3d_tile_apply<double>(v3, op, (const double *)in, (double *)out, (double *)scratch,
                                                  nbatch, stride, s)
                        : fe3d_tile_apply<float>(v3, op, (const float *)in, (float *)out, (float *)scratch, nbatch,
                                                 stride, s);
    if (!ok) pint_throw(PINT_EARG, "unknown PINT_FE3D_VARIANT");
    return;
  }
  if (wave3) {
    if (op->desc.dtype == PINT_F64)
      fe3d_wave_apply<double>(op, (const double *)in, (double *)out, (double *)scratch, nbatch, stride, s);
    else
      fe3d_wave_apply<float>(op, (const float *)in, (float *)out, (float *)scratch, nbatch, stride, s);
    return;
  }
  if (wave2) {
    if (op->desc.dtype == PINT_F64)
      fe2d_wave_apply<double>(op, (const double *)in, (double *)out, (double *)scratch, nbatch, stride, s);
    else
      fe2d_wave_apply<float>(op, (const float *)in, (float *)out, (float *)scratch, nbatch, stride, s);
    return;
  }
  if (op->desc.dtype == PINT_F64) {
    if (nd == 1) fe_launch<double, 1>(op, (const double *)in, (double *)out, (double *)scratch, nbatch, stride, s);
    else if (nd == 2) fe_launch<double, 2>(op, (const double *)in, (double *)out, (double *)scratch, nbatch, stride, s);
    else fe_launch<double, 3>(op, (const double *)in, (double *)out, (double *)scratch, nbatch, stride, s);
  } else {
    if (nd == 1) fe_launch<float, 1>(op, (const float *)in, (float *)out, (float *)scratch, nbatch, stride, s);
    else if (nd == 2) fe_launch<float, 2>(op, (const float *)in, (float *)out, (float *)scratch, nbatch, stride, s);
    else fe_launch<float, 3>(op, (const float *)in, (float *)out, (float *)scratch, nbatch, stride, s);
  }
}
