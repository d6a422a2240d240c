// Temporally blocked explicit heat stencil, 2-D (5-point) — the fine
// propagator of BASELINE C3 (reference route: fine_from_onestep(
// AffinePropagator(I + dt A, dt c, 1), S), model.py:147-154).
//
// 2.5-D wavefront: a CTA owns an x-tile (plus a halo of S columns per side)
// and a chunk of rows (plus S halo rows), and sweeps the rows once. It carries
// S time levels in registers: when input row y arrives, level 1 is advanced at
// row y-1, level 2 at row y-2, ..., level S at row y-S (each level keeps its
// last three rows per column in registers). x-neighbours of a level's
// previous row come from shared memory written one row earlier (double
// buffered: one barrier per row). Each thread owns CPT = 2 adjacent columns,
// so only the outer neighbours cost a shared-memory read. HBM sees one read
// and one write of the state per pass of S steps: 2*sizeof(T)/S bytes per
// grid-point update. Zero Dirichlet: values outside the domain are 0 at every
// level. Arithmetic per point is the same expression everywhere (batch ==
// single, any tiling).
#include <cuda_runtime.h>

#include <algorithm>

#include "pint_internal.cuh"

namespace {

constexpr int SMAX2 = 8;                 // time levels per pass
constexpr int CPT2 = 2;                  // columns per thread
constexpr int BX2 = 256;                 // output columns per tile
constexpr int W2 = BX2 + 2 * SMAX2;      // loaded columns per tile
constexpr int WT2 = W2 / CPT2;           // threads per CTA (136)
constexpr int YC2 = 128;                 // output rows per chunk

template <typename T, int S>
__global__ void __launch_bounds__(WT2)
fe2d_wave(const T *__restrict__ in, T *__restrict__ out, int64_t stride, int nx, int ny, T r) {
  __shared__ T sm[2][S][W2 + 2];
  const int tid = threadIdx.x;
  const int x0 = blockIdx.x * BX2 - S;  // first loaded column (halo S)
  const int y0 = blockIdx.y * YC2;
  const T *src = in + (int64_t)blockIdx.z * stride;
  T *dst = out + (int64_t)blockIdx.z * stride;
  const int cx = x0 + CPT2 * tid;
  bool colin[CPT2], colout[CPT2];
#pragma unroll
  for (int c = 0; c < CPT2; ++c) {
    colin[c] = cx + c >= 0 && cx + c < nx;
    const int lc = CPT2 * tid + c;  // local column
    colout[c] = colin[c] && lc >= S && lc < S + BX2;
  }
  for (int i = tid; i < 2 * S * (W2 + 2); i += WT2) (&sm[0][0][0])[i] = T(0);
  T cur[S][CPT2], prv[S][CPT2], pp[S][CPT2];
#pragma unroll
  for (int L = 0; L < S; ++L)
#pragma unroll
    for (int c = 0; c < CPT2; ++c) cur[L][c] = prv[L][c] = pp[L][c] = T(0);
  __syncthreads();
  const T four = T(4);
  const int ys = y0 - S, ye = min(y0 + YC2, ny) - 1 + S;
  int par = 0;
  for (int yy = ys; yy <= ye; ++yy, par ^= 1) {
    // level 0: the input row yy
    const bool rowin = yy >= 0 && yy < ny;
#pragma unroll
    for (int c = 0; c < CPT2; ++c) cur[0][c] = (rowin && colin[c]) ? __ldg(src + (int64_t)yy * nx + cx + c) : T(0);
#pragma unroll
    for (int c = 0; c < CPT2; ++c) sm[par][0][1 + CPT2 * tid + c] = cur[0][c];
    // levels 1..S: level L+1 at row yy-L-1 from level L rows (pp, prv, cur)
#pragma unroll
    for (int L = 0; L < S; ++L) {
      const int yr = yy - L - 1;
      const bool rin = yr >= 0 && yr < ny;
      const T left = sm[par ^ 1][L][CPT2 * tid];
      const T right = sm[par ^ 1][L][1 + CPT2 * tid + CPT2];
      T v[CPT2];
#pragma unroll
      for (int c = 0; c < CPT2; ++c) {
        const T l = (c == 0) ? left : prv[L][c - 1];
        const T rr = (c == CPT2 - 1) ? right : prv[L][c + 1];
        const T ctr = prv[L][c];
        const T nb = (l + rr) + (pp[L][c] + cur[L][c]);
        v[c] = (rin && colin[c]) ? ctr + r * (nb - four * ctr) : T(0);
      }
      if (L + 1 < S) {
#pragma unroll
        for (int c = 0; c < CPT2; ++c) {
          cur[L + 1][c] = v[c];
          sm[par][L + 1][1 + CPT2 * tid + c] = v[c];
        }
      } else if (yr >= y0 && yr < y0 + YC2 && rin) {
#pragma unroll
        for (int c = 0; c < CPT2; ++c)
          if (colout[c]) dst[(int64_t)yr * nx + cx + c] = v[c];
      }
    }
#pragma unroll
    for (int L = 0; L < S; ++L)
#pragma unroll
      for (int c = 0; c < CPT2; ++c) {
        pp[L][c] = prv[L][c];
        prv[L][c] = cur[L][c];
      }
    __syncthreads();
  }
}

template <typename T, int S>
void launch2(const T *in, T *out, int64_t nb, int64_t stride, int nx, int ny, T r, cudaStream_t st) {
  const unsigned tx = (unsigned)((nx + BX2 - 1) / BX2), ty = (unsigned)((ny + YC2 - 1) / YC2);
  for (int64_t b0 = 0; b0 < nb; b0 += 65535) {
    const unsigned n = (unsigned)std::min<int64_t>(65535, nb - b0);
    fe2d_wave<T, S><<<dim3(tx, ty, n), WT2, 0, st>>>(in + b0 * stride, out + b0 * stride, stride, nx, ny, r);
  }
  PINT_CUDA(cudaGetLastError());
}

template <typename T>
void pass2(int s, const T *in, T *out, int64_t nb, int64_t stride, int nx, int ny, T r, cudaStream_t st) {
  switch (s) {
    case 1: launch2<T, 1>(in, out, nb, stride, nx, ny, r, st); break;
    case 2: launch2<T, 2>(in, out, nb, stride, nx, ny, r, st); break;
    case 3: launch2<T, 3>(in, out, nb, stride, nx, ny, r, st); break;
    case 4: launch2<T, 4>(in, out, nb, stride, nx, ny, r, st); break;
    case 5: launch2<T, 5>(in, out, nb, stride, nx, ny, r, st); break;
    case 6: launch2<T, 6>(in, out, nb, stride, nx, ny, r, st); break;
    case 7: launch2<T, 7>(in, out, nb, stride, nx, ny, r, st); break;
    default: launch2<T, 8>(in, out, nb, stride, nx, ny, r, st); break;
  }
}

}  // namespace

// S steps of the 2-D explicit stencil as ceil(S / 8) wavefront passes,
// ping-ponging between out and scratch so the last pass writes out.
template <typename T>
void fe2d_wave_apply(const pint_op *op, const T *in, T *out, T *scratch, int64_t nb, int64_t stride,
                     cudaStream_t st) {
  const int64_t S = op->desc.steps;
  const int64_t npass = (S + SMAX2 - 1) / SMAX2;
  const T r = (T)(op->dt / (op->desc.h * op->desc.h));
  int64_t done = 0;
  for (int64_t pass = 0; pass < npass; ++pass) {
    const int s = (int)std::min<int64_t>(SMAX2, S - done);
    const T *src = pass == 0 ? in : (((npass - pass) % 2 == 0) ? out : scratch);
    T *dstp = ((npass - 1 - pass) % 2 == 0) ? out : scratch;
    pass2<T>(s, src, dstp, nb, stride, (int)op->nx, (int)op->ny, r, st);
    done += s;
  }
}

template void fe2d_wave_apply<float>(const pint_op *, const float *, float *, float *, int64_t, int64_t,
                                     cudaStream_t);
template void fe2d_wave_apply<double>(const pint_op *, const double *, double *, double *, int64_t, int64_t,
                                      cudaStream_t);

// --------------------------------------------------------------- 3-D (7-point)
// Same wavefront with z as the sweep axis: a CTA owns an xy tile (plus S
// halo cells per side) of z-columns and a chunk of z planes; each thread owns
// CPT3 x-adjacent columns and carries S levels x 3 planes in registers; the
// xy neighbours of a level's previous plane come from a double-buffered
// shared tile. HBM traffic 2*sizeof(T)/S bytes per update; the halo costs
// (BX3+2S)(BY3+2S)/(BX3 BY3) redundant updates.
namespace {

constexpr int SMAX3 = 4;
constexpr int CPT3 = 2;
constexpr int BX3 = 64, BY3 = 16;
constexpr int WX3 = BX3 + 2 * SMAX3, WY3 = BY3 + 2 * SMAX3;  // 72 x 24 loaded columns
constexpr int TX3 = WX3 / CPT3;                               // 36 threads in x
constexpr int ZC3 = 64;                                        // output planes per chunk

template <typename T, int S>
__global__ void __launch_bounds__(TX3 *WY3)
fe3d_wave(const T *__restrict__ in, T *__restrict__ out, int64_t stride, int nx, int ny, int nz, T r, int tiles_x) {
  extern __shared__ __align__(16) unsigned char smraw3[];
  T(*sm)[S][WY3 + 2][WX3 + 2] = reinterpret_cast<T(*)[S][WY3 + 2][WX3 + 2]>(smraw3);
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int tid = ty * TX3 + tx;
  const int bx = blockIdx.x % tiles_x, by = blockIdx.x / tiles_x;
  const int x0 = bx * BX3 - S, y0 = by * BY3 - S, z0 = blockIdx.y * ZC3;
  const int64_t plane = (int64_t)nx * ny;
  const T *src = in + (int64_t)blockIdx.z * stride;
  T *dst = out + (int64_t)blockIdx.z * stride;
  const int cx = x0 + CPT3 * tx, cy = y0 + ty;
  bool colin[CPT3], colout[CPT3];
#pragma unroll
  for (int c = 0; c < CPT3; ++c) {
    colin[c] = cx + c >= 0 && cx + c < nx && cy >= 0 && cy < ny;
    const int lx = CPT3 * tx + c;
    colout[c] = colin[c] && lx >= S && lx < S + BX3 && ty >= S && ty < S + BY3;
  }
  for (int i = tid; i < 2 * S * (WY3 + 2) * (WX3 + 2); i += TX3 * WY3) (&sm[0][0][0][0])[i] = T(0);
  T cur[S][CPT3], prv[S][CPT3], pp[S][CPT3];
#pragma unroll
  for (int L = 0; L < S; ++L)
#pragma unroll
    for (int c = 0; c < CPT3; ++c) cur[L][c] = prv[L][c] = pp[L][c] = T(0);
  __syncthreads();
  const T six = T(6);
  const int zs = z0 - S, ze = min(z0 + ZC3, nz) - 1 + S;
  const int sx = 1 + CPT3 * tx, sy = 1 + ty;
  int par = 0;
  for (int zz = zs; zz <= ze; ++zz, par ^= 1) {
    const bool pin = zz >= 0 && zz < nz;
#pragma unroll
    for (int c = 0; c < CPT3; ++c) {
      cur[0][c] = (pin && colin[c]) ? __ldg(src + (int64_t)zz * plane + (int64_t)cy * nx + cx + c) : T(0);
      sm[par][0][sy][sx + c] = cur[0][c];
    }
#pragma unroll
    for (int L = 0; L < S; ++L) {
      const int zr = zz - L - 1;
      const bool rin = zr >= 0 && zr < nz;
      const T left = sm[par ^ 1][L][sy][sx - 1];
      const T right = sm[par ^ 1][L][sy][sx + CPT3];
      T v[CPT3];
#pragma unroll
      for (int c = 0; c < CPT3; ++c) {
        const T ctr = prv[L][c];
        const T xl = (c == 0) ? left : prv[L][c - 1];
        const T xr = (c == CPT3 - 1) ? right : prv[L][c + 1];
        const T yl = sm[par ^ 1][L][sy - 1][sx + c];
        const T yr = sm[par ^ 1][L][sy + 1][sx + c];
        const T nb = ((xl + xr) + (yl + yr)) + (pp[L][c] + cur[L][c]);
        v[c] = (rin && colin[c]) ? ctr + r * (nb - six * ctr) : T(0);
      }
      if (L + 1 < S) {
#pragma unroll
        for (int c = 0; c < CPT3; ++c) {
          cur[L + 1][c] = v[c];
          sm[par][L + 1][sy][sx + c] = v[c];
        }
      } else if (zr >= z0 && zr < z0 + ZC3 && rin) {
#pragma unroll
        for (int c = 0; c < CPT3; ++c)
          if (colout[c]) dst[(int64_t)zr * plane + (int64_t)cy * nx + cx + c] = v[c];
      }
    }
#pragma unroll
    for (int L = 0; L < S; ++L)
#pragma unroll
      for (int c = 0; c < CPT3; ++c) {
        pp[L][c] = prv[L][c];
        prv[L][c] = cur[L][c];
      }
    __syncthreads();
  }
}

template <typename T, int S>
void launch3(const T *in, T *out, int64_t nb, int64_t stride, int nx, int ny, int nz, T r, cudaStream_t st) {
  const int tiles_x = (nx + BX3 - 1) / BX3, tiles_y = (ny + BY3 - 1) / BY3;
  const unsigned tz = (unsigned)((nz + ZC3 - 1) / ZC3);
  const size_t smem = sizeof(T) * 2 * S * (WY3 + 2) * (WX3 + 2);
  PINT_CUDA(cudaFuncSetAttribute(fe3d_wave<T, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  for (int64_t b0 = 0; b0 < nb; b0 += 65535) {
    const unsigned n = (unsigned)std::min<int64_t>(65535, nb - b0);
    fe3d_wave<T, S><<<dim3((unsigned)(tiles_x * tiles_y), tz, n), dim3(TX3, WY3), smem, st>>>(
        in + b0 * stride, out + b0 * stride, stride, nx, ny, nz, r, tiles_x);
  }
  PINT_CUDA(cudaGetLastError());
}

template <typename T>
void pass3(int s, const T *in, T *out, int64_t nb, int64_t stride, int nx, int ny, int nz, T r, cudaStream_t st) {
  switch (s) {
    case 1: launch3<T, 1>(in, out, nb, stride, nx, ny, nz, r, st); break;
    case 2: launch3<T, 2>(in, out, nb, stride, nx, ny, nz, r, st); break;
    case 3: launch3<T, 3>(in, out, nb, stride, nx, ny, nz, r, st); break;
    default: launch3<T, 4>(in, out, nb, stride, nx, ny, nz, r, st); break;
  }
}

}  // namespace

template <typename T>
void fe3d_wave_apply(const pint_op *op, const T *in, T *out, T *scratch, int64_t nb, int64_t stride,
                     cudaStream_t st) {
  const int64_t S = op->desc.steps;
  const int64_t npass = (S + SMAX3 - 1) / SMAX3;
  const T r = (T)(op->dt / (op->desc.h * op->desc.h));
  int64_t done = 0;
  for (int64_t pass = 0; pass < npass; ++pass) {
    const int s = (int)std::min<int64_t>(SMAX3, S - done);
    const T *src = pass == 0 ? in : (((npass - pass) % 2 == 0) ? out : scratch);
    T *dstp = ((npass - 1 - pass) % 2 == 0) ? out : scratch;
    pass3<T>(s, src, dstp, nb, stride, (int)op->nx, (int)op->ny, (int)op->nz, r, st);
    done += s;
  }
}

template void fe3d_wave_apply<float>(const pint_op *, const float *, float *, float *, int64_t, int64_t,
                                     cudaStream_t);
template void fe3d_wave_apply<double>(const pint_op *, const double *, double *, double *, int64_t, int64_t,
                                      cudaStream_t);
