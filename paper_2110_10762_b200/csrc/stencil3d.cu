// Temporally blocked explicit 7-point heat stencil, 3-D — the fine propagator
// of BASELINE C4/C5 (reference route: fine_from_onestep(AffinePropagator(
// I + dt A, dt c, 1), S), model.py:147-154), second-generation tiling.
//
// 2.5-D wavefront with z as the sweep axis (as fe3d_wave in stencil_wave.cu):
// a CTA owns an xy tile of z-columns, 32*CPT columns x RW rows including S
// halo cells per side, and a chunk of ZC planes. When input plane z arrives,
// level 1 is advanced at plane z-1, ..., level S at plane z-S; each level
// keeps three planes per column in registers. Warp w owns tile row w and each
// lane CPT adjacent columns: x-neighbours by warp shuffle (lane +-1),
// y-neighbours from a double-buffered shared tile written one plane earlier
// (one vector load per neighbour row), z-neighbours from registers. One
// barrier per plane. HBM traffic 2*sizeof(T)/S bytes per update.
//
// What is new against fe3d_wave: (1) the steady state (every level's plane
// inside the domain) runs six planes per loop trip, the period of the
// three-plane register rotation times the two shared-buffer parities, so the
// rotation is register renaming instead of moves; (2) input prefetch and
// output addresses advance by pointer increments; (3) tiles that lie wholly
// inside the domain skip the Dirichlet mask; (4) the tile shape is a template
// (CPT = 2 or 4 columns per lane, RW rows, S levels) so the halo redundancy
// 32 CPT RW / ((32 CPT - 2S)(RW - 2S)) can be traded against registers.
// The per-point arithmetic is the same expression in every variant,
//   nb = ((x- + x+) + (y- + y+)) + (z- + z+);  v = fma(r, fma(-6, c, nb), c),
// so every tiling (and fe3d_wave) produces bitwise identical results.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "pint_internal.cuh"

namespace {

constexpr int ZC = 128;  // output planes per chunk

template <typename T, int CPT>
struct Vec;
template <>
struct Vec<float, 2> { using V = float2; };
template <>
struct Vec<float, 4> { using V = float4; };
template <>
struct Vec<double, 2> { using V = double2; };

template <int CPT, typename V, typename T>
__device__ __forceinline__ void vload(const V &v, T (&o)[CPT]) {
  if constexpr (CPT == 2) {
    o[0] = v.x;
    o[1] = v.y;
  } else {
    o[0] = v.x;
    o[1] = v.y;
    o[2] = v.z;
    o[3] = v.w;
  }
}
template <int CPT, typename V, typename T>
__device__ __forceinline__ V vmake(const T (&a)[CPT]) {
  if constexpr (CPT == 2) return V{a[0], a[1]};
  else return V{a[0], a[1], a[2], a[3]};
}

// packed FP32 pairs (FADD2 / FFMA2 / FMUL2 on sm_100a); same per-element
// IEEE result as the scalar expression
__device__ __forceinline__ unsigned long long pk(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void upk(unsigned long long v, float &a, float &b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ unsigned long long add2(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ unsigned long long fma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ unsigned long long mul2(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

// One level update of CPT columns: v = fma(r, fma(-6, c, nb), c), masked.
template <typename T, int CPT, bool MASK>
__device__ __forceinline__ void level_update(const T (&p)[CPT], T left, T right, const T (&up)[CPT],
                                             const T (&dn)[CPT], const T (&zm)[CPT], const T (&zp)[CPT], T r,
                                             const T (&m)[CPT], T (&v)[CPT]) {
  if constexpr (sizeof(T) == 4) {
#pragma unroll
    for (int j = 0; j < CPT; j += 2) {
      const float xl0 = j == 0 ? left : p[j - 1], xr1 = j + 2 == CPT ? right : p[j + 2];
      const unsigned long long ctr = pk(p[j], p[j + 1]);
      // x-pair sums (xl0 + p[j+1], p[j] + xr1) as (xl0, xr1) + (p[j+1], p[j]): the swapped
      // halves are an operand swizzle and the shuffles land in one register pair (no moves);
      // per element the same IEEE sum as xl + xr
      const unsigned long long nb =
          add2(add2(add2(pk(xl0, xr1), pk(p[j + 1], p[j])), add2(pk(up[j], up[j + 1]), pk(dn[j], dn[j + 1]))),
               add2(pk(zm[j], zm[j + 1]), pk(zp[j], zp[j + 1])));
      const unsigned long long t = fma2(pk(-6.0f, -6.0f), ctr, nb);
      unsigned long long vv = fma2(pk(r, r), t, ctr);
      if (MASK) vv = mul2(vv, pk(m[j], m[j + 1]));
      upk(vv, v[j], v[j + 1]);
    }
  } else {
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const T xl = c == 0 ? left : p[c - 1], xr = c == CPT - 1 ? right : p[c + 1];
      const T nb = ((xl + xr) + (up[c] + dn[c])) + (zm[c] + zp[c]);
      const T t = fma(T(-6), p[c], nb);
      v[c] = fma(r, t, p[c]);
      if (MASK) v[c] *= m[c];
    }
  }
}

struct PlaneCtx {
  int w;            // warp = strip index
  int zz;           // input plane arriving
  int z0, nz, ze;   // chunk start, domain depth, last input plane of the sweep
};

// Shared exchange rows of one level: the top and bottom row of every warp's
// strip (one array when a strip is one row).
template <typename T, int S, int NW, int RPT, int CPT>
struct Xchg {
  using V = typename Vec<T, CPT>::V;
  V top[2][S][NW][32];
  V bot[RPT > 1 ? 2 : 1][RPT > 1 ? S : 1][RPT > 1 ? NW : 1][32];
  __device__ __forceinline__ V &tp(int par, int L, int w, int lane) { return top[par][L][w][lane]; }
  __device__ __forceinline__ V &bt(int par, int L, int w, int lane) {
    if constexpr (RPT > 1) return bot[par][L][w][lane];
    else return top[par][L][w][lane];
  }
};

// One plane of the wavefront for a strip of RPT rows x CPT columns per lane.
// EDGE: some level's plane may lie outside the domain (per-level plane mask);
// PAR: shared-buffer parity (compile time).
template <typename T, int S, int NW, int RPT, int CPT, bool EDGE, bool MASK, int PAR>
__device__ __forceinline__ void plane(T (&cur)[S][RPT][CPT], T (&prv)[S][RPT][CPT], T (&pp)[S][RPT][CPT],
                                      T (&pre)[RPT][CPT], Xchg<T, S, NW, RPT, CPT> &X, const PlaneCtx &q,
                                      const T (&m)[RPT][CPT], const bool (&colout)[RPT][CPT],
                                      const bool (&colin)[RPT][CPT], const T *&src_next, T *&dst_out,
                                      int64_t plane_stride, int64_t row_stride, T r) {
  using V = typename Vec<T, CPT>::V;
  const int lane = threadIdx.x & 31;
  const int wu = q.w > 0 ? q.w - 1 : 0, wd = q.w < NW - 1 ? q.w + 1 : NW - 1;
#pragma unroll
  for (int y = 0; y < RPT; ++y)
#pragma unroll
    for (int c = 0; c < CPT; ++c) cur[0][y][c] = pre[y][c];
  X.tp(PAR, 0, q.w, lane) = vmake<CPT, V>(cur[0][0]);
  if constexpr (RPT > 1) X.bt(PAR, 0, q.w, lane) = vmake<CPT, V>(cur[0][RPT - 1]);
  {
    const int zn = q.zz + 1;
    const bool pin = zn < q.nz && zn <= q.ze && (!EDGE || zn >= 0);
#pragma unroll
    for (int y = 0; y < RPT; ++y)
#pragma unroll
      for (int c = 0; c < CPT; ++c)
        pre[y][c] = (pin && colin[y][c]) ? __ldg(src_next + y * row_stride + c) : T(0);
    src_next += plane_stride;
  }
#pragma unroll
  for (int L = 0; L < S; ++L) {
    const int zr = q.zz - L - 1;
    const bool rin = !EDGE || (zr >= 0 && zr < q.nz);
    T upe[CPT], dne[CPT];  // neighbours of the strip's top / bottom row from the adjacent strips
    vload<CPT>(X.bt(PAR ^ 1, L, wu, lane), upe);
    vload<CPT>(X.tp(PAR ^ 1, L, wd, lane), dne);
    T v[RPT][CPT];
#pragma unroll
    for (int y = 0; y < RPT; ++y) {
      const T left = __shfl_up_sync(0xffffffffu, prv[L][y][CPT - 1], 1);
      const T right = __shfl_down_sync(0xffffffffu, prv[L][y][0], 1);
      const T(&up)[CPT] = y == 0 ? upe : prv[L][y > 0 ? y - 1 : 0];
      const T(&dn)[CPT] = y == RPT - 1 ? dne : prv[L][y < RPT - 1 ? y + 1 : 0];
      if (EDGE) {
        T mm[CPT];
#pragma unroll
        for (int c = 0; c < CPT; ++c) mm[c] = rin ? m[y][c] : T(0);
        level_update<T, CPT, true>(prv[L][y], left, right, up, dn, pp[L][y], cur[L][y], r, mm, v[y]);
      } else {
        level_update<T, CPT, MASK>(prv[L][y], left, right, up, dn, pp[L][y], cur[L][y], r, m[y], v[y]);
      }
    }
    if (L + 1 < S) {
#pragma unroll
      for (int y = 0; y < RPT; ++y)
#pragma unroll
        for (int c = 0; c < CPT; ++c) cur[L + 1][y][c] = v[y][c];
      X.tp(PAR, L + 1, q.w, lane) = vmake<CPT, V>(v[0]);
      if constexpr (RPT > 1) X.bt(PAR, L + 1, q.w, lane) = vmake<CPT, V>(v[RPT - 1]);
    } else if (zr >= q.z0 && zr < q.z0 + ZC && rin) {
#pragma unroll
      for (int y = 0; y < RPT; ++y)
#pragma unroll
        for (int c = 0; c < CPT; ++c)
          if (colout[y][c]) dst_out[y * row_stride + c] = v[y][c];
    }
  }
  dst_out += plane_stride;
#pragma unroll
  for (int L = 0; L < S; ++L)
#pragma unroll
    for (int y = 0; y < RPT; ++y)
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        pp[L][y][c] = prv[L][y][c];
        prv[L][y][c] = cur[L][y][c];
      }
  __syncthreads();
}

template <typename T, int S, int NW, int RPT, int CPT, bool MASK>
__device__ __forceinline__ void sweep(Xchg<T, S, NW, RPT, CPT> &X, PlaneCtx q, int zs, const T (&m)[RPT][CPT],
                                      const bool (&colout)[RPT][CPT], const bool (&colin)[RPT][CPT],
                                      const T *src_col, T *dst_col, int64_t pl, int64_t rs, T r) {
  T cur[S][RPT][CPT], prv[S][RPT][CPT], pp[S][RPT][CPT];
#pragma unroll
  for (int L = 0; L < S; ++L)
#pragma unroll
    for (int y = 0; y < RPT; ++y)
#pragma unroll
      for (int c = 0; c < CPT; ++c) cur[L][y][c] = prv[L][y][c] = pp[L][y][c] = T(0);
  T pre[RPT][CPT];
  {
    const bool pin = zs >= 0 && zs < q.nz;
#pragma unroll
    for (int y = 0; y < RPT; ++y)
#pragma unroll
      for (int c = 0; c < CPT; ++c)
        pre[y][c] = (pin && colin[y][c]) ? __ldg(src_col + (int64_t)zs * pl + y * rs + c) : T(0);
  }
  // pointer offsets may start before the array (never dereferenced there)
  const T *src_next = src_col + (int64_t)(zs + 1) * pl;
  T *dst_out = dst_col + (int64_t)(zs - S) * pl;
  int zz = zs;
  while (zz <= q.ze) {
    if (zz >= S && zz + 5 <= q.nz && zz + 5 <= q.ze) {
      // steady state: six planes (three-plane register rotation x two buffer
      // parities), every level's plane inside the domain
#pragma unroll
      for (int u = 0; u < 6; u += 2) {
        q.zz = zz + u;
        plane<T, S, NW, RPT, CPT, false, MASK, 0>(cur, prv, pp, pre, X, q, m, colout, colin, src_next, dst_out, pl,
                                                  rs, r);
        q.zz = zz + u + 1;
        plane<T, S, NW, RPT, CPT, false, MASK, 1>(cur, prv, pp, pre, X, q, m, colout, colin, src_next, dst_out, pl,
                                                  rs, r);
      }
      zz += 6;
    } else {
      q.zz = zz;
      plane<T, S, NW, RPT, CPT, true, true, 0>(cur, prv, pp, pre, X, q, m, colout, colin, src_next, dst_out, pl, rs,
                                               r);
      if (zz + 1 > q.ze) break;
      q.zz = zz + 1;
      plane<T, S, NW, RPT, CPT, true, true, 1>(cur, prv, pp, pre, X, q, m, colout, colin, src_next, dst_out, pl, rs,
                                               r);
      zz += 2;
    }
  }
}

// Tile: (32 CPT) columns x (NW RPT) rows including the S-cell halo; warp w
// owns rows RPT w .. RPT w + RPT - 1 (inner y-neighbours stay in registers).
template <typename T, int S, int NW, int RPT, int CPT, int MINB>
__global__ void __launch_bounds__(32 * NW, MINB)
fe3d_tile(const T *__restrict__ in, T *__restrict__ out, int64_t stride, int nx, int ny, int nz, T r, int tiles_x) {
  using X_t = Xchg<T, S, NW, RPT, CPT>;
  extern __shared__ __align__(16) unsigned char smraw[];
  X_t &X = *reinterpret_cast<X_t *>(smraw);
  constexpr int W = 32 * CPT, H = NW * RPT;
  constexpr int BX = W - 2 * S, BY = H - 2 * S;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int bx = blockIdx.x % tiles_x, by = blockIdx.x / tiles_x;
  const int x0 = bx * BX - S, y0 = by * BY - S, z0 = blockIdx.y * ZC;
  const int64_t pl = (int64_t)nx * ny;
  const int cx = x0 + CPT * lane, cy0 = y0 + RPT * w;
  T m[RPT][CPT];
  bool colout[RPT][CPT], colin[RPT][CPT];
#pragma unroll
  for (int y = 0; y < RPT; ++y)
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const int cy = cy0 + y, ly = RPT * w + y, lx = CPT * lane + c;
      colin[y][c] = cx + c >= 0 && cx + c < nx && cy >= 0 && cy < ny;
      m[y][c] = colin[y][c] ? T(1) : T(0);
      colout[y][c] = colin[y][c] && lx >= S && lx < S + BX && ly >= S && ly < S + BY;
    }
  {
    using V = typename Vec<T, CPT>::V;
    T z[CPT];
#pragma unroll
    for (int c = 0; c < CPT; ++c) z[c] = T(0);
    V *flat = reinterpret_cast<V *>(smraw);
    for (int i = threadIdx.x; i < (int)(sizeof(X_t) / sizeof(V)); i += 32 * NW) flat[i] = vmake<CPT, V>(z);
  }
  __syncthreads();
  // column base pointers (rows/columns outside the domain are never dereferenced)
  const int64_t col = (int64_t)cy0 * nx + cx;
  const T *src_col = in + (int64_t)blockIdx.z * stride + col;
  T *dst_col = out + (int64_t)blockIdx.z * stride + col;
  PlaneCtx q;
  q.w = w;
  q.z0 = z0;
  q.nz = nz;
  q.zz = 0;
  const int zs = z0 - S;
  q.ze = min(z0 + ZC, nz) - 1 + S;
  // tiles wholly inside the domain skip the Dirichlet mask
  const bool tile_in = x0 >= 0 && x0 + W <= nx && y0 >= 0 && y0 + H <= ny;
  if (tile_in) sweep<T, S, NW, RPT, CPT, false>(X, q, zs, m, colout, colin, src_col, dst_col, pl, nx, r);
  else sweep<T, S, NW, RPT, CPT, true>(X, q, zs, m, colout, colin, src_col, dst_col, pl, nx, r);
}

template <typename T, int S, int NW, int RPT, int CPT, int MINB>
void launch_tile(const T *in, T *out, int64_t nb, int64_t stride, int nx, int ny, int nz, T r, cudaStream_t st) {
  constexpr int BX = 32 * CPT - 2 * S, BY = NW * RPT - 2 * S;
  const int tiles_x = (nx + BX - 1) / BX, tiles_y = (ny + BY - 1) / BY;
  const unsigned tz = (unsigned)((nz + ZC - 1) / ZC);
  const size_t smem = sizeof(Xchg<T, S, NW, RPT, CPT>);
  auto kern = fe3d_tile<T, S, NW, RPT, CPT, MINB>;
  PINT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  for (int64_t b0 = 0; b0 < nb; b0 += 65535) {
    const unsigned n = (unsigned)std::min<int64_t>(65535, nb - b0);
    kern<<<dim3((unsigned)(tiles_x * tiles_y), tz, n), 32 * NW, smem, st>>>(in + b0 * stride, out + b0 * stride,
                                                                            stride, nx, ny, nz, r, tiles_x);
  }
  PINT_CUDA(cudaGetLastError());
}

// one pass of s <= SMAX levels
template <typename T, int SMAX, int NW, int RPT, int CPT, int MINB>
void pass_tile(int s, const T *in, T *out, int64_t nb, int64_t stride, int nx, int ny, int nz, T r, cudaStream_t st) {
  if constexpr (SMAX >= 4) if (s == 4) return launch_tile<T, 4, NW, RPT, CPT, MINB>(in, out, nb, stride, nx, ny, nz, r, st);
  if constexpr (SMAX >= 3) if (s == 3) return launch_tile<T, 3, NW, RPT, CPT, MINB>(in, out, nb, stride, nx, ny, nz, r, st);
  if constexpr (SMAX >= 2) if (s == 2) return launch_tile<T, 2, NW, RPT, CPT, MINB>(in, out, nb, stride, nx, ny, nz, r, st);
  launch_tile<T, 1, NW, RPT, CPT, MINB>(in, out, nb, stride, nx, ny, nz, r, st);
}

template <typename T, int SMAX, int NW, int RPT, int CPT, int MINB>
void apply_tile(const pint_op *op, const T *in, T *out, T *scratch, int64_t nb, int64_t stride, cudaStream_t st) {
  const int64_t S = op->desc.steps;
  const int64_t npass = (S + SMAX - 1) / SMAX;
  const T r = (T)(op->dt / (op->desc.h * op->desc.h));
  int64_t done = 0;
  for (int64_t pass = 0; pass < npass; ++pass) {
    const int s = (int)std::min<int64_t>(SMAX, S - done);
    const T *src = pass == 0 ? in : (((npass - pass) % 2 == 0) ? out : scratch);
    T *dstp = ((npass - 1 - pass) % 2 == 0) ? out : scratch;
    pass_tile<T, SMAX, NW, RPT, CPT, MINB>(s, src, dstp, nb, stride, (int)op->nx, (int)op->ny, (int)op->nz, r, st);
    done += s;
  }
}

}  // namespace

// Tile variants (PINT_FE3D_VARIANT selects one for measurement; 0 = the
// first-generation fe3d_wave in stencil_wave.cu). Tile = (32 CPT) x (NW RPT)
// incl. halo; NW warps per CTA, RPT rows per thread.
//   fp32: 1 = S4 64x32 (NW32 RPT1), 2 = S3 64x32, 3 = S4 64x32 (NW16 RPT2), 4 = S4 64x48 (NW24 RPT2),
//         5 = S2 128x32 (NW16 RPT2 CPT4), 6 = S3 64x32 (NW16 RPT2), 7 = S4 64x64 (NW32 RPT2),
//         8 = S3 64x48 (NW16 RPT3), 9 = S4 64x36 (NW12 RPT3), 10 = S3 64x40 (NW20 RPT2), 11 = S4 64x40 (NW20 RPT2)
//   fp64: 1 = S4 64x16, 2 = S3 64x24, 3 = S3 64x20, 4 = S4 64x32 (NW16 RPT2), 5 = S3 64x32 (NW16 RPT2),
//         6 = S2 64x32 (NW16 RPT2), 7 = S3 64x40 (NW20 RPT2)
// Defaults measured at the C4 shape (profiles/r01_fe3d_variants.jsonl).
int fe3d_tile_default(int esz) { return esz == 4 ? 8 : 5; }

template <typename T>
bool fe3d_tile_apply(int variant, const pint_op *op, const T *in, T *out, T *scratch, int64_t nb, int64_t stride,
                     cudaStream_t st) {
  if constexpr (sizeof(T) == 4) {
    switch (variant) {
      case 1: apply_tile<T, 4, 32, 1, 2, 1>(op, in, out, scratch, nb, stride, st); return true;
      case 2: apply_tile<T, 3, 32, 1, 2, 1>(op, in, out, scratch, nb, stride, st); return true;
      case 3: apply_tile<T, 4, 16, 2, 2, 1>(op, in, out, scratch, nb, stride, st); return true;
      case 4: apply_tile<T, 4, 24, 2, 2, 1>(op, in, out, scratch, nb, stride, st); return true;
      case 5: apply_tile<T, 2, 16, 2, 4, 1>(op, in, out, scratch, nb, stride, st); return true;
      case 6: apply_tile<T, 3, 16, 2, 2, 1>(op, in, out, scratch, nb, stride, st); return true;
      case 7: apply_tile<T, 4, 32, 2, 2, 1>(op, in, out, scratch, nb, stride, st); return true;
      case 8: apply_tile<T, 3, 16, 3, 2, 1>(op, in, out, scratch, nb, stride, st); return true;
      case 9: apply_tile<T, 4, 12, 3, 2, 1>(op, in, out, scratch, nb, stride, st); return true;
      case 10: apply_tile<T, 3, 20, 2, 2, 1>(op, in, out, scratch, nb, stride, st); return true;
      case 11: apply_tile<T, 4, 20, 2, 2, 1>(op, in, out, scratch, nb, stride, st); return true;
      default: return false;
    }
  } else {
    switch (variant) {
      case 1: apply_tile<T, 4, 16, 1, 2, 1>(op, in, out, scratch, nb, stride, st); return true;
      case 2: apply_tile<T, 3, 24, 1, 2, 1>(op, in, out, scratch, nb, stride, st); return true;
      case 3: apply_tile<T, 3, 20, 1, 2, 1>(op, in, out, scratch, nb, stride, st); return true;
      case 4: apply_tile<T, 4, 16, 2, 2, 1>(op, in, out, scratch, nb, stride, st); return true;
      case 5: apply_tile<T, 3, 16, 2, 2, 1>(op, in, out, scratch, nb, stride, st); return true;
      case 6: apply_tile<T, 2, 16, 2, 2, 1>(op, in, out, scratch, nb, stride, st); return true;
      case 7: apply_tile<T, 3, 20, 2, 2, 1>(op, in, out, scratch, nb, stride, st); return true;
      default: return false;
    }
  }
}

template bool fe3d_tile_apply<float>(int, const pint_op *, const float *, float *, float *, int64_t, int64_t,
                                     cudaStream_t);
template bool fe3d_tile_apply<double>(int, const pint_op *, const double *, double *, double *, int64_t, int64_t,
                                      cudaStream_t);
