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
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "pint_internal.cuh"

namespace {

constexpr int ZC = 128;  // output planes per chunk
constexpr int TMA_D = 4;  // input planes in flight per CTA (TMA ring depth)

// ---- TMA input ring (variants with TMA = true): the CTA's xy tile of each
// input plane arrives in shared memory by one cp.async.bulk.tensor load
// (4-D tensor map x, y, z, slice; the halo outside the grid is zero-filled by
// the TMA unit, i.e. the zero Dirichlet values), TMA_D planes ahead of the
// wavefront, each completing on its own mbarrier.
// x extent of a tile: halo HL on the left, BX output columns. With TMA the
// box origin x0 must be a multiple of 16 bytes (the unit refuses other inner
// coordinates), so the TMA tilings use 4-column halos (x0 = 56 bx - 4 is a
// multiple of 4 floats / 2 doubles; S <= 4 levels fit in the halo).
template <int S, int CPT, bool TMA>
struct XTile {
  static constexpr int HL = TMA ? 4 : S;
  static constexpr int BX = 32 * CPT - HL - (TMA ? 4 : S);
};

struct TmaCtx {
  uint32_t ring;  // shared address of slot 0
  uint32_t bars;  // shared address of TMA_D mbarriers
  int x0, y0, b;  // tile origin (incl. halo) and slice
  int zs;         // first input plane of the sweep
  const CUtensorMap *map;
};

__device__ __forceinline__ uint32_t smem_addr(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void tma_bar_init(uint32_t bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tma_bar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "TW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra TW_%=;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
// load plane z of the tile into ring slot `slot` (one elected thread)
template <int W, int H, typename T>
__device__ __forceinline__ void tma_plane(const TmaCtx &t, int slot, int z) {
  const uint32_t bar = t.bars + 8u * (uint32_t)slot;
  const uint32_t dst = t.ring + (uint32_t)(slot * W * H * (int)sizeof(T));
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads of the slot before the async write
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"((uint32_t)(W * H * sizeof(T)))
               : "memory");
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(t.map)), "r"(t.x0), "r"(t.y0), "r"(z), "r"(t.b), "r"(bar)
      : "memory");
}

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
template <typename T, int S, int NW, int RPT, int CPT, bool EDGE, bool MASK, int PAR, bool TMA>
__device__ __forceinline__ void plane(T (&cur)[S][RPT][CPT], T (&prv)[S][RPT][CPT], T (&pp)[S][RPT][CPT],
                                      T (&pre)[RPT][CPT], Xchg<T, S, NW, RPT, CPT> &X, const PlaneCtx &q,
                                      const T (&m)[RPT][CPT], const bool (&colout)[RPT][CPT],
                                      const bool (&colin)[RPT][CPT], const T *&src_next, T *&dst_out,
                                      int64_t plane_stride, int64_t row_stride, T r, const TmaCtx &tm) {
  using V = typename Vec<T, CPT>::V;
  constexpr int W = 32 * CPT, H = NW * RPT;
  const int lane = threadIdx.x & 31;
  const int wu = q.w > 0 ? q.w - 1 : 0, wd = q.w < NW - 1 ? q.w + 1 : NW - 1;
  if constexpr (TMA) {
    const int pi = q.zz - tm.zs;
    const int slot = pi & (TMA_D - 1);
    tma_bar_wait(tm.bars + 8u * (uint32_t)slot, (uint32_t)(pi / TMA_D) & 1u);
    const unsigned a = tm.ring + (unsigned)(((slot * H + RPT * q.w) * W + CPT * lane) * (int)sizeof(T));
#pragma unroll
    for (int y = 0; y < RPT; ++y) {
      T tmp[CPT];
      const unsigned ay = a + (unsigned)(y * W * (int)sizeof(T));
      if constexpr (sizeof(T) * CPT == 8) {
        unsigned long long u;
        asm volatile("ld.shared.b64 %0, [%1];" : "=l"(u) : "r"(ay));
        memcpy(tmp, &u, 8);
      } else {
        uint4 u;
        asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w) : "r"(ay));
        memcpy(tmp, &u, 16);
      }
#pragma unroll
      for (int c = 0; c < CPT; ++c) cur[0][y][c] = tmp[c];
    }
  } else {
#pragma unroll
    for (int y = 0; y < RPT; ++y)
#pragma unroll
      for (int c = 0; c < CPT; ++c) cur[0][y][c] = pre[y][c];
  }
  X.tp(PAR, 0, q.w, lane) = vmake<CPT, V>(cur[0][0]);
  if constexpr (RPT > 1) X.bt(PAR, 0, q.w, lane) = vmake<CPT, V>(cur[0][RPT - 1]);
  if constexpr (!TMA) {
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
  if constexpr (TMA) {
    // every thread has read this plane's slot: refill it TMA_D planes ahead
    const int zn = q.zz + TMA_D;
    if (threadIdx.x == 0 && zn <= q.ze) tma_plane<W, H, T>(tm, (zn - tm.zs) & (TMA_D - 1), zn);
  }
}

template <typename T, int S, int NW, int RPT, int CPT, bool MASK, bool TMA>
__device__ __forceinline__ void sweep(Xchg<T, S, NW, RPT, CPT> &X, PlaneCtx q, int zs, const T (&m)[RPT][CPT],
                                      const bool (&colout)[RPT][CPT], const bool (&colin)[RPT][CPT],
                                      const T *src_col, T *dst_col, int64_t pl, int64_t rs, T r, const TmaCtx &tm) {
  T cur[S][RPT][CPT], prv[S][RPT][CPT], pp[S][RPT][CPT];
#pragma unroll
  for (int L = 0; L < S; ++L)
#pragma unroll
    for (int y = 0; y < RPT; ++y)
#pragma unroll
      for (int c = 0; c < CPT; ++c) cur[L][y][c] = prv[L][y][c] = pp[L][y][c] = T(0);
  T pre[RPT][CPT];
  if constexpr (!TMA) {
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
        plane<T, S, NW, RPT, CPT, false, MASK, 0, TMA>(cur, prv, pp, pre, X, q, m, colout, colin, src_next, dst_out,
                                                       pl, rs, r, tm);
        q.zz = zz + u + 1;
        plane<T, S, NW, RPT, CPT, false, MASK, 1, TMA>(cur, prv, pp, pre, X, q, m, colout, colin, src_next, dst_out,
                                                       pl, rs, r, tm);
      }
      zz += 6;
    } else {
      q.zz = zz;
      plane<T, S, NW, RPT, CPT, true, true, 0, TMA>(cur, prv, pp, pre, X, q, m, colout, colin, src_next, dst_out, pl,
                                                    rs, r, tm);
      if (zz + 1 > q.ze) break;
      q.zz = zz + 1;
      plane<T, S, NW, RPT, CPT, true, true, 1, TMA>(cur, prv, pp, pre, X, q, m, colout, colin, src_next, dst_out, pl,
                                                    rs, r, tm);
      zz += 2;
    }
  }
}

// Tile: (32 CPT) columns x (NW RPT) rows including the S-cell halo; warp w
// owns rows RPT w .. RPT w + RPT - 1 (inner y-neighbours stay in registers).
template <typename T, int S, int NW, int RPT, int CPT>
constexpr size_t tile_smem(bool tma) {
  return tma ? (sizeof(Xchg<T, S, NW, RPT, CPT>) + 127) / 128 * 128 + (size_t)TMA_D * 32 * CPT * NW * RPT * sizeof(T) +
                   8 * TMA_D
             : sizeof(Xchg<T, S, NW, RPT, CPT>);
}

template <typename T, int S, int NW, int RPT, int CPT, int MINB, bool TMA>
__global__ void __launch_bounds__(32 * NW, MINB)
fe3d_tile(const T *__restrict__ in, T *__restrict__ out, int64_t stride, int nx, int ny, int nz, T r, int tiles_x,
          const __grid_constant__ CUtensorMap tmap) {
  using X_t = Xchg<T, S, NW, RPT, CPT>;
  extern __shared__ __align__(16) unsigned char smraw[];
  X_t &X = *reinterpret_cast<X_t *>(smraw);
  constexpr int W = 32 * CPT, H = NW * RPT;
  constexpr int BX = XTile<S, CPT, TMA>::BX, HL = XTile<S, CPT, TMA>::HL, BY = H - 2 * S;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int bx = blockIdx.x % tiles_x, by = blockIdx.x / tiles_x;
  const int x0 = bx * BX - HL, y0 = by * BY - S, z0 = blockIdx.y * ZC;
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
      colout[y][c] = colin[y][c] && lx >= HL && lx < HL + BX && ly >= S && ly < S + BY;
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
  TmaCtx tm{};
  if constexpr (TMA) {
    const uint32_t base = smem_addr(smraw);
    tm.ring = base + (uint32_t)((sizeof(X_t) + 127) / 128 * 128);
    tm.bars = tm.ring + (uint32_t)(TMA_D * W * H * sizeof(T));
    tm.x0 = x0;
    tm.y0 = y0;
    tm.b = (int)blockIdx.z;
    tm.zs = zs;
    tm.map = &tmap;
    if (threadIdx.x == 0) {
      for (int d = 0; d < TMA_D; ++d) tma_bar_init(tm.bars + 8u * (uint32_t)d);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int d = 0; d < TMA_D && zs + d <= q.ze; ++d) tma_plane<W, H, T>(tm, d, zs + d);
  }
  if (tile_in) sweep<T, S, NW, RPT, CPT, false, TMA>(X, q, zs, m, colout, colin, src_col, dst_col, pl, nx, r, tm);
  else sweep<T, S, NW, RPT, CPT, true, TMA>(X, q, zs, m, colout, colin, src_col, dst_col, pl, nx, r, tm);
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link)
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    PINT_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p) pint_throw(PINT_ECUDA, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 4-D map of nb slices (x fastest), box = one plane of a W x H tile; zero OOB fill
template <typename T>
bool make_plane_map(CUtensorMap *m, const T *base, int nx, int ny, int nz, int64_t nb, int64_t stride, int W, int H) {
  const uint64_t esz = sizeof(T);
  if (((uintptr_t)base & 15u) || (nx * esz) % 16 || (stride * esz) % 16 || nb > 0x7fffffff) return false;
  cuuint64_t dims[4] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)nz, (cuuint64_t)nb};
  cuuint64_t strides[3] = {(cuuint64_t)nx * esz, (cuuint64_t)nx * ny * esz, (cuuint64_t)stride * esz};
  cuuint32_t box[4] = {(cuuint32_t)W, (cuuint32_t)H, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  const CUresult rc = tensor_map_encoder()(m, esz == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                                           4, const_cast<T *>(base), dims, strides, box, es,
                                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return rc == CUDA_SUCCESS;
}

template <typename T, int S, int NW, int RPT, int CPT, int MINB, bool TMA>
void launch_tile(const T *in, T *out, int64_t nb, int64_t stride, int nx, int ny, int nz, T r, cudaStream_t st) {
  constexpr int BY = NW * RPT - 2 * S;
  // the TMA tiling has its own x step; a layout the tensor map cannot describe
  // runs the non-TMA kernel with the non-TMA step
  const bool tma_ok = TMA && ((uintptr_t)in & 15u) == 0 && (nx * sizeof(T)) % 16 == 0 && (stride * sizeof(T)) % 16 == 0;
  const int BX = tma_ok ? XTile<S, CPT, true>::BX : XTile<S, CPT, false>::BX;
  const int tiles_x = (nx + BX - 1) / BX, tiles_y = (ny + BY - 1) / BY;
  const unsigned tz = (unsigned)((nz + ZC - 1) / ZC);
  for (int64_t b0 = 0; b0 < nb; b0 += 65535) {
    const unsigned n = (unsigned)std::min<int64_t>(65535, nb - b0);
    CUtensorMap map;
    memset(&map, 0, sizeof(map));
    const bool tma = tma_ok && make_plane_map<T>(&map, in + b0 * stride, nx, ny, nz, n, stride, 32 * CPT, NW * RPT);
    if (tma_ok && !tma) pint_throw(PINT_ECUDA, "cuTensorMapEncodeTiled refused the plane map");
    if (tma) {
      auto kern = fe3d_tile<T, S, NW, RPT, CPT, MINB, true>;
      const size_t smem = tile_smem<T, S, NW, RPT, CPT>(true);
      PINT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      kern<<<dim3((unsigned)(tiles_x * tiles_y), tz, n), 32 * NW, smem, st>>>(in + b0 * stride, out + b0 * stride,
                                                                              stride, nx, ny, nz, r, tiles_x, map);
    } else {
      // no TMA (variant without it, or a layout the tensor map cannot describe:
      // rows or slice strides not multiples of 16 bytes)
      auto kern = fe3d_tile<T, S, NW, RPT, CPT, MINB, false>;
      const size_t smem = tile_smem<T, S, NW, RPT, CPT>(false);
      PINT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      kern<<<dim3((unsigned)(tiles_x * tiles_y), tz, n), 32 * NW, smem, st>>>(in + b0 * stride, out + b0 * stride,
                                                                              stride, nx, ny, nz, r, tiles_x, map);
    }
  }
  PINT_CUDA(cudaGetLastError());
}

// one pass of s <= SMAX levels
template <typename T, int SMAX, int NW, int RPT, int CPT, int MINB, bool TMA>
void pass_tile(int s, const T *in, T *out, int64_t nb, int64_t stride, int nx, int ny, int nz, T r, cudaStream_t st) {
  if constexpr (SMAX >= 4) if (s == 4) return launch_tile<T, 4, NW, RPT, CPT, MINB, TMA>(in, out, nb, stride, nx, ny, nz, r, st);
  if constexpr (SMAX >= 3) if (s == 3) return launch_tile<T, 3, NW, RPT, CPT, MINB, TMA>(in, out, nb, stride, nx, ny, nz, r, st);
  if constexpr (SMAX >= 2) if (s == 2) return launch_tile<T, 2, NW, RPT, CPT, MINB, TMA>(in, out, nb, stride, nx, ny, nz, r, st);
  launch_tile<T, 1, NW, RPT, CPT, MINB, TMA>(in, out, nb, stride, nx, ny, nz, r, st);
}

template <typename T, int SMAX, int NW, int RPT, int CPT, int MINB, bool TMA = false>
void apply_tile(const pint_op *op, const T *in, T *out, T *scratch, int64_t nb, int64_t stride, cudaStream_t st) {
  const int64_t S = op->desc.steps;
  const int64_t npass = (S + SMAX - 1) / SMAX;
  const T r = (T)(op->dt / (op->desc.h * op->desc.h));
  int64_t done = 0;
  for (int64_t pass = 0; pass < npass; ++pass) {
    const int s = (int)std::min<int64_t>(SMAX, S - done);
    const T *src = pass == 0 ? in : (((npass - pass) % 2 == 0) ? out : scratch);
    T *dstp = ((npass - 1 - pass) % 2 == 0) ? out : scratch;
    pass_tile<T, SMAX, NW, RPT, CPT, MINB, TMA>(s, src, dstp, nb, stride, (int)op->nx, (int)op->ny, (int)op->nz, r, st);
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
//         12 = variant 8 with TMA input planes, 13 = variant 3 with TMA, 14 = variant 9 with TMA,
//         15 = TMA S2 128x48 (NW16 RPT3 CPT4), 16 = TMA S3 64x48 (NW24 RPT2), 17 = TMA S3 64x64 (NW16 RPT4),
//         18 = TMA S3 64x48 (NW12 RPT4), 19 = TMA S4 64x48 (NW8 RPT6), 20 = TMA S4 64x50 (NW10 RPT5),
//         21 = TMA S4 64x48 (NW12 RPT4), 22 = TMA S4 64x32 (NW8 RPT4), 23 = TMA S4 64x60 (NW12 RPT5),
//         24 = TMA S3 64x48 (NW8 RPT6), 25 = TMA S4 64x40 (NW8 RPT5), 26 = TMA S4 64x36 (NW6 RPT6)
//         (2-CTA/SM caps of the TMA tiles were dropped: ptxas 12.9 crashes on them)
//   fp64: 1 = S4 64x16, 2 = S3 64x24, 3 = S3 64x20, 4 = S4 64x32 (NW16 RPT2), 5 = S3 64x32 (NW16 RPT2),
//         6 = S2 64x32 (NW16 RPT2), 7 = S3 64x40 (NW20 RPT2), 8 = variant 5 with TMA input planes,
//         9 = TMA S3 64x48 (NW16 RPT3), 10 = TMA S2 64x48 (NW16 RPT3), 11 = TMA S3 64x36 (NW12 RPT3),
//         12 = TMA S3 64x32 (NW8 RPT4), 13 = TMA S3 64x30 (NW10 RPT3), 14 = TMA S2 64x36 (NW12 RPT3),
//         15 = TMA S3 64x40 (NW8 RPT5), 16 = TMA S4 64x32 (NW8 RPT4), 17 = TMA S3 64x30 (NW6 RPT5),
//         18 = TMA S3 64x48 (NW8 RPT6), 19 = TMA S3 64x36 (NW6 RPT6), 20 = TMA S2 64x48 (NW8 RPT6)
// Defaults measured at the C4 shape (profiles/r02_fe3d_variants.jsonl): the
// TMA input ring with deep strips and few warps (fewer y-exchange rows per
// cell), fp32 948 -> 1331 GPt/s (variant 8 -> 19: S4, 8 warps x 6 rows),
// fp64 457 -> 707 (variant 5 -> 12: S3, 8 warps x 4 rows); 512^3 fp32
// 1178 -> 1533.
int fe3d_tile_default(int esz) { return esz == 4 ? 19 : 12; }

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
      case 12: apply_tile<T, 3, 16, 3, 2, 1, true>(op, in, out, scratch, nb, stride, st); return true;
      case 13: apply_tile<T, 4, 16, 2, 2, 1, true>(op, in, out, scratch, nb, stride, st); return true;
      case 14: apply_tile<T, 4, 12, 3, 2, 1, true>(op, in, out, scratch, nb, stride, st); return true;
      case 15: apply_tile<T, 2, 16, 3, 4, 1, true>(op, in, out, scratch, nb, stride, st); return true;
      case 16: apply_tile<T, 3, 24, 2, 2, 1, true>(op, in, out, scratch, nb, stride, st); return true;
      case 17: apply_tile<T, 3, 16, 4, 2, 1, true>(op, in, out, scratch, nb, stride, st); return true;
      case 18: apply_tile<T, 3, 12, 4, 2, 1, true>(op, in, out, scratch, nb, stride, st); return true;
      case 19: apply_tile<T, 4, 8, 6, 2, 1, true>(op, in, out, scratch, nb, stride, st); return true;
      case 20: apply_tile<T, 4, 10, 5, 2, 1, true>(op, in, out, scratch, nb, stride, st); return true;
      case 21: apply_tile<T, 4, 12, 4, 2, 1, true>(op, in, out, scratch, nb, stride, st); return true;
      case 22: apply_tile<T, 4, 8, 4, 2, 1, true>(op, in, out, scratch, nb, stride, st); return true;
      case 23: apply_tile<T, 4, 12, 5, 2, 1, true>(op, in, out, scratch, nb, stride, st); return true;
      case 24: apply_tile<T, 3, 8, 6, 2, 1, true>(op, in, out, scratch, nb, stride, st); return true;
      case 25: apply_tile<T, 4, 8, 5, 2, 1, true>(op, in, out, scratch, nb, stride, st); return true;
      case 26: apply_tile<T, 4, 6, 6, 2, 1, true>(op, in, out, scratch, nb, stride, st); return true;
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
      case 8: apply_tile<T, 3, 16, 2, 2, 1, true>(op, in, out, scratch, nb, stride, st); return true;
      case 9: apply_tile<T, 3, 16, 3, 2, 1, true>(op, in, out, scratch, nb, stride, st); return true;
      case 10: apply_tile<T, 2, 16, 3, 2, 1, true>(op, in, out, scratch, nb, stride, st); return true;
      case 11: apply_tile<T, 3, 12, 3, 2, 1, true>(op, in, out, scratch, nb, stride, st); return true;
      case 12: apply_tile<T, 3, 8, 4, 2, 1, true>(op, in, out, scratch, nb, stride, st); return true;
      case 13: apply_tile<T, 3, 10, 3, 2, 1, true>(op, in, out, scratch, nb, stride, st); return true;
      case 14: apply_tile<T, 2, 12, 3, 2, 1, true>(op, in, out, scratch, nb, stride, st); return true;
      case 15: apply_tile<T, 3, 8, 5, 2, 1, true>(op, in, out, scratch, nb, stride, st); return true;
      case 16: apply_tile<T, 4, 8, 4, 2, 1, true>(op, in, out, scratch, nb, stride, st); return true;
      case 17: apply_tile<T, 3, 6, 5, 2, 1, true>(op, in, out, scratch, nb, stride, st); return true;
      case 18: apply_tile<T, 3, 8, 6, 2, 1, true>(op, in, out, scratch, nb, stride, st); return true;
      case 19: apply_tile<T, 3, 6, 6, 2, 1, true>(op, in, out, scratch, nb, stride, st); return true;
      case 20: apply_tile<T, 2, 8, 6, 2, 1, true>(op, in, out, scratch, nb, stride, st); return true;
      default: return false;
    }
  }
}

template bool fe3d_tile_apply<float>(int, const pint_op *, const float *, float *, float *, int64_t, int64_t,
                                     cudaStream_t);
template bool fe3d_tile_apply<double>(int, const pint_op *, const double *, double *, double *, int64_t, int64_t,
                                      cudaStream_t);
