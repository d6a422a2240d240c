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
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "pint_internal.cuh"

namespace {

constexpr int SMAX2 = 8;                 // time levels per pass
constexpr int CPT2 = 2;                  // columns per thread
constexpr int BX2 = 256;                 // output columns per tile
constexpr int W2 = BX2 + 2 * SMAX2;      // loaded columns per tile
constexpr int WT2 = W2 / CPT2;           // threads per CTA (136)
constexpr int YC2 = 128;                 // output rows per chunk

// TMA input ring of the 2-D wavefront (TMA = true): groups of RB2 input rows
// of the tile arrive in shared memory by two cp.async.bulk.tensor loads each
// (272 columns exceed the 256-element box limit: two 136-column boxes), the
// rows outside the grid zero-filled by the TMA unit (the Dirichlet values),
// D2<T> groups ahead of the wavefront, one mbarrier per ring slot. The tile
// origin is x0 = 256 bx - 8 for every pass depth (16-byte aligned inner
// coordinate, as the unit requires).
constexpr int RB2 = 8;
template <typename T>
constexpr int D2() { return sizeof(T) == 8 ? 2 : 4; }

__device__ __forceinline__ void bar_init2(uint32_t bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void bar_wait2(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "TW2_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra TW2_%=;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
template <typename T>
__device__ __forceinline__ void tma_rows2(const CUtensorMap *map, uint32_t ring, uint32_t bars, int slot, int x0,
                                          int y, int b) {
  const uint32_t bar = bars + 8u * (uint32_t)slot;
  const uint32_t dst = ring + (uint32_t)(slot * RB2 * W2 * (int)sizeof(T));
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
               "r"((uint32_t)(RB2 * W2 * sizeof(T)))
               : "memory");
#pragma unroll
  for (int h = 0; h < 2; ++h)
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(dst + (uint32_t)(h * RB2 * (W2 / 2) * (int)sizeof(T))),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x0 + h * (W2 / 2)), "r"(y), "r"(b), "r"(bar)
        : "memory");
}

template <typename T, int S, bool UNROLL, int MINB, bool TMA>
__global__ void __launch_bounds__(WT2, MINB)
fe2d_wave(const T *__restrict__ in, T *__restrict__ out, int64_t stride, int nx, int ny, T r,
          const __grid_constant__ CUtensorMap tmap) {
  const int tid = threadIdx.x;
  // fp64: the edge columns of every thread in two planes (a thread's first /
  // last column), so a warp's neighbour loads and edge stores are contiguous
  // (no two-way bank conflicts from the CPT2 column stride; C3 fp64 778 -> 817
  // GPt/s). fp32: interleaved row (the split layout measured 7 % slower).
  constexpr bool SPLIT = sizeof(T) == 8;
  __shared__ T sm[2][S][2][WT2 + 2];
  auto st_edge = [&](int pr, int L, const T (&vv)[CPT2]) {
    if constexpr (SPLIT) {
      sm[pr][L][0][1 + tid] = vv[0];
      sm[pr][L][1][1 + tid] = vv[CPT2 - 1];
    } else {
      T *row = &sm[pr][L][0][0];
#pragma unroll
      for (int c = 0; c < CPT2; ++c) row[1 + CPT2 * tid + c] = vv[c];
    }
  };
  constexpr int HL = TMA ? SMAX2 : S;   // left halo (TMA: 16-byte aligned origin)
  const int x0 = blockIdx.x * BX2 - HL;  // first loaded column
  const int y0 = blockIdx.y * YC2;
  const T *src = in + (int64_t)blockIdx.z * stride;
  T *dst = out + (int64_t)blockIdx.z * stride;
  const int cx = x0 + CPT2 * tid;
  bool colin[CPT2], colout[CPT2];
#pragma unroll
  for (int c = 0; c < CPT2; ++c) {
    colin[c] = cx + c >= 0 && cx + c < nx;
    const int lc = CPT2 * tid + c;  // local column
    colout[c] = colin[c] && lc >= HL && lc < HL + BX2;
  }
  for (int i = tid; i < 2 * S * 2 * (WT2 + 2); i += WT2) (&sm[0][0][0][0])[i] = T(0);
  T cur[S][CPT2], prv[S][CPT2], pp[S][CPT2];
#pragma unroll
  for (int L = 0; L < S; ++L)
#pragma unroll
    for (int c = 0; c < CPT2; ++c) cur[L][c] = prv[L][c] = pp[L][c] = T(0);
  __syncthreads();
  const T four = T(4);
  const int ys = y0 - S, ye = min(y0 + YC2, ny) - 1 + S;
  // TMA ring (dynamic shared memory): D2 slots of RB2 rows x W2 columns, stored
  // as two column halves [h][row][136], then D2 mbarriers
  extern __shared__ __align__(128) unsigned char ring_raw[];
  uint32_t ring = 0, bars = 0;
  if constexpr (TMA) {
    ring = static_cast<uint32_t>(__cvta_generic_to_shared(ring_raw));
    bars = ring + (uint32_t)(D2<T>() * RB2 * W2 * (int)sizeof(T));
    if (tid == 0) {
      for (int d = 0; d < D2<T>(); ++d) bar_init2(bars + 8u * (uint32_t)d);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0)
      for (int d = 0; d < D2<T>() && ys + d * RB2 <= ye; ++d)
        tma_rows2<T>(&tmap, ring, bars, d, x0, ys + d * RB2, (int)blockIdx.z);
  }
  // input rows are prefetched one iteration ahead (the load latency would
  // otherwise sit in front of every row's barrier)
  T pre[CPT2];
  if constexpr (!TMA) {
    const bool rowin = ys >= 0 && ys < ny;
#pragma unroll
    for (int c = 0; c < CPT2; ++c) pre[c] = (rowin && colin[c]) ? __ldg(src + (int64_t)ys * nx + cx + c) : T(0);
  }
  // one row of the wavefront; PAR = shared-buffer parity, EDGE = some level's
  // row may lie outside the domain
  auto row = [&](auto par_c, auto edge_c, int yy) {
    constexpr int par = decltype(par_c)::value;
    constexpr bool EDGE = decltype(edge_c)::value;
    // level 0: the input row yy
    if constexpr (TMA) {
      const int rr = yy - ys, g = rr / RB2, slot = g % D2<T>();
      if (rr % RB2 == 0) bar_wait2(bars + 8u * (uint32_t)slot, (uint32_t)(g / D2<T>()) & 1u);
      // this thread's two columns: half h = tid / 68 of the slot, row rr % RB2
      const int h = tid >= WT2 / 2 ? 1 : 0;
      const uint32_t a = ring + (uint32_t)(((slot * 2 + h) * RB2 + rr % RB2) * (W2 / 2) * (int)sizeof(T) +
                                           (CPT2 * tid - h * (W2 / 2)) * (int)sizeof(T));
      if constexpr (sizeof(T) == 8) {
        double2 v;
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
        cur[0][0] = v.x;
        cur[0][1] = v.y;
      } else {
        float2 v;
        asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
        cur[0][0] = v.x;
        cur[0][1] = v.y;
      }
    } else {
#pragma unroll
      for (int c = 0; c < CPT2; ++c) cur[0][c] = pre[c];
    }
    if constexpr (!TMA) {
      const int yn = yy + 1;
      const bool rowin = yn >= 0 && yn < ny && yn <= ye;
#pragma unroll
      for (int c = 0; c < CPT2; ++c) pre[c] = (rowin && colin[c]) ? __ldg(src + (int64_t)yn * nx + cx + c) : T(0);
    }
    st_edge(par, 0, cur[0]);
    // levels 1..S: level L+1 at row yy-L-1 from level L rows (pp, prv, cur)
#pragma unroll
    for (int L = 0; L < S; ++L) {
      const int yr = yy - L - 1;
      const bool rin = !EDGE || (yr >= 0 && yr < ny);
      // last column of thread tid-1, first column of thread tid+1
      const T left = SPLIT ? sm[par ^ 1][L][1][tid] : (&sm[par ^ 1][L][0][0])[CPT2 * tid];
      const T right = SPLIT ? sm[par ^ 1][L][0][tid + 2] : (&sm[par ^ 1][L][0][0])[1 + CPT2 * tid + CPT2];
      T v[CPT2];
#pragma unroll
      for (int c = 0; c < CPT2; ++c) {
        const T l = (c == 0) ? left : prv[L][c - 1];
        const T rr = (c == CPT2 - 1) ? right : prv[L][c + 1];
        const T ctr = prv[L][c];
        const T nb = (l + rr) + (pp[L][c] + cur[L][c]);
        v[c] = (rin && colin[c]) ? fma(r, fma(-four, ctr, nb), ctr) : T(0);
      }
      if (L + 1 < S) {
#pragma unroll
        for (int c = 0; c < CPT2; ++c) cur[L + 1][c] = v[c];
        st_edge(par, L + 1, v);
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
    if constexpr (TMA) {
      // the last row of a group has been read by every thread: refill its slot
      const int rr = yy - ys;
      if (rr % RB2 == RB2 - 1 && tid == 0) {
        const int g = rr / RB2 + D2<T>();
        if (ys + g * RB2 <= ye) tma_rows2<T>(&tmap, ring, bars, g % D2<T>(), x0, ys + g * RB2, (int)blockIdx.z);
      }
    }
  };
  using P0 = std::integral_constant<int, 0>;
  using P1 = std::integral_constant<int, 1>;
  using Steady = std::false_type;
  using Edge = std::true_type;
  int yy = ys;
  while (yy <= ye) {
    if (UNROLL && yy >= S && yy + 5 <= ny && yy + 5 <= ye) {
      // steady state: six rows per trip (three-row register rotation x two
      // buffer parities: the rotation is register renaming, not moves)
      row(P0{}, Steady{}, yy);
      row(P1{}, Steady{}, yy + 1);
      row(P0{}, Steady{}, yy + 2);
      row(P1{}, Steady{}, yy + 3);
      row(P0{}, Steady{}, yy + 4);
      row(P1{}, Steady{}, yy + 5);
      yy += 6;
    } else {
      row(P0{}, Edge{}, yy);
      if (yy + 1 > ye) break;
      row(P1{}, Edge{}, yy + 1);
      yy += 2;
    }
  }
}

// PINT_FE2D_VARIANT (measurement): 0 = rolled row loop, 1 = six-row steady
// unroll (no register cap), 2 = six-row unroll capped for 3 CTAs/SM (default:
// C3 fp64 +7 %, fp32 +10 % over 0, profiles/r01_fe2d_variants.jsonl),
// 3 = variant 2 with the TMA input ring, 4 = TMA ring capped for 2 CTAs/SM
int fe2d_variant() {
  const char *e = getenv("PINT_FE2D_VARIANT");
  return e ? atoi(e) : 3;  // TMA ring: C3 fp64 848 -> 1025 GPt/s, fp32 1399 -> 1407 (profiles/r02_fe2d_variants.jsonl)
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link)
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder2() {
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

template <typename T, int S, bool UNROLL, int MINB, bool TMA>
void launch2v(const T *in, T *out, int64_t nb, int64_t stride, int nx, int ny, T r, cudaStream_t st) {
  const unsigned tx = (unsigned)((nx + BX2 - 1) / BX2), ty = (unsigned)((ny + YC2 - 1) / YC2);
  const bool tma = TMA && ((uintptr_t)in & 15u) == 0 && (nx * sizeof(T)) % 16 == 0 && (stride * sizeof(T)) % 16 == 0;
  for (int64_t b0 = 0; b0 < nb; b0 += 65535) {
    const unsigned n = (unsigned)std::min<int64_t>(65535, nb - b0);
    CUtensorMap map;
    memset(&map, 0, sizeof(map));
    if (tma) {
      cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)n};
      cuuint64_t strides[2] = {(cuuint64_t)nx * sizeof(T), (cuuint64_t)stride * sizeof(T)};
      cuuint32_t box[3] = {(cuuint32_t)(W2 / 2), (cuuint32_t)RB2, 1};
      cuuint32_t es[3] = {1, 1, 1};
      const CUresult rc = tensor_map_encoder2()(
          &map, sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
          const_cast<T *>(in + b0 * stride), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (rc != CUDA_SUCCESS) pint_throw(PINT_ECUDA, "cuTensorMapEncodeTiled refused the row map");
      auto kern = fe2d_wave<T, S, UNROLL, MINB, true>;
      const int smem = D2<T>() * RB2 * W2 * (int)sizeof(T) + 8 * D2<T>();
      PINT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      kern<<<dim3(tx, ty, n), WT2, smem, st>>>(in + b0 * stride, out + b0 * stride, stride, nx, ny, r, map);
    } else {
      fe2d_wave<T, S, UNROLL, MINB, false><<<dim3(tx, ty, n), WT2, 0, st>>>(in + b0 * stride, out + b0 * stride,
                                                                            stride, nx, ny, r, map);
    }
  }
  PINT_CUDA(cudaGetLastError());
}

template <typename T, int S>
void launch2(const T *in, T *out, int64_t nb, int64_t stride, int nx, int ny, T r, cudaStream_t st) {
  switch (fe2d_variant()) {
    case 1: launch2v<T, S, true, 1, false>(in, out, nb, stride, nx, ny, r, st); break;
    case 2: launch2v<T, S, true, 3, false>(in, out, nb, stride, nx, ny, r, st); break;
    case 3: launch2v<T, S, true, 3, true>(in, out, nb, stride, nx, ny, r, st); break;
    case 4: launch2v<T, S, true, 2, true>(in, out, nb, stride, nx, ny, r, st); break;
    default: launch2v<T, S, false, 1, false>(in, out, nb, stride, nx, ny, r, st); break;
  }
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
// Same wavefront with z as the sweep axis. A CTA owns an xy tile of z-columns
// (64 columns x RW rows, including S halo cells per side) and a chunk of ZC3
// z planes; warp w owns tile row w and each lane two adjacent columns, so
// x-neighbours come from warp shuffles (lane +-1), y-neighbours from the rows
// above/below in a double-buffered shared tile (8-byte vector accesses, no
// bank conflicts) and z-neighbours from registers (three planes per level).
// One barrier per plane. HBM traffic 2*sizeof(T)/S bytes per update; the
// halo costs 64 RW / ((64 - 2S)(RW - 2S)) redundant xy updates and
// (ZC3 + 2S) / ZC3 in z. Values outside the domain are the Dirichlet zeros;
// out-of-tile neighbours read 0 (only halo cells see them).
namespace {

constexpr int SMAX3 = 4;
constexpr int CPT3 = 2;
constexpr int W3 = 32 * CPT3;  // tile columns (incl. halo)
constexpr int ZC3 = 128;       // output planes per chunk

// packed FP32 pairs (FADD2 / FFMA2 / FMUL2 on sm_100a): the two columns of
// a lane in one instruction, same per-element IEEE result as scalar code
__device__ __forceinline__ unsigned long long pk2(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 upk2(unsigned long long v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
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

template <typename T>
struct Pair;
template <>
struct Pair<float> { using V = float2; };
template <>
struct Pair<double> { using V = double2; };

// One plane of the wavefront (input plane zz arrives; level L+1 is advanced
// at plane zz-L-1). EDGE: some level's plane lies outside the domain (the
// first/last S planes of the sweep), so the plane mask is applied per level;
// PAR: shared buffer parity (compile time, the caller unrolls by two).
template <typename T, int S, int RW, bool EDGE, int PAR>
__device__ __forceinline__ void plane3(T (&cur)[S][CPT3], T (&prv)[S][CPT3], T (&pp)[S][CPT3], T (&pre)[CPT3],
                                       typename Pair<T>::V (*sm)[S][RW][32], int w, int w_up, int w_dn, int lane,
                                       const bool (&colin)[CPT3], const bool (&colout)[CPT3], int zz, int z0,
                                       int nz, int ze, const T *src, T *dst, int64_t plane, int64_t col, T r) {
  using V = typename Pair<T>::V;
  const T six = T(6);
#pragma unroll
  for (int c = 0; c < CPT3; ++c) cur[0][c] = pre[c];
  sm[PAR][0][w][lane] = V{cur[0][0], cur[0][1]};
  {
    const int zn = zz + 1;
    const bool pin = zn >= 0 && zn < nz && zn <= ze;
#pragma unroll
    for (int c = 0; c < CPT3; ++c) pre[c] = (pin && colin[c]) ? __ldg(src + (int64_t)zn * plane + col + c) : T(0);
  }
#pragma unroll
  for (int L = 0; L < S; ++L) {
    const int zr = zz - L - 1;
    const bool rin = !EDGE || (zr >= 0 && zr < nz);
    // out-of-tile neighbours (lane 0/31 shuffles, clamped rows) are garbage
    // that only reaches halo cells
    const T left = __shfl_up_sync(0xffffffffu, prv[L][CPT3 - 1], 1);
    const T right = __shfl_down_sync(0xffffffffu, prv[L][0], 1);
    const V up = sm[PAR ^ 1][L][w_up][lane];
    const V dn = sm[PAR ^ 1][L][w_dn][lane];
    T v[CPT3];
    if constexpr (sizeof(T) == 4) {
      // ((xl + xr) + (up + dn)) + (pz + nz), then ctr + r (nb - 6 ctr): the scalar path's order
      const unsigned long long ctr = pk2(prv[L][0], prv[L][1]);
      const unsigned long long nb = add2(add2(add2(pk2(left, prv[L][0]), pk2(prv[L][1], right)),
                                              add2(pk2(up.x, up.y), pk2(dn.x, dn.y))),
                                         add2(pk2(pp[L][0], pp[L][1]), pk2(cur[L][0], cur[L][1])));
      const unsigned long long t = fma2(pk2(-six, -six), ctr, nb);
      unsigned long long vv = fma2(pk2(r, r), t, ctr);
      const float m0 = (rin && colin[0]) ? 1.0f : 0.0f, m1 = (rin && colin[1]) ? 1.0f : 0.0f;
      vv = mul2(vv, pk2(m0, m1));
      const float2 f = upk2(vv);
      v[0] = f.x;
      v[1] = f.y;
    } else {
      const T upv[2] = {up.x, up.y}, dnv[2] = {dn.x, dn.y};
#pragma unroll
      for (int c = 0; c < CPT3; ++c) {
        const T ctr = prv[L][c];
        const T xl = (c == 0) ? left : prv[L][c - 1];
        const T xr = (c == CPT3 - 1) ? right : prv[L][c + 1];
        const T nb = ((xl + xr) + (upv[c] + dnv[c])) + (pp[L][c] + cur[L][c]);
        v[c] = (rin && colin[c]) ? fma(r, fma(-six, ctr, nb), ctr) : T(0);
      }
    }
    if (L + 1 < S) {
#pragma unroll
      for (int c = 0; c < CPT3; ++c) cur[L + 1][c] = v[c];
      sm[PAR][L + 1][w][lane] = V{v[0], v[1]};
    } else if (zr >= z0 && zr < z0 + ZC3 && rin) {
#pragma unroll
      for (int c = 0; c < CPT3; ++c)
        if (colout[c]) dst[(int64_t)zr * plane + col + c] = v[c];
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

template <typename T, int S, int RW>
__global__ void __launch_bounds__(32 * RW)
fe3d_wave(const T *__restrict__ in, T *__restrict__ out, int64_t stride, int nx, int ny, int nz, T r, int tiles_x) {
  using V = typename Pair<T>::V;
  extern __shared__ __align__(16) unsigned char smraw3[];
  V(*sm)[S][RW][32] = reinterpret_cast<V(*)[S][RW][32]>(smraw3);  // [par][level][row][lane] pairs
  constexpr int BX = W3 - 2 * S, BY = RW - 2 * S;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int w_up = w > 0 ? w - 1 : 0, w_dn = w < RW - 1 ? w + 1 : RW - 1;
  const int bx = blockIdx.x % tiles_x, by = blockIdx.x / tiles_x;
  const int x0 = bx * BX - S, y0 = by * BY - S, z0 = blockIdx.y * ZC3;
  const int64_t plane = (int64_t)nx * ny;
  const T *src = in + (int64_t)blockIdx.z * stride;
  T *dst = out + (int64_t)blockIdx.z * stride;
  const int cx = x0 + CPT3 * lane, cy = y0 + w;
  bool colin[CPT3], colout[CPT3];
#pragma unroll
  for (int c = 0; c < CPT3; ++c) {
    colin[c] = cx + c >= 0 && cx + c < nx && cy >= 0 && cy < ny;
    const int lx = CPT3 * lane + c;
    colout[c] = colin[c] && lx >= S && lx < S + BX && w >= S && w < S + BY;
  }
  T cur[S][CPT3], prv[S][CPT3], pp[S][CPT3];
#pragma unroll
  for (int L = 0; L < S; ++L)
#pragma unroll
    for (int c = 0; c < CPT3; ++c) cur[L][c] = prv[L][c] = pp[L][c] = T(0);
  // both parities of every level start at 0 (the first planes read them)
  for (int i = threadIdx.x; i < 2 * S * RW * 32; i += 32 * RW) (&sm[0][0][0][0])[i] = V{T(0), T(0)};
  __syncthreads();
  const int zs = z0 - S, ze = min(z0 + ZC3, nz) - 1 + S;
  const int64_t col = (int64_t)cy * nx + cx;
  T pre[CPT3];  // next input plane, prefetched one iteration ahead
  {
    const bool pin = zs >= 0 && zs < nz;
#pragma unroll
    for (int c = 0; c < CPT3; ++c) pre[c] = (pin && colin[c]) ? __ldg(src + (int64_t)zs * plane + col + c) : T(0);
  }
  // planes zz in [S, nz] have every level's plane inside the domain
  for (int zz = zs; zz <= ze; zz += 2) {
    if (zz >= S && zz + 1 <= nz)
      plane3<T, S, RW, false, 0>(cur, prv, pp, pre, sm, w, w_up, w_dn, lane, colin, colout, zz, z0, nz, ze, src, dst,
                                 plane, col, r);
    else
      plane3<T, S, RW, true, 0>(cur, prv, pp, pre, sm, w, w_up, w_dn, lane, colin, colout, zz, z0, nz, ze, src, dst,
                                plane, col, r);
    if (zz + 1 > ze) break;
    if (zz + 1 >= S && zz + 1 <= nz)
      plane3<T, S, RW, false, 1>(cur, prv, pp, pre, sm, w, w_up, w_dn, lane, colin, colout, zz + 1, z0, nz, ze, src,
                                 dst, plane, col, r);
    else
      plane3<T, S, RW, true, 1>(cur, prv, pp, pre, sm, w, w_up, w_dn, lane, colin, colout, zz + 1, z0, nz, ze, src,
                                dst, plane, col, r);
  }
}

template <typename T, int S>
void launch3(const T *in, T *out, int64_t nb, int64_t stride, int nx, int ny, int nz, T r, cudaStream_t st) {
  // fp32: 32 rows (1024 threads); fp64: 16 rows (register budget)
  constexpr int RW = sizeof(T) == 4 ? 32 : 16;
  constexpr int BX = W3 - 2 * S, BY = RW - 2 * S;
  const int tiles_x = (nx + BX - 1) / BX, tiles_y = (ny + BY - 1) / BY;
  const unsigned tz = (unsigned)((nz + ZC3 - 1) / ZC3);
  const size_t smem = sizeof(T) * 2 * 2 * S * RW * 32;
  PINT_CUDA(cudaFuncSetAttribute(fe3d_wave<T, S, RW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  for (int64_t b0 = 0; b0 < nb; b0 += 65535) {
    const unsigned n = (unsigned)std::min<int64_t>(65535, nb - b0);
    fe3d_wave<T, S, RW><<<dim3((unsigned)(tiles_x * tiles_y), tz, n), 32 * RW, smem, st>>>(
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
