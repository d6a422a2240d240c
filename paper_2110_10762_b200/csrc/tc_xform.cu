// Sine-transform GEMMs of the direct 2-D/3-D coarse solve (spectral.cu) on
// the 5th-generation tensor cores, fp32 data in 3xTF32 (split) precision.
//
// Each transform is C = A' B' with the parity fold of the sine transform
// (spectral.cu, GemmArgs): for every output parity p the K extent is halved,
//   FOLD 1 (transform along the fastest axis, "xform_last"):
//        A'_p[m][k] = A[m][k] +- A[m][n-1-k],  B_p = Qh[p] (kh x n/2), out column 2q + p
//   FOLD 2 (transform along the middle axis, per z plane, "xform_mid"):
//        A_p = QhT[p] (n/2 x kh),  B'_p[k][x] = B[k][x] +- B[n-1-k][x],  out row 2q + p
// One CTA computes one 128 x 128 output tile for BOTH parities (two TMEM
// accumulators, 256 columns), so it reads the source once and writes whole
// output rows.
//
// Precision: every fp32 operand is split a = hi + lo with hi = tf32(a) and
// lo = tf32(a - hi); D += lo_A hi_B + hi_A lo_B + hi_A hi_B (fp32 accumulate
// in TMEM). The dropped lo_A lo_B term and the tf32 rounding of lo are below
// 2^-21 relative per product — fp32-level accuracy, which plain TF32 (2^-11)
// would not give.
//
// Pipeline (canonical sm_100 structure, one CTA of 4 warps): all threads load
// a 16-deep K block from global memory (folding on the way), split it and
// store it into a double-buffered shared stage in the UMMA no-swizzle
// K-major layout (core matrices of 8 rows x 16 B; K chunks 2048 B apart =
// LBO, 8-row groups 128 B apart = SBO); one elected thread issues the
// tcgen05.mma instructions and a tcgen05.commit onto the stage's mbarrier,
// which the loaders wait on before refilling that stage. The epilogue reads
// the accumulators with tcgen05.ld (warp w owns TMEM lanes 32w..32w+31) and
// stores whole rows.
#include <cuda_runtime.h>

#include <cstdint>

#include "pint_internal.cuh"

namespace {

constexpr int TM = 128;           // output rows per tile (TMEM lanes, UMMA M)
constexpr int TN = 128;           // output columns per parity (UMMA N)
constexpr int BK = 16;            // K per stage (two UMMA K-steps of 8 tf32)
constexpr int KC = BK / 4;        // 16-byte K chunks per stage
constexpr int OPB = KC * TM * 16; // bytes of one operand tile (128 rows x 16 K) = 8 KB
// stage layout: [A0h A0l A1h A1l B0h B0l B1h B1l], 8 operand tiles = 64 KB
constexpr int STAGE = 8 * OPB;
constexpr int SMEM = 2 * STAGE + 64;  // + mbarriers and the TMEM base

__device__ __forceinline__ uint32_t smem_addr(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void split_tf32(float a, uint32_t &hi, uint32_t &lo) {
  uint32_t h, l;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(a));
  const float r = a - __uint_as_float(h);
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(l) : "f"(r));
  hi = h;
  lo = l;
}

// four consecutive K values of one row -> hi / lo 16-byte chunks of an operand tile
__device__ __forceinline__ void put4(uint8_t *tile_hi, uint8_t *tile_lo, int kc, int row, const float (&v)[4]) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) split_tf32(v[i], h[i], l[i]);
  const uint32_t off = (uint32_t)kc * (TM * 16) + (uint32_t)row * 16;
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(smem_addr(tile_hi + off)), "r"(h[0]), "r"(h[1]),
               "r"(h[2]), "r"(h[3]) : "memory");
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(smem_addr(tile_lo + off)), "r"(l[0]), "r"(l[1]),
               "r"(l[2]), "r"(l[3]) : "memory");
}

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr) {
  // SWIZZLE_NONE, K-major: LBO = distance between the two 16-byte K chunks of
  // an MMA (2048 B), SBO = distance between 8-row core-matrix groups (128 B),
  // descriptor version 1 (sm_100)
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)(((TM * 16) >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((128 >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

// kind::tf32, D fp32, A/B tf32 K-major, M = 128, N = 128
constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TN >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(IDESC), "r"(accumulate));
}

__device__ __forceinline__ void mbar_init1(uint32_t bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

struct TcArgs {
  const float *src;   // A (FOLD 1) or B (FOLD 2) of the transform
  const float *h0;    // Qh[0] (FOLD 1: kh x n/2) or QhT[0] (FOLD 2: n/2 x kh)
  const float *h1;
  float *dst;
  int n;              // transform length (even)
  int kh;             // folded K = n / 2
  int rows;           // FOLD 1: source rows (M); FOLD 2: columns per plane (= n)
  int64_t plane;      // FOLD 2: elements per z plane (n * n)
};

template <int FOLD>
__global__ void __launch_bounds__(128, 1) xform_tc(const TcArgs g) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint64_t *bars = reinterpret_cast<uint64_t *>(sm + 2 * STAGE);
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(sm + 2 * STAGE + 32);
  const int n = g.n, kh = g.kh, half = n / 2;
  // tile coordinates
  const int m0 = blockIdx.x * TM;   // FOLD 1: source rows; FOLD 2: q (output row pairs)
  const int c0 = blockIdx.y * TN;   // FOLD 1: q (output column pairs); FOLD 2: x
  const int z = blockIdx.z;         // FOLD 2: plane
  const float *src = g.src + (FOLD == 2 ? (int64_t)z * g.plane : 0);
  float *dst = g.dst + (FOLD == 2 ? (int64_t)z * g.plane : 0);

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_addr(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init1(smem_addr(&bars[0]));
    mbar_init1(smem_addr(&bars[1]));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t *>(tmem_slot);

  const int nk = kh / BK;
  for (int t = 0; t < nk; ++t) {
    const int s = t & 1;
    const int k0 = t * BK;
    // ---- global loads of K block t (thread = one operand row)
    float a0[BK], a1[BK], b0[BK], b1[BK];
    if (FOLD == 1) {
      const int m = m0 + tid;
      if (m < g.rows) {
        const float *row = src + (int64_t)m * n;
#pragma unroll
        for (int i = 0; i < BK; i += 4) {
          const float4 f = *reinterpret_cast<const float4 *>(row + k0 + i);
          const float4 r = *reinterpret_cast<const float4 *>(row + n - 4 - k0 - i);  // A[n-1-k] for k = k0+i..+3
          const float fv[4] = {f.x, f.y, f.z, f.w}, rv[4] = {r.w, r.z, r.y, r.x};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            a0[i + j] = fv[j] + rv[j];
            a1[i + j] = fv[j] - rv[j];
          }
        }
      } else {
#pragma unroll
        for (int i = 0; i < BK; ++i) a0[i] = a1[i] = 0.0f;
      }
      // B_p[k][q]: thread = output column pair q (row of the K-major B tile)
      const int q = c0 + tid;
#pragma unroll
      for (int i = 0; i < BK; ++i) {
        b0[i] = q < half ? __ldg(g.h0 + (int64_t)(k0 + i) * half + q) : 0.0f;
        b1[i] = q < half ? __ldg(g.h1 + (int64_t)(k0 + i) * half + q) : 0.0f;
      }
    } else {
      // A_p[q][k] = QhT[p][q][k]: thread = output row pair q
      const int q = m0 + tid;
      if (q < half) {
#pragma unroll
        for (int i = 0; i < BK; i += 4) {
          const float4 u = *reinterpret_cast<const float4 *>(g.h0 + (int64_t)q * kh + k0 + i);
          const float4 v = *reinterpret_cast<const float4 *>(g.h1 + (int64_t)q * kh + k0 + i);
          a0[i] = u.x; a0[i + 1] = u.y; a0[i + 2] = u.z; a0[i + 3] = u.w;
          a1[i] = v.x; a1[i + 1] = v.y; a1[i + 2] = v.z; a1[i + 3] = v.w;
        }
      } else {
#pragma unroll
        for (int i = 0; i < BK; ++i) a0[i] = a1[i] = 0.0f;
      }
      // B'_p[k][x] = B[k][x] +- B[n-1-k][x]: thread = column x
      const int x = c0 + tid;
#pragma unroll
      for (int i = 0; i < BK; ++i) {
        float f = 0.0f, r = 0.0f;
        if (x < g.rows) {
          f = src[(int64_t)(k0 + i) * n + x];
          r = src[(int64_t)(n - 1 - k0 - i) * n + x];
        }
        b0[i] = f + r;
        b1[i] = f - r;
      }
    }
    // ---- the stage is free once the MMAs of block t-2 have completed
    if (t >= 2) mbar_wait(smem_addr(&bars[s]), (uint32_t)(((t - 2) >> 1) & 1));
    uint8_t *st = sm + s * STAGE;
#pragma unroll
    for (int kc = 0; kc < KC; ++kc) {
      const float va0[4] = {a0[4 * kc], a0[4 * kc + 1], a0[4 * kc + 2], a0[4 * kc + 3]};
      const float va1[4] = {a1[4 * kc], a1[4 * kc + 1], a1[4 * kc + 2], a1[4 * kc + 3]};
      const float vb0[4] = {b0[4 * kc], b0[4 * kc + 1], b0[4 * kc + 2], b0[4 * kc + 3]};
      const float vb1[4] = {b1[4 * kc], b1[4 * kc + 1], b1[4 * kc + 2], b1[4 * kc + 3]};
      put4(st + 0 * OPB, st + 1 * OPB, kc, tid, va0);
      put4(st + 2 * OPB, st + 3 * OPB, kc, tid, va1);
      put4(st + 4 * OPB, st + 5 * OPB, kc, tid, vb0);
      put4(st + 6 * OPB, st + 7 * OPB, kc, tid, vb1);
    }
    // generic-proxy smem writes -> visible to the tensor core (async proxy)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t base = smem_addr(st);
#pragma unroll
      for (int ks = 0; ks < BK / 8; ++ks) {
        const uint32_t koff = (uint32_t)(2 * ks) * (TM * 16);
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          const uint32_t d = tmem + (uint32_t)(p * TN);
          const uint64_t ah = make_desc(base + (uint32_t)((2 * p) * OPB) + koff);
          const uint64_t al = make_desc(base + (uint32_t)((2 * p + 1) * OPB) + koff);
          const uint64_t bh = make_desc(base + (uint32_t)((4 + 2 * p) * OPB) + koff);
          const uint64_t bl = make_desc(base + (uint32_t)((5 + 2 * p) * OPB) + koff);
          const uint32_t acc0 = (t > 0 || ks > 0) ? 1u : 0u;
          mma_tf32(d, al, bh, acc0);  // small terms first
          mma_tf32(d, ah, bl, 1u);
          mma_tf32(d, ah, bh, 1u);
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_addr(&bars[s]))
                   : "memory");
    }
  }
  // ---- all MMAs issued by thread 0 complete with the last commit
  mbar_wait(smem_addr(&bars[(nk - 1) & 1]), (uint32_t)(((nk - 1) >> 1) & 1));
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

  // ---- epilogue: warp w owns TMEM lanes (tile rows) 32w .. 32w+31
  const int r = warp * 32 + lane;
  const uint32_t lane_base = tmem + ((uint32_t)(warp * 32) << 16);
#pragma unroll 1
  for (int cc = 0; cc < TN; cc += 32) {
    uint32_t v[2][32];
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      const uint32_t a = lane_base + (uint32_t)(p * TN + cc);
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
          "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
          : "=r"(v[p][0]), "=r"(v[p][1]), "=r"(v[p][2]), "=r"(v[p][3]), "=r"(v[p][4]), "=r"(v[p][5]),
            "=r"(v[p][6]), "=r"(v[p][7]), "=r"(v[p][8]), "=r"(v[p][9]), "=r"(v[p][10]), "=r"(v[p][11]),
            "=r"(v[p][12]), "=r"(v[p][13]), "=r"(v[p][14]), "=r"(v[p][15]), "=r"(v[p][16]), "=r"(v[p][17]),
            "=r"(v[p][18]), "=r"(v[p][19]), "=r"(v[p][20]), "=r"(v[p][21]), "=r"(v[p][22]), "=r"(v[p][23]),
            "=r"(v[p][24]), "=r"(v[p][25]), "=r"(v[p][26]), "=r"(v[p][27]), "=r"(v[p][28]), "=r"(v[p][29]),
            "=r"(v[p][30]), "=r"(v[p][31])
          : "r"(a));
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (FOLD == 1) {
      // row m, columns 2q + p for q = c0 + cc .. +31: 64 contiguous floats
      const int m = m0 + r;
      if (m < g.rows && c0 + cc < half) {
        float4 *out = reinterpret_cast<float4 *>(dst + (int64_t)m * n + 2 * (c0 + cc));
#pragma unroll
        for (int j = 0; j < 32; j += 2)
          out[j / 2] = make_float4(__uint_as_float(v[0][j]), __uint_as_float(v[1][j]), __uint_as_float(v[0][j + 1]),
                                   __uint_as_float(v[1][j + 1]));
      }
    } else {
      // rows 2q + p, columns x = c0 + cc .. +31
      const int q = m0 + r;
      if (q < half && c0 + cc < g.rows) {
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          float4 *out = reinterpret_cast<float4 *>(dst + (int64_t)(2 * q + p) * n + c0 + cc);
#pragma unroll
          for (int j = 0; j < 32; j += 4)
            out[j / 4] = make_float4(__uint_as_float(v[p][j]), __uint_as_float(v[p][j + 1]),
                                     __uint_as_float(v[p][j + 2]), __uint_as_float(v[p][j + 3]));
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

}  // namespace

// Eligible shapes: n a multiple of 64 (kh = n/2 a multiple of the 16-deep K
// stage, output pairs in whole 32-column epilogue chunks).
bool tc_xform_supported(int n) { return n >= 64 && n % 64 == 0; }

// dst = src Q along the fastest axis (rows x n, row-major), Q the folded sine transform
void tc_xform_last(const float *src, float *dst, const float *qh0, const float *qh1, int n, int64_t rows,
                   cudaStream_t s) {
  TcArgs g{src, qh0, qh1, dst, n, n / 2, (int)rows, 0};
  PINT_CUDA(cudaFuncSetAttribute(xform_tc<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
  dim3 grid((unsigned)((rows + TM - 1) / TM), (unsigned)((n / 2 + TN - 1) / TN), 1);
  xform_tc<1><<<grid, 128, SMEM, s>>>(g);
  PINT_CUDA(cudaGetLastError());
}

// dst_z = Q src_z for each of the `planes` n x n planes
void tc_xform_mid(const float *src, float *dst, const float *qt0, const float *qt1, int n, int planes,
                  cudaStream_t s) {
  TcArgs g{src, qt0, qt1, dst, n, n / 2, n, (int64_t)n * n};
  PINT_CUDA(cudaFuncSetAttribute(xform_tc<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
  dim3 grid((unsigned)((n / 2 + TM - 1) / TM), (unsigned)((n + TN - 1) / TN), (unsigned)planes);
  xform_tc<2><<<grid, 128, SMEM, s>>>(g);
  PINT_CUDA(cudaGetLastError());
}
