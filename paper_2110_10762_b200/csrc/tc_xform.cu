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
#include <cstring>
#include <vector>

#include "pint_internal.cuh"

namespace {

constexpr int TM = 128;            // tile rows (TMEM lanes, UMMA M)
constexpr int TN = 128;            // tile columns per parity (UMMA N)
constexpr int BK = 8;              // K per stage = one UMMA K-step of tf32
constexpr int TILE = 2 * TM * 16;  // one operand tile: 2 K chunks x 128 rows x 16 B = 4 KB
// stage: [data: X0h X0l X1h X1l][constant Q: Q0h Q0l Q1h Q1l], 32 KB
constexpr int STAGE = 8 * TILE;
constexpr int QBLK = 4 * TILE;     // constant tiles of one K block (one bulk copy)
// raw data ring: each thread streams its own row (FOLD 1) / column (FOLD 2)
// of RAWS K blocks ahead with cp.async (forward + reversed 8 values = 64 B
// per thread per block), then folds and splits from shared memory
constexpr int RAWS = 6;
constexpr int RAWB = 128 * 64;  // one K block of raw data for the CTA (8 KB)
constexpr int RAW_OFF = 2 * STAGE + 64;
// 2 x 32 KB UMMA stages + barriers + 48 KB ring = 112 KB: two CTAs per SM,
// exactly the TMEM they need (2 x 256 columns)
constexpr int SMEM = RAW_OFF + RAWS * RAWB;

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

// four consecutive K values of one row -> hi / lo 16-byte chunks of two tiles
__device__ __forceinline__ void put4(uint32_t tile_hi, uint32_t tile_lo, int kc, int row, const float *v) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) split_tf32(v[i], h[i], l[i]);
  const uint32_t off = (uint32_t)kc * (TM * 16) + (uint32_t)row * 16;
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(tile_hi + off), "r"(h[0]), "r"(h[1]), "r"(h[2]),
               "r"(h[3]) : "memory");
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(tile_lo + off), "r"(l[0]), "r"(l[1]), "r"(l[2]),
               "r"(l[3]) : "memory");
}

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr) {
  // SWIZZLE_NONE, K-major: LBO = distance between the two 16-byte K chunks
  // (2048 B), SBO = distance between 8-row core-matrix groups (128 B),
  // descriptor version 1 (sm_100)
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)(((TM * 16) >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((128 >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

// kind::tf32, D fp32, A/B tf32 K-major, M = 128, N = 128
constexpr uint32_t IDESC =
    (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TN >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);

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
  const float *src;     // the data operand: A (FOLD 1) or the z planes of B (FOLD 2)
  const uint32_t *qs;   // constant operand, pre-split tf32 tiles [qblock][kblock][p][hi|lo][kc][row][4]
  float *dst;
  int n;                // transform length
  int kh;               // folded K = n / 2
  int rows;             // FOLD 1: source rows (M); FOLD 2: columns per plane (= n)
  int64_t plane;        // FOLD 2: elements per z plane (n * n)
};

template <int FOLD>
__global__ void __launch_bounds__(128, 2) xform_tc(const TcArgs g) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint64_t *bars = reinterpret_cast<uint64_t *>(sm + 2 * STAGE);  // full[2], empty[2]
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(sm + 2 * STAGE + 32);
  const int n = g.n, kh = g.kh, half = n / 2, nkb = kh / BK;
  const int m0 = blockIdx.x * TM;   // FOLD 1: source rows;  FOLD 2: q (output row pairs)
  const int c0 = blockIdx.y * TN;   // FOLD 1: q (output column pairs);  FOLD 2: x
  const float *src = g.src + (FOLD == 2 ? (int64_t)blockIdx.z * g.plane : 0);
  float *dst = g.dst + (FOLD == 2 ? (int64_t)blockIdx.z * g.plane : 0);
  // the constant operand's tile rows are the output pairs q of this CTA
  const uint8_t *qblk = reinterpret_cast<const uint8_t *>(g.qs) +
                        (size_t)((FOLD == 1 ? c0 : m0) / TM) * nkb * QBLK;
  const uint32_t s_base = smem_addr(sm);
  const uint32_t full0 = smem_addr(&bars[0]), empty0 = smem_addr(&bars[2]);

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_addr(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < 4; ++i) mbar_init1(smem_addr(&bars[i]));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t *>(tmem_slot);

  // raw ring: K block slot = 4 chunks of 16 B per thread, chunk-major
  // ([chunk][thread][16 B]) so the fold's 16-byte reads are conflict-free.
  // chunks: 0, 1 = values k0..k0+7; 2, 3 = the mirrored values
  // (FOLD 1: A[m][n-8-k0 .. n-1-k0] in memory order; FOLD 2: B[n-1-k0-i][x], i = 0..7)
  const uint32_t raw_base = s_base + (uint32_t)RAW_OFF + (uint32_t)tid * 16u;
  auto issue = [&](int kb) {  // cp.async of K block kb into ring slot kb % RAWS (always commits a group)
    if (kb < nkb) {
      const int k0 = kb * BK;
      const uint32_t dst = raw_base + (uint32_t)((kb % RAWS) * RAWB);
      if (FOLD == 1) {  // thread = source row m
        const int m = m0 + tid;
        if (m < g.rows) {
          const float *row = src + (int64_t)m * n;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(row + k0) : "memory");
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 2048u), "l"(row + k0 + 4)
                       : "memory");
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 4096u), "l"(row + n - 8 - k0)
                       : "memory");
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 6144u), "l"(row + n - 4 - k0)
                       : "memory");
        }
      } else {  // thread = column x
        const int x = c0 + tid;
        if (x < g.rows) {
#pragma unroll
          for (int i = 0; i < BK; ++i) {
            const uint32_t o = (uint32_t)(i / 4) * 2048u + 4u * (uint32_t)(i % 4);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst + o),
                         "l"(src + (int64_t)(k0 + i) * n + x) : "memory");
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst + 4096u + o),
                         "l"(src + (int64_t)(n - 1 - k0 - i) * n + x) : "memory");
          }
        }
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  // fold K block kb from the ring: d0 = f + r, d1 = f - r
  float d0[BK], d1[BK];
  auto fold = [&](int kb) {
    const uint8_t *rb = sm + RAW_OFF + (kb % RAWS) * RAWB + tid * 16;
    const bool ok = FOLD == 1 ? (m0 + tid < g.rows) : (c0 + tid < g.rows);
    float v[16];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const float4 q = *reinterpret_cast<const float4 *>(rb + c * 2048);
      v[4 * c] = q.x;
      v[4 * c + 1] = q.y;
      v[4 * c + 2] = q.z;
      v[4 * c + 3] = q.w;
    }
#pragma unroll
    for (int i = 0; i < BK; ++i) {
      const float f = ok ? v[i] : 0.0f;
      const float r = ok ? (FOLD == 1 ? v[8 + (BK - 1 - i)] : v[8 + i]) : 0.0f;
      d0[i] = f + r;
      d1[i] = f - r;
    }
  };

  for (int q = 0; q < RAWS - 1; ++q) issue(q);
  for (int t = 0; t < nkb; ++t) {
    const int s = t & 1;
    const uint32_t st = s_base + (uint32_t)(s * STAGE);
    issue(t + RAWS - 1);  // keep RAWS - 1 K blocks in flight
    asm volatile("cp.async.wait_group %0;" ::"n"(RAWS - 1) : "memory");  // block t (this thread's copies) landed
    fold(t);
    if (t >= 2) mbar_wait(empty0 + 8u * s, (uint32_t)(((t - 2) >> 1) & 1));
    if (tid == 0) {  // constant tiles of this K block: one bulk copy (TMA engine)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(full0 + 8u * s), "r"(QBLK)
                   : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              st + 4u * TILE),
          "l"(qblk + (size_t)t * QBLK), "r"(QBLK), "r"(full0 + 8u * s)
          : "memory");
    }
#pragma unroll
    for (int kc = 0; kc < 2; ++kc) {
      put4(st + 0u * TILE, st + 1u * TILE, kc, tid, d0 + 4 * kc);
      put4(st + 2u * TILE, st + 3u * TILE, kc, tid, d1 + 4 * kc);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      mbar_wait(full0 + 8u * s, (uint32_t)((t >> 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        const uint32_t d = tmem + (uint32_t)(p * TN);
        const uint32_t xh = st + (uint32_t)(2 * p) * TILE, xl = xh + TILE;          // data tiles
        const uint32_t qh = st + (uint32_t)(4 + 2 * p) * TILE, ql = qh + TILE;      // constant tiles
        // FOLD 1: A = data (rows m), B = Q (rows q); FOLD 2: A = Q (rows q), B = data (rows x)
        const uint64_t ah = make_desc(FOLD == 1 ? xh : qh), al = make_desc(FOLD == 1 ? xl : ql);
        const uint64_t bh = make_desc(FOLD == 1 ? qh : xh), bl = make_desc(FOLD == 1 ? ql : xl);
        const uint32_t acc0 = t > 0 ? 1u : 0u;
        mma_tf32(d, al, bh, acc0);  // small terms first
        mma_tf32(d, ah, bl, 1u);
        mma_tf32(d, ah, bh, 1u);
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       empty0 + 8u * s)
                   : "memory");
    }
  }
  // all MMAs of thread 0 complete with its last commit
  mbar_wait(empty0 + 8u * ((nkb - 1) & 1), (uint32_t)(((nkb - 1) >> 1) & 1));
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
          __stcs(out + j / 2, make_float4(__uint_as_float(v[0][j]), __uint_as_float(v[1][j]),
                                          __uint_as_float(v[0][j + 1]), __uint_as_float(v[1][j + 1])));
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
            __stcs(out + j / 4, make_float4(__uint_as_float(v[p][j]), __uint_as_float(v[p][j + 1]),
                                            __uint_as_float(v[p][j + 2]), __uint_as_float(v[p][j + 3])));
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

}  // namespace

// Eligible shapes: n a multiple of 256 (output pairs in whole 128-row
// tiles, kh = n/2 a multiple of the K block).
bool tc_xform_supported(int n) { return n >= 256 && n % 256 == 0; }

// The constant operand, split once on the host from the long-double sine
// transform (better than splitting its fp32 rounding): tiles
// [q block][k block][parity][hi|lo][kc][row q][4 k], tf32 bit patterns.
// Qh[p][k][q] = Q[k][2q + p] (FOLD 1 B, rows q) equals QhT[p][q][k] (FOLD 2 A).
static uint32_t tf32_rna(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) return u;
  return (u + 0x1000u) & 0xffffe000u;
}
std::vector<uint32_t> tc_split_q(int n, const long double *q) {
  const int half = n / 2, kh = n / 2, nqb = half / TM, nkb = kh / BK;
  std::vector<uint32_t> out((size_t)nqb * nkb * QBLK / 4);
  for (int qb = 0; qb < nqb; ++qb)
    for (int kb = 0; kb < nkb; ++kb)
      for (int p = 0; p < 2; ++p)
        for (int hl = 0; hl < 2; ++hl)
          for (int kc = 0; kc < 2; ++kc)
            for (int r = 0; r < TM; ++r)
              for (int e = 0; e < 4; ++e) {
                const int k = kb * BK + kc * 4 + e, qq = qb * TM + r;
                const long double v = q[(size_t)k * n + 2 * qq + p];
                const uint32_t hbits = tf32_rna((float)v);
                float hf;
                memcpy(&hf, &hbits, 4);
                const uint32_t bits = hl == 0 ? hbits : tf32_rna((float)(v - (long double)hf));
                const size_t idx = ((((((size_t)qb * nkb + kb) * 2 + p) * 2 + hl) * 2 + kc) * TM + r) * 4 + e;
                out[idx] = bits;
              }
  return out;
}

// dst = src Q along the fastest axis (rows x n, row-major)
void tc_xform_last(const float *src, float *dst, const uint32_t *qs, int n, int64_t rows, cudaStream_t s) {
  TcArgs g{src, qs, dst, n, n / 2, (int)rows, 0};
  PINT_CUDA(cudaFuncSetAttribute(xform_tc<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
  dim3 grid((unsigned)((rows + TM - 1) / TM), (unsigned)(n / 2 / TN), 1);
  xform_tc<1><<<grid, 128, SMEM, s>>>(g);
  PINT_CUDA(cudaGetLastError());
}

// dst_z = Q src_z for each of the `planes` n x n planes
void tc_xform_mid(const float *src, float *dst, const uint32_t *qs, int n, int planes, cudaStream_t s) {
  TcArgs g{src, qs, dst, n, n / 2, n, (int64_t)n * n};
  PINT_CUDA(cudaFuncSetAttribute(xform_tc<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
  dim3 grid((unsigned)(n / 2 / TM), (unsigned)(n / TN), (unsigned)planes);
  xform_tc<2><<<grid, 128, SMEM, s>>>(g);
  PINT_CUDA(cudaGetLastError());
}
