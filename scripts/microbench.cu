// Microbenchmarks of the latencies that bound the 1-D fine kernel's step
// (B200, sm_100a): dependent DFMA, 64-bit shuffle, DSMEM st.async +
// mbarrier round trip in an 8-CTA cluster, FP64 FMA throughput per SM.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a scripts/microbench.cu -o /tmp/mb && /tmp/mb
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void dfma_chain(double *out, long long *cyc, double a, double b) {
  double x = threadIdx.x;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < 4096; ++i) x = fma(x, a, b);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

__global__ void shfl_chain(double *out, long long *cyc) {
  double x = threadIdx.x;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < 4096; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1) + 1.0;
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

__global__ void dfma_tput(double *out, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < 8192; ++i) {
    x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
    x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// ping-pong exchange: every CTA of the cluster writes one value to every CTA
// (lane c -> rank c), then waits on its own mbarrier for all CL values.
__global__ void __cluster_dims__(8, 1, 1) cluster_exchange(long long *cyc, int iters) {
  __shared__ alignas(8) unsigned long long bar[2];
  __shared__ double buf[2][64];
  cg::cluster_group cluster = cg::this_cluster();
  const int CL = 8;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar[0])), "r"(1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar[1])), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  cluster.sync();
  const int rank = cluster.block_rank();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const uint32_t par = it & 1;
    const uint32_t gb = smem_u32(&buf[par][0]);
    const uint32_t b = smem_u32(&bar[par]);
    if (lane < CL) {
      uint32_t rgb, rb;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rgb) : "r"(gb), "r"(lane));
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(b), "r"(lane));
      const uint32_t o = (uint32_t)(rank * nwarps + warp) * 8u;
      asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(rgb + o),
                   "l"((long long)it), "r"(rb) : "memory");
    }
    if (threadIdx.x == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(CL * nwarps * 8) : "memory");
    asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n}" ::"r"(b),
                 "r"((it >> 1) & 1) : "memory");
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = (t1 - t0) / iters;
  cluster.sync();
}

int main() {
  double *out;
  long long *cyc, h;
  cudaMalloc(&out, 1 << 24);
  cudaMalloc(&cyc, 8);
  dfma_chain<<<1, 32>>>(out, cyc, 1.0000001, 1e-9);
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("dependent DFMA latency: %.2f cycles\n", h / 4096.0);
  shfl_chain<<<1, 32>>>(out, cyc);
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("dependent SHFL(f64)+DADD latency: %.2f cycles\n", h / 4096.0);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    dfma_tput<<<sms * 4, 256>>>(out, 1.0000001, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
  }
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  double fmas = (double)sms * 4 * 256 * 8192 * 8;
  printf("FP64 FMA throughput: %.2f TFMA/s (%.1f TFLOP/s)\n", fmas / ms / 1e9, 2 * fmas / ms / 1e9);
  for (int nw : {1, 8}) {
    cluster_exchange<<<8, 32 * nw>>>(cyc, 2000);
    cudaError_t err = cudaDeviceSynchronize();
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("cluster(8) st.async all-to-all + mbarrier wait, %d warps/CTA: %lld cycles/round (%s)\n", nw, h,
           cudaGetErrorString(err));
  }
  return 0;
}
