// Standalone probe of the TMA plane load used by fe3d_tile (variants 12-14):
// loads tiles of a 4-D fp32 tensor (incl. out-of-bounds halo) through
// cp.async.bulk.tensor and compares them with the expected zero-filled box.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstring>
#include <vector>

constexpr int W = 64, H = 48;

__global__ void probe(const __grid_constant__ CUtensorMap tmap, float *out, int x0, int y0, int z, int b, int mode) {
  extern __shared__ __align__(128) unsigned char sm[];
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm);
  const uint32_t dst = base, bar = base + W * H * 4;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"((uint32_t)(W * H * 4))
                 : "memory");
    if (mode == 0)
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
          "[%6];" ::"r"(dst),
          "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(x0), "r"(y0), "r"(z), "r"(b), "r"(bar)
          : "memory");
    else
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
          "[%6];" ::"r"(dst),
          "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(x0), "r"(y0), "r"(z), "r"(b), "r"(bar)
          : "memory");
  }
  asm volatile(
      "{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W_%=;\n}" ::"r"(bar)
      : "memory");
  for (int i = threadIdx.x; i < W * H; i += blockDim.x) out[i] = reinterpret_cast<float *>(sm)[i];
}

int main(int argc, char **argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 0;
  const int nx = 64, ny = 64, nz = 64, nb = 2;
  const size_t n = (size_t)nx * ny * nz * nb;
  std::vector<float> h(n);
  for (size_t i = 0; i < n; ++i) h[i] = (float)(i % 1000003) + 1.0f;
  float *d, *o;
  cudaMalloc(&d, n * 4);
  cudaMalloc(&o, W * H * 4);
  cudaMemcpy(d, h.data(), n * 4, cudaMemcpyHostToDevice);
  void *fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp);
  CUtensorMap map;
  memset(&map, 0, sizeof(map));
  cuuint64_t dims[4] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)nz, (cuuint64_t)nb};
  cuuint64_t strides[3] = {(cuuint64_t)nx * 4, (cuuint64_t)nx * ny * 4, (cuuint64_t)nx * ny * nz * 4};
  cuuint32_t box[4] = {W, H, 1, 1}, es[4] = {1, 1, 1, 1};
  CUresult rc = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("entry point q=%d encode rc=%d\n", (int)q, (int)rc);
  int bad = 0;
  int cases[1][4] = {{0, 0, 0, 0}};
  if (argc > 5)
    for (int k = 0; k < 4; ++k) cases[0][k] = atoi(argv[2 + k]);
  for (auto &c : cases) {
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, W * H * 4 + 64);
    probe<<<1, 256, W * H * 4 + 64>>>(map, o, c[0], c[1], c[2], c[3], mode);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("case (%d,%d,%d,%d): %s\n", c[0], c[1], c[2], c[3], cudaGetErrorString(e));
      return 1;
    }
    std::vector<float> g(W * H);
    cudaMemcpy(g.data(), o, W * H * 4, cudaMemcpyDeviceToHost);
    for (int y = 0; y < H; ++y)
      for (int x = 0; x < W; ++x) {
        const int gx = c[0] + x, gy = c[1] + y, gz = c[2];
        float want = 0.0f;
        if (gx >= 0 && gx < nx && gy >= 0 && gy < ny && gz >= 0 && gz < nz)
          want = h[(((size_t)c[3] * nz + gz) * ny + gy) * nx + gx];
        if (g[y * W + x] != want) ++bad;
      }
  }
  printf("mismatches %d\n", bad);
  return bad != 0;
}
