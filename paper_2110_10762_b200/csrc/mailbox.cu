// Cross-process slice mailboxes and status boards for the multi-GPU
// asynchronous runtime of whole-GPU activations (2-D/3-D F and G; host side
// in async_mp.py). Reference semantics: async_parareal.py:24-84 (two-slot
// reads of the predecessor), async_engine.py:238-365 (versions, drained stop).
//
// * A shared workspace is plain cudaMalloc memory exported with a CUDA IPC
//   handle; the peer opens it (peer access enabled lazily) and addresses it
//   with ordinary device pointers over NVLink.
// * mailbox_push: the producer GPU's SMs store a slice state straight into
//   the consumer's ring slot (P2P stores), every CTA fences at system scope
//   and counts itself done; the last CTA release-stores the version word
//   (st.release.sys). No copy engine, no host round trip, no barrier.
// * mailbox_read: the consumer reads the freshest published version under a
//   seqlock — acquire the version, copy slot v % R, re-acquire; the copy is
//   valid iff the producer has not started overwriting that slot, i.e. the
//   version advanced by at most R - 2 (the producer writes slot (v+R) % R only
//   after publishing v + R - 1). Three stream-ordered launches: a one-thread
//   version pick, the grid copy, a one-thread validation writing v and a torn
//   flag the host checks.
// * boards: one 8-word slot per writer rank in every rank's board, written
//   with a seqlock (seq odd, fields, seq even; system-scope release) and read
//   slot by slot with acquire loads until the two sequence reads agree.
#include <cuda_runtime.h>

#include "pint_internal.cuh"

namespace {

__device__ __forceinline__ long long ld_acq_sys(const long long *p) {
  long long v;
  asm volatile("ld.acquire.sys.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel_sys(long long *p, long long v) {
  asm volatile("st.release.sys.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys(long long *p, long long v) {
  asm volatile("st.relaxed.sys.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ long long ld_relaxed_sys(const long long *p) {
  long long v;
  asm volatile("ld.relaxed.sys.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// 16-byte granules (every state row is 256-byte aligned in the workspaces and
// torch allocations; a ragged tail is copied by bytes)
__global__ void __launch_bounds__(256) push_kernel(uint4 *__restrict__ dst, const uint4 *__restrict__ src,
                                                   int64_t n16, unsigned char *dtail, const unsigned char *stail,
                                                   int tail, long long *ver, long long version,
                                                   unsigned int *done_ctr) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = __ldcg(src + i);
  if (blockIdx.x == 0 && threadIdx.x < tail) dtail[threadIdx.x] = stail[threadIdx.x];
  __threadfence_system();  // this thread's peer stores are performed at system scope
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int prev = atomicAdd(done_ctr, 1u);
    if (prev == gridDim.x - 1) {
      // every CTA's stores are fenced: publish the version to the consumer
      asm volatile("fence.acq_rel.sys;" ::: "memory");
      st_rel_sys(ver, version);
      *done_ctr = 0u;  // re-armed for the next push on this stream
    }
  }
}

__global__ void pick_kernel(const long long *ver, long long *vsel) { *vsel = ld_acq_sys(ver); }

// Stream-ordered wait for a version published by another GPU (the chain edge
// of the synchronous multi-GPU sweep): one thread polls with acquire loads;
// gives up after timeout_ns (globaltimer) and flags it instead of hanging.
__global__ void wait_kernel(const long long *ver, long long value, unsigned long long timeout_ns, int32_t *timed_out) {
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  unsigned ns = 32;
  while (ld_acq_sys(ver) < value) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > timeout_ns) {
      *timed_out = 1;
      return;
    }
    __nanosleep(ns);
    ns = ns < 1024 ? 2 * ns : ns;
  }
}

__global__ void __launch_bounds__(256) read_kernel(uint4 *__restrict__ dst, const unsigned char *ring,
                                                   int64_t slot_bytes, int64_t nslots, const long long *vsel,
                                                   int64_t n16, unsigned char *dtail, int tail) {
  const long long v = *vsel;
  const unsigned char *slot = ring + (size_t)(v % nslots) * (size_t)slot_bytes;
  const uint4 *src = reinterpret_cast<const uint4 *>(slot);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = __ldcv(src + i);  // volatile: never a stale cached line of a peer-written slot
  if (blockIdx.x == 0 && threadIdx.x < tail) dtail[threadIdx.x] = slot[n16 * 16 + threadIdx.x];
}

__global__ void validate_kernel(const long long *ver, const long long *vsel, int64_t nslots, long long *v_out,
                                int32_t *torn) {
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  const long long v = *vsel;
  const long long v2 = ld_acq_sys(ver);
  *v_out = v;
  if (v2 > v + nslots - 2) *torn = 1;
}

__global__ void board_post_kernel(long long *slot, long long seq, long long w0, long long w1, long long w2,
                                  long long w3, long long w4, long long w5, long long w6) {
  st_relaxed_sys(slot, seq + 1);  // odd: write in progress
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  const long long w[7] = {w0, w1, w2, w3, w4, w5, w6};
  for (int q = 0; q < 7; ++q) st_relaxed_sys(slot + 1 + q, w[q]);
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  st_rel_sys(slot, seq + 2);
}

__global__ void board_read_kernel(const long long *board, int nslots, long long *out) {
  const int s = threadIdx.x;
  if (s >= nslots) return;
  const long long *slot = board + 8 * s;
  for (int spin = 0; spin < (1 << 20); ++spin) {
    const long long a = ld_acq_sys(slot);
    long long w[7];
    for (int q = 0; q < 7; ++q) w[q] = ld_relaxed_sys(slot + 1 + q);
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    const long long b = ld_relaxed_sys(slot);
    if (a == b && (a & 1) == 0) {
      out[8 * s] = a;
      for (int q = 0; q < 7; ++q) out[8 * s + 1 + q] = w[q];
      return;
    }
    __nanosleep(64);
  }
  out[8 * s] = -1;  // a writer died mid-post: reported, never silently accepted
}

unsigned grid_for(int64_t n16) {
  const int64_t per = (n16 + 255) / 256;
  return (unsigned)(per < 148 * 4 ? (per > 0 ? per : 1) : 148 * 4);
}

}  // namespace

// ----------------------------------------------------------------- C ABI

extern "C" {

int pint_shared_alloc(pint_ctx *ctx, int64_t bytes, void **dev_ptr) {
  if (!ctx || !dev_ptr || bytes <= 0) return PINT_EARG;
  return pint_guarded(ctx, [&] {
    void *p = nullptr;
    PINT_CUDA(cudaMalloc(&p, (size_t)bytes));
    PINT_CUDA(cudaMemset(p, 0, (size_t)bytes));
    PINT_CUDA(cudaDeviceSynchronize());
    *dev_ptr = p;
  });
}

int pint_shared_free(pint_ctx *ctx, void *dev_ptr) {
  if (!ctx) return PINT_EARG;
  return pint_guarded(ctx, [&] {
    if (dev_ptr) PINT_CUDA(cudaFree(dev_ptr));
  });
}

int pint_ipc_export(pint_ctx *ctx, void *dev_ptr, uint8_t *handle64) {
  if (!ctx || !dev_ptr || !handle64) return PINT_EARG;
  return pint_guarded(ctx, [&] {
    cudaIpcMemHandle_t h;
    PINT_CUDA(cudaIpcGetMemHandle(&h, dev_ptr));
    static_assert(sizeof(h) == 64, "CUDA IPC handles are 64 bytes");
    memcpy(handle64, &h, 64);
  });
}

int pint_ipc_open(pint_ctx *ctx, const uint8_t *handle64, void **dev_ptr) {
  if (!ctx || !handle64 || !dev_ptr) return PINT_EARG;
  return pint_guarded(ctx, [&] {
    cudaIpcMemHandle_t h;
    memcpy(&h, handle64, 64);
    void *p = nullptr;
    PINT_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    *dev_ptr = p;
  });
}

int pint_ipc_close(pint_ctx *ctx, void *dev_ptr) {
  if (!ctx) return PINT_EARG;
  return pint_guarded(ctx, [&] {
    if (dev_ptr) PINT_CUDA(cudaIpcCloseMemHandle(dev_ptr));
  });
}

int pint_mailbox_push(pint_ctx *ctx, void *dst, const void *src, int64_t bytes, int64_t *ver, int64_t version,
                      uint32_t *done_ctr, void *stream) {
  if (!ctx || !dst || !src || !ver || !done_ctr || bytes < 0) return PINT_EARG;
  return pint_guarded(ctx, [&] {
    if (((uintptr_t)dst | (uintptr_t)src) & 15u) pint_throw(PINT_EARG, "mailbox rows must be 16-byte aligned");
    const int64_t n16 = bytes / 16;
    const int tail = (int)(bytes - n16 * 16);
    push_kernel<<<grid_for(n16), 256, 0, (cudaStream_t)stream>>>(
        (uint4 *)dst, (const uint4 *)src, n16, (unsigned char *)dst + n16 * 16,
        (const unsigned char *)src + n16 * 16, tail, (long long *)ver, (long long)version, done_ctr);
    PINT_CUDA(cudaGetLastError());
  });
}

int pint_mailbox_read(pint_ctx *ctx, const void *ring, int64_t slot_bytes, int64_t nslots, const int64_t *ver,
                      void *dst, int64_t bytes, int64_t *vsel, int64_t *v_out, int32_t *torn, void *stream) {
  if (!ctx || !ring || !ver || !dst || !vsel || !v_out || !torn || nslots < 2 || bytes > slot_bytes) return PINT_EARG;
  return pint_guarded(ctx, [&] {
    if (((uintptr_t)dst | (uintptr_t)ring | (uintptr_t)slot_bytes) & 15u)
      pint_throw(PINT_EARG, "mailbox rows must be 16-byte aligned");
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t n16 = bytes / 16;
    const int tail = (int)(bytes - n16 * 16);
    pick_kernel<<<1, 1, 0, s>>>((const long long *)ver, (long long *)vsel);
    read_kernel<<<grid_for(n16), 256, 0, s>>>((uint4 *)dst, (const unsigned char *)ring, slot_bytes, nslots,
                                              (const long long *)vsel, n16, (unsigned char *)dst + n16 * 16, tail);
    validate_kernel<<<1, 1, 0, s>>>((const long long *)ver, (const long long *)vsel, nslots, (long long *)v_out,
                                    torn);
    PINT_CUDA(cudaGetLastError());
  });
}

int pint_mailbox_wait(pint_ctx *ctx, const int64_t *ver, int64_t value, double timeout_s, int32_t *timed_out,
                      void *stream) {
  if (!ctx || !ver || !timed_out || !(timeout_s > 0.0)) return PINT_EARG;
  return pint_guarded(ctx, [&] {
    wait_kernel<<<1, 1, 0, (cudaStream_t)stream>>>((const long long *)ver, (long long)value,
                                                   (unsigned long long)(timeout_s * 1e9), timed_out);
    PINT_CUDA(cudaGetLastError());
  });
}

int pint_board_post(pint_ctx *ctx, int64_t *slot, int64_t seq, const int64_t *words7, void *stream) {
  if (!ctx || !slot || !words7) return PINT_EARG;
  return pint_guarded(ctx, [&] {
    board_post_kernel<<<1, 1, 0, (cudaStream_t)stream>>>((long long *)slot, (long long)seq, words7[0], words7[1],
                                                         words7[2], words7[3], words7[4], words7[5], words7[6]);
    PINT_CUDA(cudaGetLastError());
  });
}

int pint_board_read(pint_ctx *ctx, const int64_t *board, int32_t nslots, int64_t *out_dev, void *stream) {
  if (!ctx || !board || !out_dev || nslots < 1 || nslots > 1024) return PINT_EARG;
  return pint_guarded(ctx, [&] {
    board_read_kernel<<<1, ((nslots + 31) / 32) * 32, 0, (cudaStream_t)stream>>>((const long long *)board, nslots,
                                                                                  (long long *)out_dev);
    PINT_CUDA(cudaGetLastError());
  });
}

}  // extern "C"
