// ======================================================= asynchronous runtime
//
// Asynchronous Parareal with real concurrency (reference semantics:
// async_parareal.py:24-84, Algorithm 2), single- or multi-GPU.
//
// The slices 1..P are split into W contiguous DOMAINS (one per GPU; W = 1 on a
// single GPU). A domain owns a workspace with its slices' version rings plus
// one GHOST row, the mailbox of its predecessor slice lo-1 (owned by the
// previous domain). Persistent thread-block clusters of the domain's launch
// repeatedly claim one of the domain's slices from an atomic ticket queue
// (round-robin order, per-slice try-lock) and run
//     F(remembered) -> read the freshest published predecessor -> G(fresh)
//     -> new = F-only ? F(rem) : (G(fresh) + F(rem)) - G(rem) -> publish
// and never wait on another cluster: predecessor states are read from a ring
// of R version-stamped buffers with a seqlock check (retry if the writer
// lapped the slot), so no co-residency is required and staleness is whatever
// the hardware schedule produces. G(rem) is the previous activation's
// G(fresh) (cached per slice).
//
// Crossing a GPU boundary: when the cluster that publishes the domain's LAST
// slice writes the new version into its own ring it also stores it, with
// plain P2P stores over NVLink, into the ghost ring of the next domain, and
// then release-stores the version counter there (system scope). The next
// domain reads its ghost exactly like a local predecessor — no message
// queue, no barrier, no NCCL on the data path.
//
// Termination. W = 1: the publishing cluster checks "every slice drained
// (consumed the newest predecessor version) and every last change < eps"
// (async_parareal.py:52-58), or exact quiescence with eps < 0. W > 1: each
// domain publishes a status word {done, ghost version seen, version of its
// last slice, publish count} into a board held by EVERY domain (system-scope
// release stores, serialised per domain by a lock, each written after the
// acquire of the ghost version it reports). A domain whose own word says
// done double-collects its local board; if both collects agree, every word
// says done and every ghost version equals the predecessor domain's last
// published version (no push in flight), it sets the stop flag of every
// domain. Causality of the release/acquire chain makes each collect a
// consistent cut, so the stop predicate held globally at one instant.
// NCCL is used afterwards only to reduce the run's outcome (distributed.py).
//
// On one GPU the W domains can be hosted by a single launch (the clusters are
// split among them and the "peer" pointers are local): the emulation of a
// multi-GPU run that the tests use, with the same kernel code path.
#include <algorithm>
#include <cmath>
#include <vector>

#include "tri1d_device.cuh"

constexpr int ASYNC_TRACE_FIELDS = 8;
constexpr int ASYNC_MAX_DOMAINS = 64;
constexpr int ASYNC_R = 3;
constexpr int ASYNC_INFO = 6;

// trace record: slice, fresh predecessor version read, remembered version,
// F-only flag, delta (bits), globaltimer at F start / at publish,
// cluster id (+ 65536 * domain). Stored at the GLOBAL event index.

// status word: done (bit 63) | ghost version (21 bits) | last-slice version (21) | publishes (21)
constexpr unsigned long long SW_M = (1ull << 21) - 1;
__host__ __device__ __forceinline__ unsigned long long sw_pack(bool done, long long ghost, long long vlast,
                                                               long long pubs) {
  return ((unsigned long long)(done ? 1 : 0) << 63) | (((unsigned long long)ghost & SW_M) << 42) |
         (((unsigned long long)vlast & SW_M) << 21) | ((unsigned long long)pubs & SW_M);
}

struct AsyncShared {
  int64_t P, N;
  double eps;          // < 0: exact quiescence
  int64_t max_events;
  double delay_frac;   // injected delay per activation: U(0, delay_frac) * t_F
  unsigned long long seed;
  int claim;           // 0: round-robin ticket; 1: lowest ready slice of the domain first
};

// One domain as seen by the kernel (device memory; peers may be IPC mappings).
struct AsyncDomain {
  // local rows r = 0..nloc  (row r = global slice lo - 1 + r; row 0 = ghost)
  double *ring;            // (nloc+1) x R x N published versions
  double *remb;            // (nloc+1) x N   remembered predecessor reading
  double *gremb;           // (nloc+1) x N   G(remembered)
  double *scratch;         // ncl x 2 x N    (F result, fresh reading)
  long long *ver;          // (nloc+1) newest published version per row (ver[0]: mailbox)
  long long *vrem;         // version of the remembered reading
  long long *consumed;     // predecessor version consumed at the last activation
  long long *counts;       // activations per row
  int *busy;               // try-lock per row
  int *stable;             // last activation was F-only
  double *last_delta;
  unsigned long long *board;  // W status words (written by every domain)
  unsigned long long *ticket;
  int *stop;               // 1 = converged, 2 = max_events reached
  int *nonfinite;
  int *lock;               // serialises status-word updates
  long long *events;       // local publishes
  long long *retries;
  long long *gevents;      // global event counter (domain 0's)
  double *next_ring;       // ghost row of the next domain's ring (null: last domain)
  long long *next_ver;     // its mailbox version
  unsigned long long *peer_board[ASYNC_MAX_DOMAINS];
  int *peer_stop[ASYNC_MAX_DOMAINS];
  long long *trace;        // indexed by global event, ASYNC_TRACE_FIELDS each
  long long trace_cap;
  long long lo, nloc;
  int d, W;
  int cl_first, cl_count;  // clusters of the launch that serve this domain
};

// ------------------------------------------------------------- memory model
__device__ __forceinline__ long long ld_acquire_sys(const long long *p) {
  long long v;
  asm volatile("ld.acquire.sys.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(long long *p, long long v) {
  asm volatile("st.release.sys.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_release_sys_u64(unsigned long long *p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// Stop predicate over the domain's own slices (async_parareal.py:52-58 /
// quiescence): every slice drained and every last change < eps (eps >= 0), or
// every slice stable (eps < 0). *ghost receives the ghost version it used.
__device__ bool domain_done(const AsyncDomain &D, double eps, long long *ghost) {
  for (long long r = 1; r <= D.nloc; ++r) {
    const long long vp = ld_acquire_sys(D.ver + r - 1);
    if (r == 1) *ghost = vp;
    if (*(volatile long long *)(D.consumed + r) != vp) return false;
    if (eps >= 0.0 ? !(*(volatile double *)(D.last_delta + r) < eps) : !*(volatile int *)(D.stable + r))
      return false;
  }
  return true;
}

__device__ void stop_all(const AsyncDomain &D, int code) {
  if (D.W == 1) {
    if (code == 1) atomicExch(D.stop, 1);
    else atomicCAS(D.stop, 0, code);
    return;
  }
  for (int x = 0; x < D.W; ++x) {
    if (code == 1) atomicExch_system(D.peer_stop[x], 1);
    else atomicCAS_system(D.peer_stop[x], 0, code);
  }
}

// Consistent-cut check on the local board (see the header comment); a =
// shared-memory scratch of W words.
__device__ bool board_all_done(const AsyncDomain &D, unsigned long long *a) {
  for (int x = 0; x < D.W; ++x) {
    a[x] = ld_acquire_sys_u64(D.board + x);
    if (!(a[x] >> 63)) return false;
    if (x > 0 && ((a[x] >> 42) & SW_M) != ((a[x - 1] >> 21) & SW_M)) return false;
  }
  for (int x = 0; x < D.W; ++x)
    if (ld_acquire_sys_u64(D.board + x) != a[x]) return false;
  return true;
}

// Called by a cluster's control thread after every state change of the
// domain (publish or zero-change activation): evaluates the domain's stop
// predicate and, for W > 1, publishes the status word and checks the board.
__device__ void status_update(const AsyncDomain &D, double eps, unsigned long long *scratch) {
  long long ghost = 0;
  if (D.W == 1) {
    if (domain_done(D, eps, &ghost)) stop_all(D, 1);
    return;
  }
  while (atomicCAS(D.lock, 0, 1) != 0) __nanosleep(64);
  __threadfence();
  const bool done = domain_done(D, eps, &ghost);
  if (!done) ghost = ld_acquire_sys(D.ver);
  const long long vlast = ld_acquire_sys(D.ver + D.nloc);
  const long long pubs = *(volatile long long *)D.events;
  const unsigned long long w = sw_pack(done, ghost, vlast, pubs);
  for (int x = 0; x < D.W; ++x) st_release_sys_u64(D.peer_board[x] + D.d, w);
  __threadfence_system();
  atomicExch(D.lock, 0);
  if (done && board_all_done(D, scratch)) stop_all(D, 1);
}

template <int CH>
__device__ __forceinline__ void load_chunk_cg(double (&x)[CH], const double *src, int64_t N, int t) {
  const int64_t base = (int64_t)t * CH;
#pragma unroll
  for (int j = 0; j < CH; ++j) x[j] = (base + j < N) ? __ldcg(src + base + j) : 0.0;
}

// broadcast a few int64 control words from rank 0 / thread 0 to every CTA
__device__ __forceinline__ void ctl_broadcast(long long *ctl, int CL, int n) {
  cg::cluster_group cluster = cg::this_cluster();
  for (int r = 0; r < CL; ++r) {
    long long *dst = cluster.map_shared_rank(ctl, r);
    for (int q = 0; q < n; ++q) dst[q] = ctl[q];
  }
}

template <int CH, int J, bool CNF, bool CNG, bool GENERAL>
__global__ void __launch_bounds__(256, 1)
tri1d_async_kernel(const __grid_constant__ Tri1DParams<CH> PF, const __grid_constant__ Tri1DParams<CH> PG,
                   const AsyncShared S, const AsyncDomain *__restrict__ doms, int ndom) {
  extern __shared__ double smem[];
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int TB = blockDim.x;
  const int NF = TRI1D_NF(J);
  const int nW = PF.nW;
  // layout: [tabF][tabG][gather 8(nW+1)][2 mbarriers][ctl 8 x int64][red 128 (delta reduction / board collect)]
  double *tabF = smem;
  double *tabG = smem + NF * TB;
  double *gbuf = tabG + NF * TB;
  uint64_t *bars = reinterpret_cast<uint64_t *>(gbuf + 8 * (nW + 1));
  long long *ctl = reinterpret_cast<long long *>(bars + 2);
  double *red = reinterpret_cast<double *>(ctl + 8);
  StepCtx cF, cG;
  cF.TB = cG.TB = TB;
  cF.CL = cG.CL = PF.T / TB;
  cF.nW = cG.nW = nW;
  cF.t = cG.t = rank * TB + threadIdx.x;
  cF.lane = cG.lane = threadIdx.x & 31;
  cF.Wg = cG.Wg = cF.t >> 5;
  for (int f = 0; f < NF; ++f) {
    tabF[threadIdx.x * NF + f] = PF.table[(size_t)f * PF.T + cF.t];
    tabG[threadIdx.x * NF + f] = PG.table[(size_t)f * PG.T + cF.t];
  }
  cF.tab = smem_u32(tabF + threadIdx.x * NF);
  cG.tab = smem_u32(tabG + threadIdx.x * NF);
  for (int i = threadIdx.x; i < 8 * (nW + 1); i += TB) gbuf[i] = 0.0;
  cF.gbuf = cG.gbuf = smem_u32(gbuf);
  cF.mbar = cG.mbar = smem_u32(bars);
  if (threadIdx.x == 0) {
    mbar_init(cF.mbar, 1);
    mbar_init(cF.mbar + 8, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  cluster.sync();

  const int64_t N = S.N;
  const int CL = cF.CL;
  const int cid = (int)(blockIdx.x / CL);
  int h = 0;
  while (h + 1 < ndom && cid >= doms[h + 1].cl_first) ++h;
  const AsyncDomain &D = doms[h];
  const int R = ASYNC_R;
  const long long nloc = D.nloc;
  double *sF = D.scratch + (size_t)(cid - D.cl_first) * 2 * N;
  double *sFresh = sF + N;
  const int64_t base = (int64_t)cF.t * CH;
  const bool multi = D.W > 1;
  uint32_t sc = 0;
  double x[CH];
  bool bad = false;
  for (;;) {
    // ---- claim an activation (rank 0, thread 0), broadcast to the cluster
    if (rank == 0 && threadIdx.x == 0) {
      long long slot = -1;
      unsigned backoff = 32;
      for (;;) {
        if (*(volatile int *)D.stop) break;
        const unsigned long long tk = atomicAdd(D.ticket, 1ull);
        if (tk >= (unsigned long long)S.max_events * 64ull) {  // livelock guard
          stop_all(D, 2);
          break;
        }
        long long r = 1 + (long long)(tk % (unsigned long long)nloc);
        if (S.claim == 1) {
          // lowest slice with something to do (not stable on its newest
          // predecessor) and not busy: the pipeline order of the sweeps, so
          // activations spend F on the freshest inputs first
          long long pick = -1;
          for (long long q = 1; q <= nloc; ++q) {
            if (*(volatile int *)(D.busy + q)) continue;
            if (*(volatile int *)(D.stable + q) &&
                *(volatile long long *)(D.consumed + q) == *(volatile long long *)(D.ver + q - 1))
              continue;
            pick = q;
            break;
          }
          if (pick > 0) r = pick;
        }
        if (atomicCAS(D.busy + r, 0, 1) != 0) continue;
        const long long vp = ld_acquire_sys(D.ver + r - 1);
        if (*(volatile int *)(D.stable + r) && *(volatile long long *)(D.consumed + r) == vp) {
          // nothing new to consume: an activation would reproduce the same
          // value, i.e. a zero change; record it as such without publishing
          *(volatile double *)(D.last_delta + r) = 0.0;
          __threadfence();
          atomicExch(D.busy + r, 0);
          status_update(D, S.eps, reinterpret_cast<unsigned long long *>(red));
          __nanosleep(backoff);
          backoff = min(backoff * 2, 4096u);
          continue;
        }
        slot = r;
        break;
      }
      ctl[0] = slot;
      if (slot >= 0) {
        // acquire the previous owner's release of this slice (its busy
        // unlock follows its publish), then read the slice's bookkeeping once
        // for the whole cluster
        __threadfence();
        ctl[3] = *(volatile long long *)(D.ver + slot);
        ctl[4] = *(volatile long long *)(D.vrem + slot);
        ctl[5] = *(volatile long long *)(D.counts + slot);
      }
      ctl_broadcast(ctl, CL, 6);
    }
    cluster.sync();
    const long long r = ctl[0];
    if (r < 0) break;
    const long long vi = ctl[3], vr = ctl[4], cnt = ctl[5];
    const long long gi = D.lo - 1 + r;  // global slice index

    // ---- F(remembered)
    const unsigned long long tf0 = globaltimer();
    load_chunk_cg<CH>(x, D.remb + r * N, N, cF.t);
    run_steps<CH, J, CNF, GENERAL>(x, PF, cF, sc, PF.steps, 0.0, nullptr);
    store_chunk<CH>(x, sF, N, cF.t);
    if (S.delay_frac > 0.0 && rank == 0 && threadIdx.x == 0) {
      const unsigned long long tF = globaltimer() - tf0;
      const unsigned long long hs = mix64(S.seed ^ ((unsigned long long)gi << 32) ^ (unsigned long long)cnt);
      const double u = (double)(hs >> 11) * (1.0 / 9007199254740992.0);
      const unsigned long long until = globaltimer() + (unsigned long long)(u * S.delay_frac * (double)tF);
      while (globaltimer() < until) __nanosleep(1000);
    }

    // ---- freshest predecessor (seqlock read of the ring / mailbox)
    long long v = 0;
    for (int attempt = 0;; ++attempt) {
      if (rank == 0 && threadIdx.x == 0) {
        ctl[1] = ld_acquire_sys(D.ver + r - 1);
        ctl_broadcast(ctl + 1, CL, 1);
      }
      cluster.sync();
      v = ctl[1];
      load_chunk_cg<CH>(x, D.ring + ((size_t)(r - 1) * R + (size_t)(v % R)) * N, N, cF.t);
      // every CTA's slot loads are ordered before the version re-read
      // (barrier.cluster arrive.release / wait.acquire, then a fence)
      cluster.sync();
      if (rank == 0 && threadIdx.x == 0) {
        asm volatile("fence.acq_rel.sys;" ::: "memory");
        const long long v2 = ld_acquire_sys(D.ver + r - 1);
        ctl[2] = (v2 <= v + R - 2) ? 1 : 0;
        if (!ctl[2]) atomicAdd((unsigned long long *)D.retries, 1ull);
        ctl_broadcast(ctl + 2, CL, 1);
      }
      cluster.sync();
      if (ctl[2]) break;
    }
    // bitwise comparison with the remembered reading (array_equal semantics)
    double mism = 0.0;
#pragma unroll
    for (int j = 0; j < CH; ++j)
      if (base + j < N && !(x[j] == __ldcg(D.remb + r * N + base + j))) mism = 1.0;
    mism = warp_max(mism);
    store_chunk<CH>(x, sFresh, N, cF.t);

    // ---- G(fresh), with the mismatch flag reduced over the slice on the way
    double anymism = 0.0;
    run_steps<CH, J, CNG, GENERAL>(x, PG, cG, sc, PG.steps, mism, &anymism);
    const bool fonly = (v == vr) || (anymism == 0.0);

    // ---- correction, delta, publish into the next ring slot (+ the next domain's mailbox)
    const double *cur = D.ring + ((size_t)r * R + (size_t)(vi % R)) * N + base;
    double *dst = D.ring + ((size_t)r * R + (size_t)((vi + 1) % R)) * N + base;
    double *peer = (r == nloc && D.next_ring) ? D.next_ring + (size_t)((vi + 1) % R) * N + base : nullptr;
    double *gw = D.gremb + r * N + base;
    double *rw = D.remb + r * N + base;
    double dm = 0.0;
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      if (base + j < N) {
        const double g = x[j];
        const double f = __ldcg(sF + base + j);
        const double nv = fonly ? f : (g + f) - __ldcg(gw + j);
        dm = fmax(dm, fabs(nv - __ldcg(cur + j)));
        bad |= !isfinite(nv);
        dst[j] = nv;
        if (peer) peer[j] = nv;
        gw[j] = g;
        rw[j] = __ldcg(sFresh + base + j);
      }
    }
    dm = warp_max(dm);
    if (multi) __threadfence_system();
    else __threadfence();
    if ((threadIdx.x & 31) == 0) cluster.map_shared_rank(red, 0)[cF.Wg] = dm;
    cluster.sync();
    if (rank == 0 && threadIdx.x == 0) {
      double dd = 0.0;
      for (int w = 0; w < nW; ++w) dd = fmax(dd, red[w]);
      D.last_delta[r] = dd;
      D.vrem[r] = v;
      D.consumed[r] = v;
      D.stable[r] = fonly ? 1 : 0;
      D.counts[r] += 1;
      atomicAdd((unsigned long long *)D.events, 1ull);
      const long long ev = (long long)(multi ? atomicAdd_system((unsigned long long *)D.gevents, 1ull)
                                             : atomicAdd((unsigned long long *)D.gevents, 1ull)) + 1;
      if (D.trace && ev - 1 < D.trace_cap) {
        long long *rec = D.trace + (ev - 1) * ASYNC_TRACE_FIELDS;
        rec[0] = gi;
        rec[1] = v;
        rec[2] = vr;
        rec[3] = fonly ? 1 : 0;
        rec[4] = __double_as_longlong(dd);
        rec[5] = (long long)tf0;
        rec[6] = (long long)globaltimer();
        rec[7] = cid + 65536ll * D.d;
      }
      __threadfence_system();
      st_release_sys(D.ver + r, vi + 1);
      if (peer) st_release_sys(D.next_ver, vi + 1);
      atomicExch(D.busy + r, 0);
      status_update(D, S.eps, reinterpret_cast<unsigned long long *>(red));
      if (ev >= S.max_events && !*(volatile int *)D.stop) stop_all(D, 2);
    }
  }
  if (bad) atomicExch(D.nonfinite, 1);
  cluster.sync();
}

// ================================================================ host side

// Workspace of one domain: the offsets depend only on (nloc, N, W, ncl,
// trace_cap), so every rank can address a peer's mailbox and board from the
// peer's base pointer.
struct DomainLayout {
  size_t board, flags, ver, vrem, consumed, counts, busy, stable, last_delta, ring, remb, gremb, scratch, trace,
      bytes;
};
// flags block (64 B): ticket u64 @0, stop i32 @8, nonfinite i32 @12, lock i32 @16,
// events i64 @24, retries i64 @32, gevents i64 @40
static DomainLayout domain_layout(int64_t nloc, int64_t N, int W, int64_t ncl, int64_t trace_cap) {
  DomainLayout L;
  size_t b = 0;
  auto take = [&](size_t n) { size_t o = b; b += (n + 255) / 256 * 256; return o; };
  const size_t rows = (size_t)nloc + 1;
  L.board = take(8 * (size_t)W);
  L.flags = take(64);
  L.ver = take(8 * rows);
  L.vrem = take(8 * rows);
  L.consumed = take(8 * rows);
  L.counts = take(8 * rows);
  L.busy = take(4 * rows);
  L.stable = take(4 * rows);
  L.last_delta = take(8 * rows);
  L.ring = take(sizeof(double) * rows * ASYNC_R * (size_t)N);
  L.remb = take(sizeof(double) * rows * (size_t)N);
  L.gremb = take(sizeof(double) * rows * (size_t)N);
  L.scratch = take(sizeof(double) * (size_t)ncl * 2 * (size_t)N);
  L.trace = take(sizeof(long long) * ASYNC_TRACE_FIELDS * (size_t)trace_cap);
  L.bytes = b;
  return L;
}

struct pint_async_domain {
  pint_op *fine = nullptr, *coarse = nullptr;
  int64_t p = 0, lo = 0, hi = 0, nloc = 0, N = 0, ncl = 0, trace_cap = 0;
  int W = 1, d = 0;
  char *base = nullptr;
  DomainLayout L{};
  std::vector<char *> peer_base;   // per domain (own entry = base)
  std::vector<int64_t> peer_nloc;
  std::vector<bool> ipc_opened;
  bool connected = false;
  AsyncDomain desc{};
};

static void fill_desc(pint_async_domain *dom) {
  AsyncDomain &A = dom->desc;
  const DomainLayout &L = dom->L;
  char *w = dom->base;
  memset(&A, 0, sizeof(A));
  A.ring = (double *)(w + L.ring);
  A.remb = (double *)(w + L.remb);
  A.gremb = (double *)(w + L.gremb);
  A.scratch = (double *)(w + L.scratch);
  A.ver = (long long *)(w + L.ver);
  A.vrem = (long long *)(w + L.vrem);
  A.consumed = (long long *)(w + L.consumed);
  A.counts = (long long *)(w + L.counts);
  A.busy = (int *)(w + L.busy);
  A.stable = (int *)(w + L.stable);
  A.last_delta = (double *)(w + L.last_delta);
  A.board = (unsigned long long *)(w + L.board);
  A.ticket = (unsigned long long *)(w + L.flags);
  A.stop = (int *)(w + L.flags + 8);
  A.nonfinite = (int *)(w + L.flags + 12);
  A.lock = (int *)(w + L.flags + 16);
  A.events = (long long *)(w + L.flags + 24);
  A.retries = (long long *)(w + L.flags + 32);
  A.trace = dom->trace_cap > 0 ? (long long *)(w + L.trace) : nullptr;
  A.trace_cap = dom->trace_cap;
  A.lo = dom->lo;
  A.nloc = dom->nloc;
  A.d = dom->d;
  A.W = dom->W;
  // peers
  for (int x = 0; x < dom->W; ++x) {
    char *pb = dom->peer_base[x];
    const DomainLayout PL = domain_layout(dom->peer_nloc[x], dom->N, dom->W, 0, 0);  // board/flags/ver/ring offsets
    A.peer_board[x] = (unsigned long long *)(pb + PL.board);
    A.peer_stop[x] = (int *)(pb + PL.flags + 8);
    if (x == 0) A.gevents = (long long *)(pb + PL.flags + 40);
    if (x == dom->d + 1) {
      A.next_ring = (double *)(pb + PL.ring);
      A.next_ver = (long long *)(pb + PL.ver);
    }
  }
}

static int async_fail(pint_ctx *ctx, const PintError &e) {
  ctx->last_error = e.msg;
  ctx->last_value = e.value;
  return e.code;
}

static void check_pair(const pint_op *fine, const pint_op *coarse) {
  if (fine->desc.ndim != 1 || coarse->desc.ndim != 1 || fine->desc.rule == PINT_RULE_FORWARD_EULER ||
      coarse->desc.rule == PINT_RULE_FORWARD_EULER)
    pint_throw(PINT_EUNSUPPORTED, "the device async runtime supports 1-D implicit fine and coarse operators");
  const Tri1DPlan &pf = fine->plan, &pg = coarse->plan;
  if (pf.N != pg.N || pf.CH != pg.CH || pf.T != pg.T)
    pint_throw(PINT_EUNSUPPORTED, "fine and coarse operators must share the register layout (same rule family)");
  if (pf.CH != 16 && (pf.cn || pg.cn))
    pint_throw(PINT_EUNSUPPORTED, "trapezoidal operators need the 16-point register layout");
  if (!pf.cn && pg.cn)
    pint_throw(PINT_EUNSUPPORTED, "backward-Euler fine with trapezoidal coarse is not fused in the device runtime");
}

extern "C" int pint_async_domain_create(pint_op *fine, pint_op *coarse, int64_t p, int64_t lo, int64_t hi,
                                        int world, int index, int64_t nclusters, int64_t trace_cap,
                                        pint_async_domain **out) {
  if (!fine || !coarse || !out) return PINT_EARG;
  pint_ctx *ctx = fine->ctx;
  try {
    check_pair(fine, coarse);
    if (world < 1 || world > ASYNC_MAX_DOMAINS || index < 0 || index >= world)
      pint_throw(PINT_EARG, "domain index / world size out of range (1..64 domains)");
    if (p < 1 || lo < 1 || hi < lo || hi > p) pint_throw(PINT_EARG, "domain slice range must satisfy 1 <= lo <= hi <= p");
    if (trace_cap < 0) pint_throw(PINT_EARG, "trace_cap must be >= 0");
    auto *dom = new pint_async_domain();
    dom->fine = fine;
    dom->coarse = coarse;
    dom->p = p;
    dom->lo = lo;
    dom->hi = hi;
    dom->nloc = hi - lo + 1;
    dom->N = fine->plan.N;
    dom->W = world;
    dom->d = index;
    const int CL = fine->batch_cluster;
    const int64_t maxcl = std::max<int64_t>(1, ctx->num_sms / CL);
    dom->ncl = nclusters > 0 ? std::min<int64_t>(nclusters, dom->nloc) : std::min<int64_t>(dom->nloc, maxcl);
    dom->trace_cap = trace_cap;
    dom->L = domain_layout(dom->nloc, dom->N, world, dom->ncl, trace_cap);
    cudaError_t e = cudaMalloc((void **)&dom->base, dom->L.bytes);  // plain cudaMalloc: IPC-exportable
    if (e != cudaSuccess) {
      delete dom;
      pint_check_cuda(e, "cudaMalloc(async domain)");
    }
    dom->peer_base.assign(world, nullptr);
    dom->peer_nloc.assign(world, 0);
    dom->ipc_opened.assign(world, false);
    dom->peer_base[index] = dom->base;
    dom->peer_nloc[index] = dom->nloc;
    *out = dom;
    return PINT_OK;
  } catch (const PintError &e) {
    return async_fail(ctx, e);
  }
}

extern "C" int pint_async_domain_ipc_handle(pint_async_domain *dom, void *handle_out) {
  if (!dom || !handle_out) return PINT_EARG;
  try {
    cudaIpcMemHandle_t h;
    PINT_CUDA(cudaIpcGetMemHandle(&h, dom->base));
    memcpy(handle_out, &h, sizeof(h));
    return PINT_OK;
  } catch (const PintError &e) {
    return async_fail(dom->fine->ctx, e);
  }
}

extern "C" int pint_async_domain_connect(pint_async_domain *dom, const void *handles, const int64_t *nloc_all) {
  if (!dom || !handles || !nloc_all) return PINT_EARG;
  try {
    for (int x = 0; x < dom->W; ++x) {
      dom->peer_nloc[x] = nloc_all[x];
      if (x == dom->d) {
        if (nloc_all[x] != dom->nloc) pint_throw(PINT_EARG, "nloc_all disagrees with this domain's slice range");
        continue;
      }
      if (dom->ipc_opened[x] || dom->peer_base[x]) continue;
      cudaIpcMemHandle_t h;
      memcpy(&h, (const char *)handles + (size_t)x * sizeof(h), sizeof(h));
      void *ptr = nullptr;
      PINT_CUDA(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
      dom->peer_base[x] = (char *)ptr;
      dom->ipc_opened[x] = true;
    }
    fill_desc(dom);
    dom->connected = true;
    return PINT_OK;
  } catch (const PintError &e) {
    return async_fail(dom->fine->ctx, e);
  }
}

// Wire domains hosted by one process on one device (direct pointers).
extern "C" int pint_async_domains_connect_local(int ndom, pint_async_domain **doms) {
  if (ndom < 1 || !doms) return PINT_EARG;
  const int W = doms[0]->W;
  if (ndom != W) return PINT_EARG;
  for (int x = 0; x < W; ++x) {
    if (!doms[x] || doms[x]->d != x || doms[x]->W != W) return PINT_EARG;
  }
  for (int x = 0; x < W; ++x) {
    for (int y = 0; y < W; ++y) {
      doms[x]->peer_base[y] = doms[y]->base;
      doms[x]->peer_nloc[y] = doms[y]->nloc;
    }
    fill_desc(doms[x]);
    doms[x]->connected = true;
  }
  return PINT_OK;
}

// rows: (nloc+1) x N device doubles = the coarse initial iterate lam0[lo-1 .. hi]
extern "C" int pint_async_domain_reset(pint_async_domain *dom, const void *rows, void *stream) {
  if (!dom || !rows) return PINT_EARG;
  try {
    if (!dom->connected) pint_throw(PINT_EARG, "connect the domain before reset");
    cudaStream_t s = (cudaStream_t)stream;
    const AsyncDomain &A = dom->desc;
    const int64_t N = dom->N, nl = dom->nloc;
    const DomainLayout &L = dom->L;
    PINT_CUDA(cudaMemsetAsync(dom->base, 0, L.ring, s));  // board, flags, per-row control
    const double *Lr = (const double *)rows;
    // initial versions: ring[r][0] = lam0[r]; remembered = lam0[r-1] (version 0);
    // G(remembered) = G(lam0[r-1]) = lam0[r] (coarse initial iterate)
    PINT_CUDA(cudaMemcpy2DAsync(A.ring, sizeof(double) * ASYNC_R * N, Lr, sizeof(double) * N, sizeof(double) * N,
                                nl + 1, cudaMemcpyDeviceToDevice, s));
    PINT_CUDA(cudaMemcpyAsync(A.remb + N, Lr, sizeof(double) * nl * N, cudaMemcpyDeviceToDevice, s));
    PINT_CUDA(cudaMemcpyAsync(A.gremb + N, Lr + N, sizeof(double) * nl * N, cudaMemcpyDeviceToDevice, s));
    std::vector<double> inf(nl + 1, INFINITY);
    inf[0] = 0.0;
    std::vector<long long> minus1(nl + 1, -1);
    PINT_CUDA(cudaMemcpyAsync(A.last_delta, inf.data(), 8 * (nl + 1), cudaMemcpyHostToDevice, s));
    PINT_CUDA(cudaMemcpyAsync(A.consumed, minus1.data(), 8 * (nl + 1), cudaMemcpyHostToDevice, s));
    PINT_CUDA(cudaStreamSynchronize(s));
    return PINT_OK;
  } catch (const PintError &e) {
    return async_fail(dom->fine->ctx, e);
  }
}

// One persistent launch hosting ndom domains of the calling device.
extern "C" int pint_async_domain_launch(int ndom, pint_async_domain **doms, double epsilon, int64_t max_events,
                                        double delay_frac, uint64_t seed, void *stream) {
  if (ndom < 1 || !doms || !doms[0]) return PINT_EARG;
  pint_op *fine = doms[0]->fine, *coarse = doms[0]->coarse;
  pint_ctx *ctx = fine->ctx;
  try {
    for (int x = 0; x < ndom; ++x) {
      if (!doms[x] || !doms[x]->connected) pint_throw(PINT_EARG, "domain not connected");
      if (doms[x]->fine != fine || doms[x]->coarse != coarse) pint_throw(PINT_EARG, "hosted domains must share operators");
    }
    const int64_t me = max_events > 0 ? max_events : 20000;
    const Tri1DPlan &pf = fine->plan, &pg = coarse->plan;
    if (me * (pf.steps + pg.steps) >= (int64_t)1 << 31)
      pint_throw(PINT_EARG, "max_events * (fine + coarse steps) must stay below 2^31");
    if (doms[0]->W > 1 && me >= (int64_t)SW_M)
      pint_throw(PINT_EARG, "multi-domain runs need max_events < 2^21");
    cudaStream_t s = (cudaStream_t)stream;
    const int CL = fine->batch_cluster;
    const int TB = pf.T / CL;
    std::vector<AsyncDomain> hd(ndom);
    int ncl = 0;
    for (int x = 0; x < ndom; ++x) {
      hd[x] = doms[x]->desc;
      hd[x].cl_first = ncl;
      hd[x].cl_count = (int)doms[x]->ncl;
      ncl += (int)doms[x]->ncl;
    }
    if (ndom > 1) {  // hosted together: one shared trace buffer (domain 0's)
      for (int x = 1; x < ndom; ++x) {
        hd[x].trace = hd[0].trace;
        hd[x].trace_cap = hd[0].trace_cap;
      }
    }
    AsyncDomain *dd = nullptr;
    PINT_CUDA(cudaMallocAsync((void **)&dd, sizeof(AsyncDomain) * ndom, s));
    PINT_CUDA(cudaMemcpyAsync(dd, hd.data(), sizeof(AsyncDomain) * ndom, cudaMemcpyHostToDevice, s));
    AsyncShared S;
    S.P = doms[0]->p;
    S.N = pf.N;
    S.eps = epsilon;
    S.max_events = me;
    S.delay_frac = delay_frac;
    S.seed = seed;
    // claim policy: any order is a valid asynchronous schedule (the reads and
    // the stop rule are unchanged). Default: the lowest slice with something
    // to do first — C2 to eps = 1e-10 in 0.23 s (kappa 18, 617 activations,
    // 8 domains) against 0.40 s (kappa 46, 1566) with the round-robin ticket
    // (profiles/r02_async_claim.jsonl); PINT_ASYNC_CLAIM=0 restores the ticket.
    S.claim = 1;
    if (const char *e = getenv("PINT_ASYNC_CLAIM")) S.claim = atoi(e);
    const size_t sm = sizeof(double) * (2 * (size_t)tri1d_nfields(pf.J) * TB + 8 * (size_t)(pf.nW + 1)) + 16 +
                      64 + 32 * 8 * 4;
    const bool general = fine->tri_general || coarse->tri_general;
#define PINT_ASYNC_LAUNCH(CHV, JV, CNF, CNG, GV)                                                          \
  launch_cluster(tri1d_async_kernel<CHV, JV, CNF, CNG, GV>, ncl * CL, TB, CL, sm, s, make_params<CHV>(fine), \
                 make_params<CHV>(coarse), S, (const AsyncDomain *)dd, ndom)
#define PINT_ASYNC_J(CHV, CNF, CNG, GV)                      \
  switch (pf.J) {                                            \
    case 1: PINT_ASYNC_LAUNCH(CHV, 1, CNF, CNG, GV); break;  \
    case 2: PINT_ASYNC_LAUNCH(CHV, 2, CNF, CNG, GV); break;  \
    default: PINT_ASYNC_LAUNCH(CHV, 4, CNF, CNG, GV); break; \
  }
    if (pf.CH == 16) {
      if (pf.cn && pg.cn) {
        if (general) { PINT_ASYNC_J(16, true, true, true) } else { PINT_ASYNC_J(16, true, true, false) }
      } else if (pf.cn) {
        if (general) { PINT_ASYNC_J(16, true, false, true) } else { PINT_ASYNC_J(16, true, false, false) }
      } else {
        if (general) { PINT_ASYNC_J(16, false, false, true) } else { PINT_ASYNC_J(16, false, false, false) }
      }
    } else {
      if (general) { PINT_ASYNC_J(32, false, false, true) } else { PINT_ASYNC_J(32, false, false, false) }
    }
#undef PINT_ASYNC_J
#undef PINT_ASYNC_LAUNCH
    PINT_CUDA(cudaFreeAsync(dd, s));
    return PINT_OK;
  } catch (const PintError &e) {
    return async_fail(ctx, e);
  }
}

// rows_out: (nloc+1) x N device doubles <- newest published version of rows
// 0..nloc (row 0 = the ghost, i.e. the predecessor's last pushed version);
// counts_out (host, nloc+1); info_out (host, 6) = {global activations, stop
// code, non-finite, seqlock retries, clusters, local activations}; trace_out
// (host) <- min(global activations, cap) records at global event positions
// (records of other domains' activations are zero unless hosted together).
extern "C" int pint_async_domain_collect(pint_async_domain *dom, void *rows_out, int64_t *counts_out,
                                         int64_t *info_out, int64_t *trace_out, int64_t trace_cap, void *stream) {
  if (!dom) return PINT_EARG;
  try {
    cudaStream_t s = (cudaStream_t)stream;
    const AsyncDomain &A = dom->desc;
    const int64_t N = dom->N, nl = dom->nloc;
    std::vector<long long> ver(nl + 1), cnt(nl + 1);
    long long fl[6];
    long long gev = 0;
    PINT_CUDA(cudaStreamSynchronize(s));
    PINT_CUDA(cudaMemcpy(ver.data(), A.ver, 8 * (nl + 1), cudaMemcpyDeviceToHost));
    PINT_CUDA(cudaMemcpy(cnt.data(), A.counts, 8 * (nl + 1), cudaMemcpyDeviceToHost));
    PINT_CUDA(cudaMemcpy(fl, A.ticket, 48, cudaMemcpyDeviceToHost));
    PINT_CUDA(cudaMemcpy(&gev, A.gevents, 8, cudaMemcpyDefault));
    const int *fi = (const int *)fl;  // stop @8, nonfinite @12
    if (rows_out)
      for (int64_t r = 0; r <= nl; ++r)
        PINT_CUDA(cudaMemcpyAsync((double *)rows_out + r * N, A.ring + ((size_t)r * ASYNC_R + (size_t)(ver[r] % ASYNC_R)) * N,
                                  sizeof(double) * N, cudaMemcpyDeviceToDevice, s));
    if (trace_out && trace_cap > 0 && A.trace) {
      const size_t nrec = (size_t)std::min<long long>(std::min<long long>(gev, trace_cap), dom->trace_cap);
      PINT_CUDA(cudaMemcpyAsync(trace_out, A.trace, sizeof(long long) * ASYNC_TRACE_FIELDS * nrec,
                                cudaMemcpyDeviceToHost, s));
    }
    PINT_CUDA(cudaStreamSynchronize(s));
    if (counts_out)
      for (int64_t r = 0; r <= nl; ++r) counts_out[r] = cnt[r];
    if (info_out) {
      info_out[0] = gev;
      info_out[1] = fi[2];
      info_out[2] = fi[3];
      info_out[3] = fl[4];
      info_out[4] = dom->ncl;
      info_out[5] = fl[3];
    }
    return PINT_OK;
  } catch (const PintError &e) {
    return async_fail(dom->fine->ctx, e);
  }
}

extern "C" int pint_async_domain_destroy(pint_async_domain *dom) {
  if (!dom) return PINT_OK;
  for (int x = 0; x < dom->W; ++x)
    if (dom->ipc_opened[x] && dom->peer_base[x]) cudaIpcCloseMemHandle(dom->peer_base[x]);
  if (dom->base) cudaFree(dom->base);
  delete dom;
  return PINT_OK;
}

// Single-process run over `ndom` domains hosted by one launch on the calling
// device (ndom = 1: the plain single-GPU runtime; ndom > 1: the emulation of a
// multi-GPU run, same kernel path). lam0 = coarse initial iterate ((p+1) x N
// device); final_out (device, (p+1) x N); counts_out (host, p+1); info_out
// (host, 5) = {activations, stop code, non-finite, retries, clusters}.
extern "C" int pint_async_run_domains(pint_op *fine, pint_op *coarse, const void *lam0, int64_t p, int ndom,
                                      double epsilon, int64_t max_events, double delay_frac, uint64_t seed,
                                      void *final_out, int64_t *counts_out, int64_t *info_out, int64_t *trace_out,
                                      int64_t trace_cap, void *stream) {
  if (!fine || !coarse) return PINT_EARG;
  pint_ctx *ctx = fine->ctx;
  std::vector<pint_async_domain *> doms;
  auto cleanup = [&]() {
    for (auto *d : doms) pint_async_domain_destroy(d);
  };
  try {
    if (p < 1 || !lam0 || !final_out) pint_throw(PINT_EARG, "bad arguments");
    if (ndom < 1 || ndom > p) pint_throw(PINT_EARG, "need 1 <= domains <= p");
    if (trace_cap < 0 || (trace_cap > 0 && !trace_out)) pint_throw(PINT_EARG, "trace buffer missing");
    check_pair(fine, coarse);
    const int64_t N = fine->plan.N;
    const int CL = fine->batch_cluster;
    const int64_t maxcl = std::max<int64_t>(ndom, std::min<int64_t>(p, ctx->num_sms / CL));
    for (int x = 0; x < ndom; ++x) {
      const int64_t lo = 1 + p * x / ndom, hi = p * (x + 1) / ndom;
      const int64_t ncl = std::max<int64_t>(1, maxcl * (hi - lo + 1) / p);
      pint_async_domain *d = nullptr;
      int rc = pint_async_domain_create(fine, coarse, p, lo, hi, ndom, x, ncl, x == 0 ? trace_cap : 0, &d);
      if (rc != PINT_OK) {
        cleanup();
        return rc;
      }
      doms.push_back(d);
    }
    int rc = pint_async_domains_connect_local(ndom, doms.data());
    if (rc != PINT_OK) pint_throw(rc, "connect failed");
    for (int x = 0; x < ndom; ++x) {
      rc = pint_async_domain_reset(doms[x], (const double *)lam0 + (doms[x]->lo - 1) * N, stream);
      if (rc != PINT_OK) {
        cleanup();
        return rc;
      }
    }
    rc = pint_async_domain_launch(ndom, doms.data(), epsilon, max_events, delay_frac, seed, stream);
    if (rc != PINT_OK) {
      cleanup();
      return rc;
    }
    int64_t info_all[ASYNC_INFO] = {0, 0, 0, 0, 0, 0};
    cudaStream_t s = (cudaStream_t)stream;
    for (int x = 0; x < ndom; ++x) {
      pint_async_domain *d = doms[x];
      std::vector<int64_t> cnt(d->nloc + 1);
      int64_t inf[ASYNC_INFO];
      // rows lo-1..hi land at final_out[lo-1..hi]; row lo-1 of domain x > 0 is
      // its ghost and is overwritten by the owner below (domains in order)
      rc = pint_async_domain_collect(d, (double *)final_out + (d->lo - 1) * N, cnt.data(), inf,
                                     x == 0 ? trace_out : nullptr, x == 0 ? trace_cap : 0, stream);
      if (rc != PINT_OK) {
        cleanup();
        return rc;
      }
      if (counts_out) {
        if (x == 0) counts_out[0] = cnt[0];
        for (int64_t r = 1; r <= d->nloc; ++r) counts_out[d->lo - 1 + r] = cnt[r];
      }
      info_all[0] = inf[0];
      info_all[1] = std::max(info_all[1], inf[1]);
      info_all[2] = std::max(info_all[2], inf[2]);
      info_all[3] += inf[3];
      info_all[4] += inf[4];
    }
    // the ghost rows were written before their owners' rows: rewrite owners' last rows
    for (int x = 0; x + 1 < ndom; ++x) {
      pint_async_domain *d = doms[x];
      std::vector<long long> vl(1);
      PINT_CUDA(cudaMemcpy(vl.data(), d->desc.ver + d->nloc, 8, cudaMemcpyDeviceToHost));
      PINT_CUDA(cudaMemcpyAsync((double *)final_out + d->hi * N,
                                d->desc.ring + ((size_t)d->nloc * ASYNC_R + (size_t)(vl[0] % ASYNC_R)) * N,
                                sizeof(double) * N, cudaMemcpyDeviceToDevice, s));
    }
    PINT_CUDA(cudaStreamSynchronize(s));
    if (info_out)
      for (int q = 0; q < 5; ++q) info_out[q] = info_all[q];
    cleanup();
    return PINT_OK;
  } catch (const PintError &e) {
    cleanup();
    return async_fail(ctx, e);
  }
}

extern "C" int pint_async_run_traced(pint_op *fine, pint_op *coarse, const void *lam0, int64_t p, double epsilon,
                                     int64_t max_events, double delay_frac, uint64_t seed, void *final_out,
                                     int64_t *counts_out, int64_t *info_out, int64_t *trace_out, int64_t trace_cap,
                                     void *stream) {
  return pint_async_run_domains(fine, coarse, lam0, p, 1, epsilon, max_events, delay_frac, seed, final_out,
                                counts_out, info_out, trace_out, trace_cap, stream);
}

extern "C" int pint_async_run(pint_op *fine, pint_op *coarse, const void *lam0, int64_t p, double epsilon,
                              int64_t max_events, double delay_frac, uint64_t seed, void *final_out,
                              int64_t *counts_out, int64_t *info_out, void *stream) {
  return pint_async_run_traced(fine, coarse, lam0, p, epsilon, max_events, delay_frac, seed, final_out, counts_out,
                               info_out, nullptr, 0, stream);
}
