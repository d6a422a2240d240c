/*
 * pint_abi.h — C ABI of the B200-native Parareal hot path.
 *
 * This is the drop-in boundary for the reference's propagator plugin layer
 * and its synchronous sweep. Every entry point is extern "C", takes plain
 * pointers and sizes, and never exposes torch or CUDA C++ types. The
 * reference is pure Python (pintlab); the Python-side binding that a
 * maintainer would add is the ctypes stub shown in INTEGRATION.md.
 *
 * Reference interfaces replaced (file:line under /root/reference/pkg/src/pintlab):
 *   pint_op_create          <- PROPAGATOR_RULES builders
 *                              backward_euler_propagator   model.py:172-184
 *                              trapezoidal_propagator      model.py:187-200
 *                              fine_from_onestep (explicit) model.py:147-154
 *                              _onestep + lu_solve          model.py:157-169, linalg.py:241-266
 *   pint_op_apply_batch     <- AffinePropagator.apply       model.py:123-129
 *                              (batched over independent time slices)
 *   pint_correct            <- parareal_update              parareal.py:25-36
 *                              + (new - prev).max_abs()     parareal.py:126, linalg.py:113-117
 *                              + finiteness check           linalg.py:74-75
 *   pint_coarse_init        <- coarse_init                  parareal.py:54-63
 *   pint_sync_sweep         <- one sweep of run_parareal    parareal.py:119-127
 *                              (frozen prefix, F-only branch, delta)
 *   pint_async_run          <- run_async_parareal           async_parareal.py:61-84
 *                              (real concurrency instead of the
 *                               simulate_async event loop, async_engine.py:238-365)
 *   pint_async_run_traced   <- + AsyncTrace / UpdateRecord  async_engine.py:122-190
 *                              (audited as validate_schedule, async_engine.py:402-459)
 *   pint_correct_chain      <- one step of the coarse chain of run_parareal
 *                              parareal.py:119-127 (F-only decided from the
 *                              predecessor's delta, G(old) cache refreshed)
 *   pint_shared_*, pint_ipc_*, pint_mailbox_*, pint_board_*
 *                           <- the predecessor reads of async_parareal.py:24-49
 *                              and the drained stop of async_engine.py:287-291
 *                              across processes/GPUs (async_mp.py)
 *   pint_async_domain_*     <- run_async_parareal across GPUs (one domain of
 *                              contiguous slices per GPU; the slice-boundary
 *                              state is pushed to the next GPU by P2P stores;
 *                              no reference counterpart: the reference is
 *                              single-process, async_engine.py:238-365)
 *
 * Error codes map onto the reference's exception taxonomy (errors.py):
 *   PINT_EDIM       -> DimensionError                errors.py:10-11
 *   PINT_EARG       -> ValueError
 *   PINT_ENONFINITE -> ValueError("... must be finite") linalg.py:74-75
 *   PINT_ENOCONV    -> ConvergenceFailure(estimate)  errors.py:18-26
 *   PINT_ESINGULAR  -> SingularSystemError(dt, pivot) errors.py:37-43
 *   PINT_ECUDA      -> RuntimeError(cuda error string)
 *   PINT_EUNSUPPORTED -> NotImplementedError
 * The message of the last error on a context is returned by pint_last_error.
 *
 * Threading: all compute calls are stream-ordered and asynchronous with
 * respect to the host unless stated. A context is bound to one device and is
 * not thread-safe. Operators are immutable after creation; all scratch is
 * allocated at creation (no allocation inside hot calls).
 */
#ifndef PINT_ABI_H
#define PINT_ABI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PINT_ABI_VERSION 1

enum pint_status {
  PINT_OK = 0,
  PINT_EDIM = 1,
  PINT_EARG = 2,
  PINT_ENONFINITE = 3,
  PINT_ENOCONV = 4,
  PINT_ESINGULAR = 5,
  PINT_ECUDA = 6,
  PINT_EUNSUPPORTED = 7
};

enum pint_dtype { PINT_F32 = 0, PINT_F64 = 1 };

/* Solver of the 2-D/3-D implicit (backward-Euler) step. */
enum pint_nd_solver {
  PINT_ND_DIRECT = 0, /* sine-transform diagonalisation + tridiagonal sweeps: exact to rounding */
  PINT_ND_CG = 1      /* conjugate gradients to ||r|| <= cg_rtol ||b||                        */
};

enum pint_rule {
  PINT_RULE_BACKWARD_EULER = 0, /* (I - dt A) u+ = u + dt c                */
  PINT_RULE_TRAPEZOIDAL = 1,    /* (I - dt/2 A) u+ = (I + dt/2 A) u + dt c */
  PINT_RULE_FORWARD_EULER = 2   /* u+ = (I + dt A) u + dt c               */
};

typedef struct pint_ctx pint_ctx;
typedef struct pint_op pint_op;
typedef struct pint_async_domain pint_async_domain;

/*
 * Operator description. The operator is u' = A u + c on a tensor grid of
 * ndim (1..3) axes, shape[d] interior points per axis.
 *   ndim == 1: A = a_diag * I + a_off * (S + S^T) (symmetric constant-coefficient
 *              tridiagonal; heat1d_system gives a_diag = -2/h^2, a_off = 1/h^2;
 *              scalar_decay_system gives n = 1, a_diag = -rate), and the
 *              forcing c is nonzero only at the end nodes: c[0] = c_first,
 *              c[n-1] = c_last (summed when n == 1).
 *   ndim >= 2: A = (1/h^2) * (zero-Dirichlet 5/7-point Laplacian), c = 0.
 * One propagator application advances `steps` steps of width dt = span/steps.
 * Implicit rules in 2-D/3-D are solved directly (nd_solver = PINT_ND_DIRECT,
 * the default: same system as the reference's dense LU solve, model.py:157-184)
 * or by conjugate gradients to ||r||_2 <= cg_rtol * ||b||_2 (at most cg_maxit
 * iterations; nd_solver = PINT_ND_CG).
 */
typedef struct pint_op_desc {
  int32_t ndim;
  int32_t rule;      /* enum pint_rule */
  int32_t dtype;     /* enum pint_dtype */
  int32_t nd_solver; /* enum pint_nd_solver (ndim >= 2 implicit) */
  int64_t shape[3];
  double h;          /* grid spacing (ndim >= 2) */
  double span;       /* time covered by one application */
  int64_t steps;     /* steps per application (>= 1) */
  double a_diag;     /* ndim == 1 */
  double a_off;      /* ndim == 1 */
  double c_first;    /* ndim == 1 */
  double c_last;     /* ndim == 1 */
  double cg_rtol;    /* ndim >= 2 implicit */
  int64_t cg_maxit;  /* ndim >= 2 implicit */
  int32_t layout_ch; /* 0 = auto; else points per thread (1-D: 16 or 32) */
  int32_t reserved1;
} pint_op_desc;

/* Static facts about a created operator (for cost models and benchmarks). */
typedef struct pint_op_info {
  int64_t dim;             /* points per state */
  int64_t steps;
  int32_t dtype;
  int32_t rule;
  int32_t threads_per_slice;   /* 1-D: T = 32 * warps */
  int32_t points_per_thread;   /* 1-D: CH */
  int32_t batch_cluster;       /* CTAs per slice in apply_batch */
  int32_t sweep_cluster;       /* CTAs in the fused coarse sweep */
  double dt;
  double diag;                 /* 1-D: D of the implicit step matrix */
  double offdiag;              /* 1-D: E of the implicit step matrix */
  double min_pivot;
  int32_t batch_wave_slices;   /* 1-D: slices apply_batch keeps resident at once (one wave); 0 = unknown */
  int32_t fused_sweep;         /* 1-D: 1 if pint_sync_sweep's fused kernel fits (shared memory), else 0 */
  int32_t general;             /* 1-D: 1 if the exact-pivot kernels run (tail thread, forcing, no fast path) */
  int32_t reserved0;
} pint_op_info;

int pint_abi_version(void);

int pint_ctx_create(int device, pint_ctx **out);
int pint_ctx_destroy(pint_ctx *ctx);
const char *pint_last_error(const pint_ctx *ctx);
/* Estimate payload of the last PINT_ENOCONV / pivot of the last PINT_ESINGULAR. */
double pint_last_error_value(const pint_ctx *ctx);

int pint_op_create(pint_ctx *ctx, const pint_op_desc *desc, pint_op **out);
int pint_op_destroy(pint_op *op);
int pint_op_get_info(const pint_op *op, pint_op_info *info);

/*
 * out[b] = P(in[b]) for b in [0, nbatch): in/out are device pointers to
 * nbatch states of `dim` elements, consecutive states `stride` elements
 * apart. in and out must not alias. Stream-ordered on `stream`
 * (a cudaStream_t, NULL = legacy default stream).
 */
int pint_op_apply_batch(pint_op *op, const void *in, void *out, int64_t nbatch,
                        int64_t stride, void *stream);

/*
 * Predictor-corrector update, elementwise over nbatch states of dim points:
 *   out = f_only[b] ? f : (gnew + f) - gold         (parareal.py:34-36)
 *   delta[b] = max |out - prev|                       (parareal.py:126)
 * f_only may be NULL (all zero). prev may be NULL (no delta). delta_dev is a
 * device array of nbatch doubles; *nonfinite_dev (device int32) is set to 1
 * when any output is NaN/Inf (never cleared by this call).
 */
int pint_correct(pint_ctx *ctx, int32_t dtype, int64_t dim, int64_t nbatch,
                 const void *gnew, const void *f, const void *gold,
                 const void *prev, void *out, const uint8_t *f_only,
                 double *delta_dev, int32_t *nonfinite_dev, void *stream);

/*
 * lam[i] = G(lam[i-1]) for i = 1..p, lam is (p+1) x dim contiguous with
 * lam[0] = u0 preset. If gcache != NULL it receives a copy of lam (G of the
 * coarse initial iterate, i.e. G(lam[i-1]) at row i) for the first sweep.
 */
int pint_coarse_init(pint_op *coarse, void *lam, int64_t p, void *gcache,
                     void *stream);

/*
 * One synchronous sweep k (1 <= k <= p) of run_parareal, given fv[i] =
 * F(prev[i-1]) for i in [k, p] (rows of a (p+1) x dim array):
 *   next[i] = prev[i]                       for i < k (caller-owned copy; the
 *                                           call writes next[k-1] itself)
 *   next[i] = F-only ? fv[i] : (G(next[i-1]) + fv[i]) - gcache[i]   for i >= k
 *   gcache[i] <- G(next[i-1])               for i >= k (the next sweep's G(old))
 *   deltas_dev[i] = max |next[i] - prev[i]| for i >= k, 0 for i = k-1
 * The F-only branch fires when deltas_dev[i-1] == 0 (bitwise-equal readings;
 * always at i == k). *nonfinite_dev is set to 1 on any non-finite output.
 * coarse must be the same operator that produced gcache.
 */
int pint_sync_sweep(pint_op *coarse, const void *prev, void *next,
                    const void *fv, void *gcache, int64_t k, int64_t p,
                    double *deltas_dev, int32_t *nonfinite_dev, void *stream);

/*
 * *equal_dev (device uint8) <- 1 if a[i] == b[i] for all i < dim (IEEE
 * equality: -0.0 == 0.0, NaN != NaN — numpy.array_equal semantics, the
 * F-only test of parareal.py:34), else 0.
 */
int pint_equal_flag(pint_ctx *ctx, int32_t dtype, int64_t dim, const void *a,
                    const void *b, uint8_t *equal_dev, void *stream);

/*
 * Chain-input variant for a time-slice shard (multi-GPU): next[k-1] and
 * deltas_dev[k-1] are INPUTS holding this sweep's new value of slice k-1 and
 * its delta (received from the GPU owning slice k-1); the F-only branch of
 * slice k fires when that delta is 0. Otherwise as pint_sync_sweep.
 */
int pint_sync_sweep_chain(pint_op *coarse, const void *prev, void *next,
                          const void *fv, void *gcache, int64_t k, int64_t p,
                          double *deltas_dev, int32_t *nonfinite_dev,
                          void *stream);

/*
 * One step of the serial coarse chain (generic sweep), slice i:
 *   f_only := (f_only && *f_only) || (fonly_delta_dev && *fonly_delta_dev == 0)
 *             (array_equal(fresh, old) <=> the predecessor's delta is 0)
 *   out     = f_only ? f : (gnew + f) - gcache          (parareal.py:34-36)
 *   gcache <- gnew                                      (next sweep's G(old))
 *   *delta_dev = max(*delta_dev, max |out - prev|)      (caller zeroes it per sweep)
 * out may alias prev or f (elementwise, read before write). One launch.
 */
int pint_correct_chain(pint_ctx *ctx, int32_t dtype, int64_t dim, const void *gnew,
                       const void *f, void *gcache, const void *prev, void *out,
                       const uint8_t *f_only, const double *fonly_delta_dev,
                       double *delta_dev, int32_t *nonfinite_dev, void *stream);

/*
 * Cross-process exchange for the multi-GPU asynchronous runtime (async_mp.py).
 * pint_shared_alloc: zeroed device memory that can be exported;
 * pint_ipc_export / pint_ipc_open / pint_ipc_close: 64-byte CUDA IPC handles.
 */
int pint_shared_alloc(pint_ctx *ctx, int64_t bytes, void **dev_ptr);
int pint_shared_free(pint_ctx *ctx, void *dev_ptr);
int pint_ipc_export(pint_ctx *ctx, void *dev_ptr, uint8_t *handle64);
int pint_ipc_open(pint_ctx *ctx, const uint8_t *handle64, void **dev_ptr);
int pint_ipc_close(pint_ctx *ctx, void *dev_ptr);

/*
 * Push `bytes` from src into dst (any device address, e.g. a peer's mailbox
 * slot opened through IPC) with SM stores, then publish: *ver = version with a
 * system-scope release once every CTA's stores are fenced. done_ctr: a zeroed
 * device uint32 owned by the calling stream. 16-byte aligned rows.
 */
int pint_mailbox_push(pint_ctx *ctx, void *dst, const void *src, int64_t bytes, int64_t *ver,
                      int64_t version, uint32_t *done_ctr, void *stream);

/*
 * Seqlock read of the freshest published version v of a ring of nslots
 * slots (slot_bytes apart) guarded by *ver: dst <- slot v % nslots,
 * *v_out = v, *torn = 1 if the producer may have started overwriting the
 * slot during the copy (version advanced by more than nslots - 2). vsel is a
 * device int64 scratch word of the stream.
 */
int pint_mailbox_read(pint_ctx *ctx, const void *ring, int64_t slot_bytes, int64_t nslots,
                      const int64_t *ver, void *dst, int64_t bytes, int64_t *vsel,
                      int64_t *v_out, int32_t *torn, void *stream);

/*
 * Stream-ordered wait until *ver >= value (a version another GPU publishes
 * with pint_mailbox_push): one thread polls with system-scope acquire loads;
 * after timeout_s it sets *timed_out = 1 and returns instead of hanging.
 */
int pint_mailbox_wait(pint_ctx *ctx, const int64_t *ver, int64_t value, double timeout_s,
                      int32_t *timed_out, void *stream);

/*
 * Status boards: slot = 8 int64 {seq, w0..w6}; post writes seq+1, the seven
 * words, seq+2 (system-scope release); read snapshots nslots slots with
 * acquire loads until both sequence reads agree (seq -1 if a slot never
 * settles) into out_dev (nslots x 8).
 */
int pint_board_post(pint_ctx *ctx, int64_t *slot, int64_t seq, const int64_t *words7, void *stream);
int pint_board_read(pint_ctx *ctx, const int64_t *board, int32_t nslots, int64_t *out_dev,
                    void *stream);

/*
 * Asynchronous Parareal with real concurrency on one GPU (persistent launch;
 * see tri1d.cu). lam0 = coarse initial iterate ((p+1) x dim, device). Stops
 * when every slice has consumed the newest predecessor version and every last
 * change is < epsilon; epsilon < 0 runs to exact quiescence. delay_frac > 0
 * injects a seeded per-activation delay U(0, delay_frac) * t_F. Writes the
 * newest published iterate to final_out (device), activations per slice to
 * counts_out (host, p+1), and info_out (host, 5) = {activations, stop code
 * (1 converged / 2 max_events), non-finite, seqlock retries, clusters}.
 * Synchronous with respect to the host.
 */
int pint_async_run(pint_op *fine, pint_op *coarse, const void *lam0, int64_t p,
                   double epsilon, int64_t max_events, double delay_frac,
                   uint64_t seed, void *final_out, int64_t *counts_out,
                   int64_t *info_out, void *stream);

/*
 * pint_async_run plus a per-activation trace (the device
 * analogue of the reference's UpdateRecord list, async_engine.py:122-131,
 * audited like validate_schedule, async_engine.py:402-459). trace_out (host)
 * receives min(activations, trace_cap) records of 8 int64 in publish order:
 * {slice i, fresh version of slice i-1 read, remembered version, F-only flag,
 *  delta (IEEE-754 bits), globaltimer ns at F start, globaltimer ns at
 *  publish, cluster id}. Versions count publishes per slice (0 = initial).
 */
int pint_async_run_traced(pint_op *fine, pint_op *coarse, const void *lam0,
                          int64_t p, double epsilon, int64_t max_events,
                          double delay_frac, uint64_t seed, void *final_out,
                          int64_t *counts_out, int64_t *info_out,
                          int64_t *trace_out, int64_t trace_cap, void *stream);

/*
 * Multi-GPU asynchronous runtime. One DOMAIN = the contiguous
 * slices lo..hi (1-based) owned by one GPU, plus a ghost row (mailbox) for
 * slice lo-1. The domain's workspace is one cudaMalloc block whose layout
 * depends only on (hi-lo+1, N, world, clusters, trace_cap), so peers address
 * each other's mailbox and status board from the exported base pointer.
 * Sequence per rank (distributed.py): create -> ipc_handle -> exchange
 * handles (host) -> connect -> reset -> host barrier -> launch -> stream
 * sync -> host barrier -> collect -> destroy. Domains hosted by one process
 * on one device are wired with pint_async_domains_connect_local and launched
 * together (the single-GPU emulation of a multi-GPU run).
 */
int pint_async_domain_create(pint_op *fine, pint_op *coarse, int64_t p,
                             int64_t lo, int64_t hi, int world, int index,
                             int64_t nclusters, int64_t trace_cap,
                             pint_async_domain **out);
/* handle_out: 64 bytes (cudaIpcMemHandle_t of the workspace). */
int pint_async_domain_ipc_handle(pint_async_domain *dom, void *handle_out);
/* handles: world x 64 bytes (own entry ignored); nloc_all: world slice counts. */
int pint_async_domain_connect(pint_async_domain *dom, const void *handles,
                              const int64_t *nloc_all);
/* doms[x] must have index x, x = 0..ndom-1 == world. */
int pint_async_domains_connect_local(int ndom, pint_async_domain **doms);
/* rows: device, (hi-lo+2) x N = coarse initial iterate lam0[lo-1 .. hi]. Synchronous. */
int pint_async_domain_reset(pint_async_domain *dom, const void *rows, void *stream);
/* One persistent launch hosting ndom connected domains of the calling device. */
int pint_async_domain_launch(int ndom, pint_async_domain **doms, double epsilon,
                             int64_t max_events, double delay_frac,
                             uint64_t seed, void *stream);
/*
 * After the launch completed: rows_out (device, (hi-lo+2) x N) <- newest
 * published rows lo-1..hi (row 0 = ghost); counts_out (host, hi-lo+2);
 * info_out (host, 6) = {global activations, stop code, non-finite, seqlock
 * retries, clusters, local activations}; trace_out (host) <- records at
 * global event positions (zeros where another GPU published).
 */
int pint_async_domain_collect(pint_async_domain *dom, void *rows_out,
                              int64_t *counts_out, int64_t *info_out,
                              int64_t *trace_out, int64_t trace_cap,
                              void *stream);
int pint_async_domain_destroy(pint_async_domain *dom);
/*
 * pint_async_run_traced over ndom domains hosted by ONE launch on the calling
 * device (ndom = 1 is pint_async_run_traced): the multi-GPU protocol
 * (mailbox push, status boards, distributed stop) emulated on one GPU.
 */
int pint_async_run_domains(pint_op *fine, pint_op *coarse, const void *lam0,
                           int64_t p, int ndom, double epsilon,
                           int64_t max_events, double delay_frac,
                           uint64_t seed, void *final_out, int64_t *counts_out,
                           int64_t *info_out, int64_t *trace_out,
                           int64_t trace_cap, void *stream);

/* max over deltas_dev[lo..hi) -> *out_dev (device double), deterministic. */
int pint_max_reduce(pint_ctx *ctx, const double *deltas_dev, int64_t lo,
                    int64_t hi, double *out_dev, void *stream);

/*
 * Host-only export of the exact 1-D solver plan a backward-Euler /
 * trapezoidal operator would use (no device needed): dims_out[0..5] =
 * {CH, T, nW, J, tb, NF}; fac_out = 10*CH doubles (regular then tail chunk:
 * q, e, h, w, ws); table_out = NF*T doubles ([field][thread]); scal_out =
 * {D, E, f_first, f_last, fq_first, fq_last, t_last, l_last}. Pass NULL
 * buffers to query dims only. Used by the CPU tests to emulate the kernel.
 */
int pint_tri1d_plan_host(const pint_op_desc *desc, int32_t *dims_out,
                         double *fac_out, double *table_out, double *scal_out);

/*
 * Host-only export of the backward-Euler fast path's chunk factors (the
 * constant-coefficient twisted chunk solve, csrc/tri1d.cu): *usable_out = 1
 * when the operator runs on it (every thread regular, no boundary forcing,
 * strictly diagonally dominant step matrix); fac_out = 11 + 3*(CH/2) doubles
 * {mu, kap, kapm, al, be, ga, sAB, sB, nlam, CmAB, CmN, g[CH/2],
 * 1/rho[CH/2], rho[CH/2]}. CH is desc->layout_ch (16) or 32. Used by the CPU tests to
 * emulate the kernel; replaces nothing in the reference (the reference's
 * step is a dense LU solve, linalg.py:241-266).
 */
int pint_tri1d_ccst_host(const pint_op_desc *desc, int32_t *usable_out,
                         double *fac_out);

#ifdef __cplusplus
}
#endif

#endif /* PINT_ABI_H */
