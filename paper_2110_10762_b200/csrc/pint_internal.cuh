// Internal declarations shared by the CUDA translation units of libpint_b200.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/pint_abi.h"

struct pint_ctx {
  int device = 0;
  int num_sms = 0;
  std::string last_error;
  double last_value = 0.0;
  int32_t *scratch_flag = nullptr;  // device int scratch
  double *scratch_d = nullptr;      // device double scratch (reductions)
  size_t scratch_d_len = 0;
};

// Raised inside implementation helpers, converted to a status at the ABI edge.
struct PintError {
  int code;
  std::string msg;
  double value;
};

[[noreturn]] void pint_throw(int code, const std::string &msg, double value = 0.0);
void pint_check_cuda(cudaError_t e, const char *what);
#define PINT_CUDA(call) pint_check_cuda((call), #call)

// Run fn, converting a PintError / std::exception into a status code and the
// context's last-error message (the ABI edge of every entry point).
template <typename F>
inline int pint_guarded(pint_ctx *ctx, F &&fn) {
  try {
    fn();
    return PINT_OK;
  } catch (const PintError &e) {
    if (ctx) {
      ctx->last_error = e.msg;
      ctx->last_value = e.value;
    }
    return e.code;
  } catch (const std::exception &e) {
    if (ctx) ctx->last_error = e.what();
    return PINT_ECUDA;
  }
}

// ------------------------------------------------------------ 1-D tridiagonal

// Uniform (kernel-parameter) factors of one chunk class.
template <int CH>
struct ChunkFactors {
  double q[CH];   // 1/pivot
  double e[CH];   // -E/pivot  (forward multiplier and back-substitution factor)
  double h[CH];   // forward-eliminated left-coupling vector
  double w[CH];   // row 0 of the chunk inverse (y0 = w . d)        [trapezoidal]
  double ws[CH];  // w / q: y0 from the pivot-scaled state t = q x   [backward Euler]
};

// Constant-coefficient twisted chunk solve (backward-Euler fast path, see
// tri1d.cu): the CH-1 chunk points are eliminated from both ends toward the
// middle point k with the limit factors of the Toeplitz LU (one multiplier mu
// for every row), the state is kept scaled by rho_j = lambda^|j-k| so that
// both sweeps are single FMAs with position-independent coefficients, and the
// two corner defects of the constant factorisation are folded into the
// separator terms on the host.
template <int CH>
struct CcstFactors {
  double mu;    // lambda^2: elimination multiplier (scaled variables)
  double kap;   // 1/c: substitution multiplier
  double kapm;  // 1/(c (1 - mu)): middle pivot
  double al, be, ga;  // z_0 = al P + be Q + ga w, z_L = be P + al Q + ga w
  double sAB, sB, nlam;  // effective boundary value: sAB s_near + sB (s_far - s_near) + nlam z_near
  double CmAB;  // x_k = CmAB (s_left + s) + CmN (z_0 + z_L) + kapm w
  double CmN;
  double g[CH / 2];   // psi_j += g_j sigma' (j < k; mirrored for the lower half)
  double rs[CH / 2];  // 1 / rho_j
  double ro[CH / 2];  // rho_j
};
inline int ccst_nscalars(int CH) { return 11 + 3 * (CH / 2); }

// Per-thread reduced-system constants, laid out [field][T] in device memory.
enum Tri1DField {
  TF_MASK = 0,      // 1 if the thread's separator is a real unknown
  TF_PCR_A = 1,     // 5 fields: level-1 PCR multipliers toward lane - 2^r
  TF_PCR_G = 6,     // 5 fields: level-1 PCR multipliers toward lane + 2^r
  TF_PCR_INV = 11,  // 1/diag after PCR
  TF_W1 = 12,       // level-1 left spike (coefficient of S_{W-1})
  TF_V1 = 13,       // level-1 right spike (coefficient of S_W)
  TF_CP = 14,       // lane 31: coupling of S_W to lane 30
  TF_R2 = 15,       // 2*J fields: rows W-1 / W of R2^{-1}, columns lane + 32 j
  // then TF_HQ / TF_HZ: coefficients of this warp's lane-0 values (y1_0, y0_0)
  //      in the level-2 right-hand side of the previous warp
};
#define TF_HQ(J) (15 + 2 * (J))
#define TF_HZ(J) (16 + 2 * (J))
#define TRI1D_NF(J) (17 + 2 * (J))  // odd: the per-thread table rows are bank-conflict free
inline int tri1d_nfields(int J) { return TRI1D_NF(J); }

struct Tri1DPlan {
  int64_t N = 0;
  int CH = 32;
  int T = 32;   // threads per slice
  int nW = 1;   // warps per slice
  int J = 1;    // ceil(nW / 32)
  int tb = 0;   // number of regular threads
  double D = 1, E = 0;
  double hq = 0;  // regular separator coupling Ro (fast path's uniform TF_HQ)
  bool l2win = false;  // level 2 through a 32-column window of R2^{-1} (entries outside cannot change an fp64 result)
  double f_first = 0, f_last = 0;  // per-step rhs forcing at point 0 / N-1 (raw)
  double fq_first = 0, fq_last = 0;  // the same in the pivot-scaled state
  int t_last = 0, l_last = 0;      // thread / slot of point N-1
  bool cn = false;
  int64_t steps = 1;
  double min_pivot = 0;
  std::vector<double> fac_reg, fac_tail;  // 5*CH each (q,e,h,w,ws)
  bool ccst = false;                      // constant-coefficient twisted chunk solve usable
  std::vector<double> ccst_fac;           // CcstFactors<CH> as a flat array (ccst_nscalars)
  std::vector<double> table;              // [nfields][T]
};

Tri1DPlan tri1d_plan(int64_t N, int CH, double D, double E, double f_first,
                     double f_last, bool cn, int64_t steps);

struct pint_op {
  pint_ctx *ctx = nullptr;
  pint_op_desc desc{};
  int64_t dim = 0;
  double dt = 0;
  // 1-D
  Tri1DPlan plan;
  double *d_table = nullptr;
  int batch_cluster = 1;
  int sweep_cluster = 1;
  int batch_wave_slices = 0;  // slices of apply_batch resident at once (0 = unknown)
  int batch_minb = 2;  // CTAs per SM the fine kernel is register-budgeted for (1 or 2)
  bool fused_sweep = true;  // the fused coarse sweep's shared memory fits one CTA
  bool sweep_defer = false;  // fused sweep: separate result rows fit (stores drained inside the next step's exchange)
  bool tri_general = false;  // runs the exact-pivot (GENERAL) kernels: tail thread, forcing, or no fast path
  // n-D
  int64_t nx = 1, ny = 1, nz = 1;
  void *cg_work = nullptr;   // CG scratch
  size_t cg_work_bytes = 0;
  double *cg_partials = nullptr;
  int64_t cg_nblocks = 0;
  int64_t cg_last_iters = 0;
  void *spec_q = nullptr;      // direct solve: n x n sine transform (T)
  void *spec_tcq = nullptr;    // direct solve, fp32 tensor-core path: pre-split tf32 tiles of Q
  void *spec_ip = nullptr;     // direct solve: reciprocal pivots [J][mode] (T)
  int spec_J = 0;
};

// 1-D launchers (tri1d.cu)
void tri1d_setup(pint_op *op);
void tri1d_apply_batch(pint_op *op, const double *in, double *out, int64_t nbatch,
                       int64_t stride, cudaStream_t s);
void tri1d_coarse_init(pint_op *op, double *lam, int64_t p, double *gcache,
                       cudaStream_t s);
void tri1d_sweep(pint_op *op, const double *prev, double *next, const double *fv,
                 double *gcache, int64_t k, int64_t p, double *deltas,
                 int32_t *nonfinite, cudaStream_t s, int chain);
void tri1d_destroy(pint_op *op);

// n-D launchers (stencil.cu / cg.cu)
void stencil_setup(pint_op *op);
void stencil_apply_batch(pint_op *op, const void *in, void *out, int64_t nbatch,
                         int64_t stride, cudaStream_t s);
void cg_setup(pint_op *op);
void cg_apply_batch(pint_op *op, const void *in, void *out, int64_t nbatch,
                    int64_t stride, cudaStream_t s);
void nd_destroy(pint_op *op);
void spectral_setup(pint_op *op);
void spectral_apply_batch(pint_op *op, const void *in, void *out, int64_t nbatch,
                          int64_t stride, cudaStream_t s);
void spectral_destroy(pint_op *op);
// 2-D/3-D implicit coarse apply: direct (spectral) or CG per desc.nd_solver
void nd_implicit_apply_batch(pint_op *op, const void *in, void *out, int64_t nbatch,
                             int64_t stride, cudaStream_t s);

// elementwise (correct.cu)
void correct_launch(int dtype, int64_t dim, int64_t nbatch, const void *gnew,
                    const void *f, const void *gold, const void *prev, void *out,
                    const uint8_t *f_only, double *delta, int32_t *nonfinite,
                    cudaStream_t s);
void correct_chain_launch(int dtype, int64_t dim, const void *gnew, const void *f, void *gcache, const void *prev,
                          void *out, const uint8_t *f_only, const double *fonly_delta, double *delta,
                          int32_t *nonfinite, cudaStream_t s);
void max_reduce_launch(const double *d, int64_t lo, int64_t hi, double *out,
                       cudaStream_t s);
void equal_launch(int dtype, int64_t dim, const void *a, const void *b, uint8_t *eq, cudaStream_t s);
