// C ABI surface (include/pint_abi.h): contexts, operators, dispatch and the
// exception-to-status mapping of the reference's error taxonomy (errors.py).
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <string>

#include "pint_internal.cuh"

void pint_throw(int code, const std::string &msg, double value) { throw PintError{code, msg, value}; }

void pint_check_cuda(cudaError_t e, const char *what) {
  if (e != cudaSuccess) throw PintError{PINT_ECUDA, std::string(cudaGetErrorString(e)) + " in " + what, 0.0};
}

template <typename F>
static int guarded(pint_ctx *ctx, F &&fn) {
  return pint_guarded(ctx, static_cast<F &&>(fn));
}

static thread_local std::string g_orphan_error;

extern "C" {

int pint_abi_version(void) { return PINT_ABI_VERSION; }

int pint_ctx_create(int device, pint_ctx **out) {
  if (!out) return PINT_EARG;
  *out = nullptr;
  pint_ctx *ctx = new pint_ctx();
  int rc = guarded(ctx, [&] {
    int n = 0;
    PINT_CUDA(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n) pint_throw(PINT_EARG, "invalid CUDA device ordinal");
    PINT_CUDA(cudaSetDevice(device));
    ctx->device = device;
    PINT_CUDA(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device));
    int major = 0, minor = 0;
    PINT_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
    PINT_CUDA(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device));
    if (major != 10 || minor != 0)
      pint_throw(PINT_EUNSUPPORTED, "libpint_b200 is built for sm_100a (B200); device is sm_" +
                                        std::to_string(major) + std::to_string(minor));
    PINT_CUDA(cudaMalloc(&ctx->scratch_flag, sizeof(int32_t) * 4));
  });
  if (rc != PINT_OK) {
    g_orphan_error = ctx->last_error;
    delete ctx;
    return rc;
  }
  *out = ctx;
  return PINT_OK;
}

int pint_ctx_destroy(pint_ctx *ctx) {
  if (!ctx) return PINT_OK;
  if (ctx->scratch_flag) cudaFree(ctx->scratch_flag);
  if (ctx->scratch_d) cudaFree(ctx->scratch_d);
  delete ctx;
  return PINT_OK;
}

const char *pint_last_error(const pint_ctx *ctx) {
  if (!ctx) return g_orphan_error.c_str();
  return ctx->last_error.c_str();
}

double pint_last_error_value(const pint_ctx *ctx) { return ctx ? ctx->last_value : 0.0; }

int pint_op_create(pint_ctx *ctx, const pint_op_desc *desc, pint_op **out) {
  if (!ctx || !desc || !out) return PINT_EARG;
  *out = nullptr;
  pint_op *op = new pint_op();
  op->ctx = ctx;
  op->desc = *desc;
  int rc = guarded(ctx, [&] {
    const pint_op_desc &d = *desc;
    if (d.ndim < 1 || d.ndim > 3) pint_throw(PINT_EDIM, "ndim must be 1, 2 or 3");
    int64_t dim = 1;
    for (int a = 0; a < d.ndim; ++a) {
      if (d.shape[a] < 1) pint_throw(PINT_EDIM, "every axis needs at least one interior point");
      dim *= d.shape[a];
    }
    if (d.steps < 1) pint_throw(PINT_EARG, "step count must be >= 1");
    if (!(d.span > 0.0) || !std::isfinite(d.span)) pint_throw(PINT_EARG, "span must be positive");
    if (d.dtype != PINT_F32 && d.dtype != PINT_F64) pint_throw(PINT_EARG, "dtype must be PINT_F32 or PINT_F64");
    if (d.rule < 0 || d.rule > 2) pint_throw(PINT_EARG, "unknown propagator rule");
    op->dim = dim;
    PINT_CUDA(cudaSetDevice(ctx->device));
    if (d.ndim == 1) {
      if (d.rule == PINT_RULE_FORWARD_EULER) {
        stencil_setup(op);
      } else {
        if (!std::isfinite(d.a_diag) || !std::isfinite(d.a_off) || !std::isfinite(d.c_first) ||
            !std::isfinite(d.c_last))
          pint_throw(PINT_ENONFINITE, "operator coefficients must be finite");
        tri1d_setup(op);
      }
    } else {
      if (!(d.h > 0.0)) pint_throw(PINT_EARG, "grid spacing must be positive");
      op->nx = d.shape[d.ndim - 1];
      op->ny = d.ndim >= 2 ? d.shape[d.ndim - 2] : 1;
      op->nz = d.ndim >= 3 ? d.shape[0] : 1;
      if (d.rule == PINT_RULE_FORWARD_EULER) stencil_setup(op);
      else if (d.rule == PINT_RULE_BACKWARD_EULER) {
        if (d.nd_solver == PINT_ND_CG) cg_setup(op);
        else if (d.nd_solver == PINT_ND_DIRECT) spectral_setup(op);
        else pint_throw(PINT_EARG, "nd_solver must be PINT_ND_DIRECT or PINT_ND_CG");
      }
      else pint_throw(PINT_EUNSUPPORTED, "trapezoidal rule is implemented for 1-D operators only");
    }
  });
  if (rc != PINT_OK) {
    tri1d_destroy(op);
    nd_destroy(op);
    delete op;
    return rc;
  }
  *out = op;
  return PINT_OK;
}

int pint_op_destroy(pint_op *op) {
  if (!op) return PINT_OK;
  cudaSetDevice(op->ctx->device);
  tri1d_destroy(op);
  nd_destroy(op);
  delete op;
  return PINT_OK;
}

int pint_op_get_info(const pint_op *op, pint_op_info *info) {
  if (!op || !info) return PINT_EARG;
  memset(info, 0, sizeof(*info));
  info->dim = op->dim;
  info->steps = op->desc.steps;
  info->dtype = op->desc.dtype;
  info->rule = op->desc.rule;
  info->dt = op->dt;
  if (op->desc.ndim == 1 && op->desc.rule != PINT_RULE_FORWARD_EULER) {
    info->threads_per_slice = op->plan.T;
    info->points_per_thread = op->plan.CH;
    info->batch_cluster = op->batch_cluster;
    info->sweep_cluster = op->sweep_cluster;
    info->diag = op->plan.D;
    info->offdiag = op->plan.E;
    info->min_pivot = op->plan.min_pivot;
    info->batch_wave_slices = op->batch_wave_slices;
    info->fused_sweep = op->fused_sweep ? 1 : 0;
    info->general = op->tri_general ? 1 : 0;
    info->reserved0 = 0;
  }
  return PINT_OK;
}

static bool is_tri1d(const pint_op *op) { return op->desc.ndim == 1 && op->desc.rule != PINT_RULE_FORWARD_EULER; }
static bool is_cg(const pint_op *op) { return op->desc.ndim >= 2 && op->desc.rule == PINT_RULE_BACKWARD_EULER; }

int pint_op_apply_batch(pint_op *op, const void *in, void *out, int64_t nbatch, int64_t stride, void *stream) {
  if (!op) return PINT_EARG;
  return guarded(op->ctx, [&] {
    if (nbatch < 0) pint_throw(PINT_EARG, "nbatch must be >= 0");
    if (nbatch == 0) return;
    if (!in || !out) pint_throw(PINT_EARG, "null state pointer");
    if (stride < op->dim) pint_throw(PINT_EDIM, "stride smaller than the state dimension");
    const size_t esz = op->desc.dtype == PINT_F64 ? 8 : 4;
    const char *a = (const char *)in, *b = (const char *)out;
    const size_t span = ((size_t)(nbatch - 1) * stride + op->dim) * esz;
    if (a < b + span && b < a + span) pint_throw(PINT_EARG, "in and out must not alias");
    cudaStream_t s = (cudaStream_t)stream;
    if (is_tri1d(op)) tri1d_apply_batch(op, (const double *)in, (double *)out, nbatch, stride, s);
    else if (is_cg(op)) nd_implicit_apply_batch(op, in, out, nbatch, stride, s);
    else stencil_apply_batch(op, in, out, nbatch, stride, s);
  });
}

int pint_correct(pint_ctx *ctx, int32_t dtype, int64_t dim, int64_t nbatch, const void *gnew, const void *f,
                 const void *gold, const void *prev, void *out, const uint8_t *f_only, double *delta_dev,
                 int32_t *nonfinite_dev, void *stream) {
  if (!ctx) return PINT_EARG;
  return guarded(ctx, [&] {
    if (dtype != PINT_F32 && dtype != PINT_F64) pint_throw(PINT_EARG, "dtype must be PINT_F32 or PINT_F64");
    if (dim < 0 || nbatch < 0) pint_throw(PINT_EDIM, "negative size");
    if (nbatch == 0 || dim == 0) return;
    if (!f || !out) pint_throw(PINT_EARG, "null state pointer");
    if (!f_only && (!gnew || !gold)) pint_throw(PINT_EARG, "gnew/gold required without an F-only mask");
    correct_launch(dtype, dim, nbatch, gnew, f, gold, prev, out, f_only, delta_dev, nonfinite_dev,
                   (cudaStream_t)stream);
  });
}

int pint_coarse_init(pint_op *coarse, void *lam, int64_t p, void *gcache, void *stream) {
  if (!coarse) return PINT_EARG;
  return guarded(coarse->ctx, [&] {
    if (p < 1) pint_throw(PINT_EARG, "need p >= 1 subintervals");
    if (!lam) pint_throw(PINT_EARG, "null state pointer");
    cudaStream_t s = (cudaStream_t)stream;
    if (is_tri1d(coarse)) {
      tri1d_coarse_init(coarse, (double *)lam, p, (double *)gcache, s);
      return;
    }
    const size_t esz = coarse->desc.dtype == PINT_F64 ? 8 : 4;
    const int64_t n = coarse->dim;
    char *base = (char *)lam;
    for (int64_t i = 1; i <= p; ++i) {
      if (is_cg(coarse)) nd_implicit_apply_batch(coarse, base + (i - 1) * n * esz, base + i * n * esz, 1, n, s);
      else stencil_apply_batch(coarse, base + (i - 1) * n * esz, base + i * n * esz, 1, n, s);
    }
    if (gcache)
      PINT_CUDA(cudaMemcpyAsync(gcache, lam, (size_t)(p + 1) * n * esz, cudaMemcpyDeviceToDevice, s));
  });
}

int pint_sync_sweep(pint_op *coarse, const void *prev, void *next, const void *fv, void *gcache, int64_t k,
                    int64_t p, double *deltas_dev, int32_t *nonfinite_dev, void *stream) {
  if (!coarse) return PINT_EARG;
  return guarded(coarse->ctx, [&] {
    if (k < 1 || k > p) pint_throw(PINT_EARG, "sweep index must satisfy 1 <= k <= p");
    if (!prev || !next || !fv || !gcache || !deltas_dev || !nonfinite_dev) pint_throw(PINT_EARG, "null pointer");
    if (prev == next) pint_throw(PINT_EARG, "prev and next must be distinct iterates");
    if (!is_tri1d(coarse)) pint_throw(PINT_EUNSUPPORTED, "fused sweep is implemented for 1-D implicit coarse operators");
    tri1d_sweep(coarse, (const double *)prev, (double *)next, (const double *)fv, (double *)gcache, k, p,
                deltas_dev, nonfinite_dev, (cudaStream_t)stream, 0);
  });
}

int pint_sync_sweep_chain(pint_op *coarse, const void *prev, void *next, const void *fv, void *gcache, int64_t k,
                          int64_t p, double *deltas_dev, int32_t *nonfinite_dev, void *stream) {
  if (!coarse) return PINT_EARG;
  return guarded(coarse->ctx, [&] {
    if (k < 1 || k > p) pint_throw(PINT_EARG, "sweep index must satisfy 1 <= k <= p");
    if (!prev || !next || !fv || !gcache || !deltas_dev || !nonfinite_dev) pint_throw(PINT_EARG, "null pointer");
    if (prev == next) pint_throw(PINT_EARG, "prev and next must be distinct iterates");
    if (!is_tri1d(coarse)) pint_throw(PINT_EUNSUPPORTED, "fused sweep is implemented for 1-D implicit coarse operators");
    tri1d_sweep(coarse, (const double *)prev, (double *)next, (const double *)fv, (double *)gcache, k, p,
                deltas_dev, nonfinite_dev, (cudaStream_t)stream, 1);
  });
}

int pint_correct_chain(pint_ctx *ctx, int32_t dtype, int64_t dim, const void *gnew, const void *f, void *gcache,
                       const void *prev, void *out, const uint8_t *f_only, const double *fonly_delta_dev,
                       double *delta_dev, int32_t *nonfinite_dev, void *stream) {
  if (!ctx) return PINT_EARG;
  return guarded(ctx, [&] {
    if (dtype != PINT_F32 && dtype != PINT_F64) pint_throw(PINT_EARG, "dtype must be PINT_F32 or PINT_F64");
    if (dim < 0) pint_throw(PINT_EDIM, "negative size");
    if (dim == 0) return;
    if (!gnew || !f || !gcache || !out) pint_throw(PINT_EARG, "null state pointer");
    correct_chain_launch(dtype, dim, gnew, f, gcache, prev, out, f_only, fonly_delta_dev, delta_dev, nonfinite_dev,
                         (cudaStream_t)stream);
  });
}

int pint_equal_flag(pint_ctx *ctx, int32_t dtype, int64_t dim, const void *a, const void *b, uint8_t *equal_dev,
                    void *stream) {
  if (!ctx) return PINT_EARG;
  return guarded(ctx, [&] {
    if (dtype != PINT_F32 && dtype != PINT_F64) pint_throw(PINT_EARG, "dtype must be PINT_F32 or PINT_F64");
    if (dim < 0) pint_throw(PINT_EDIM, "negative size");
    if (!a || !b || !equal_dev) pint_throw(PINT_EARG, "null pointer");
    equal_launch(dtype, dim, a, b, equal_dev, (cudaStream_t)stream);
  });
}

int pint_max_reduce(pint_ctx *ctx, const double *deltas_dev, int64_t lo, int64_t hi, double *out_dev,
                    void *stream) {
  if (!ctx) return PINT_EARG;
  return guarded(ctx, [&] {
    if (lo < 0 || hi < lo) pint_throw(PINT_EARG, "bad range");
    max_reduce_launch(deltas_dev, lo, hi, out_dev, (cudaStream_t)stream);
  });
}

}  // extern "C"
