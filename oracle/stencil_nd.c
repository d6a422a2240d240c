/* CPU ORACLE (test infrastructure only): the explicit forward-Euler fine map
 * of the 1-D/2-D/3-D zero-Dirichlet heat operator, u <- (I + dt A)^S u, the
 * reference's route fine_from_onestep(AffinePropagator(I + dt A, dt c, 1), S)
 * (model.py:147-154; A = h^-2 x the 3/5/7-point Laplacian, model.py:209-235
 * for 1-D, Kronecker sums for 2-D/3-D). Restated matrix-free, one sweep per
 * step, so config-size grids (1024^2, 256^3, 512^3) run in seconds.
 *
 * The per-point expression is fixed (no compiler contraction: build with
 * -ffp-contract=off) and is the one the GPU kernels evaluate, so the fp32 and
 * fp64 maps are comparable BITWISE with the device:
 *   1-D: nb = x- + x+;                          v = fma(r, fma(-2, c, nb), c)
 *   2-D: nb = (x- + x+) + (y- + y+);            v = fma(r, fma(-4, c, nb), c)
 *   3-D: nb = ((x- + x+) + (y- + y+)) + (z- + z+);  v = fma(r, fma(-6, c, nb), c)
 * Zero Dirichlet: neighbours outside the grid are 0.
 * The long-double variant evaluates the same map in x87 extended precision:
 * the exact-arithmetic answer to the fp64 problem (rounding floor of fp64).
 *
 * Layout: C order, last axis (x) fastest; states are nbatch contiguous grids,
 * updated in place. Threads: OpenMP over the slowest axis of each step.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define DEFINE_FE(NAME, T, FMA)                                                                   \
  static void NAME##_step(int ndim, int64_t nz, int64_t ny, int64_t nx, const T *u, T *o, T r) { \
    const int64_t sy = nx, sz = nx * ny;                                                         \
    if (ndim == 1) {                                                                             \
      _Pragma("omp parallel for schedule(static) if (nx > 65536)")                               \
      for (int64_t i = 0; i < nx; ++i) {                                                          \
        const T xm = i > 0 ? u[i - 1] : (T)0, xp = i < nx - 1 ? u[i + 1] : (T)0;                 \
        const T nb = xm + xp;                                                                    \
        o[i] = FMA(r, FMA((T)-2, u[i], nb), u[i]);                                               \
      }                                                                                          \
    } else if (ndim == 2) {                                                                      \
      _Pragma("omp parallel for schedule(static)")                                               \
      for (int64_t y = 0; y < ny; ++y) {                                                          \
        const T *row = u + y * sy;                                                               \
        for (int64_t x = 0; x < nx; ++x) {                                                        \
          const T c = row[x];                                                                    \
          const T xm = x > 0 ? row[x - 1] : (T)0, xp = x < nx - 1 ? row[x + 1] : (T)0;           \
          const T ym = y > 0 ? row[x - sy] : (T)0, yp = y < ny - 1 ? row[x + sy] : (T)0;         \
          const T nb = (xm + xp) + (ym + yp);                                                    \
          o[y * sy + x] = FMA(r, FMA((T)-4, c, nb), c);                                          \
        }                                                                                        \
      }                                                                                          \
    } else {                                                                                     \
      _Pragma("omp parallel for collapse(2) schedule(static)")                                   \
      for (int64_t z = 0; z < nz; ++z)                                                            \
        for (int64_t y = 0; y < ny; ++y) {                                                        \
          const T *row = u + z * sz + y * sy;                                                    \
          for (int64_t x = 0; x < nx; ++x) {                                                      \
            const T c = row[x];                                                                  \
            const T xm = x > 0 ? row[x - 1] : (T)0, xp = x < nx - 1 ? row[x + 1] : (T)0;         \
            const T ym = y > 0 ? row[x - sy] : (T)0, yp = y < ny - 1 ? row[x + sy] : (T)0;       \
            const T zm = z > 0 ? row[x - sz] : (T)0, zp = z < nz - 1 ? row[x + sz] : (T)0;       \
            const T nb = ((xm + xp) + (ym + yp)) + (zm + zp);                                    \
            o[z * sz + y * sy + x] = FMA(r, FMA((T)-6, c, nb), c);                               \
          }                                                                                      \
        }                                                                                        \
    }                                                                                            \
  }

DEFINE_FE(fe_f64, double, fma)
DEFINE_FE(fe_f32, float, fmaf)
DEFINE_FE(fe_ld, long double, fmal)

/* states: nbatch grids of nz*ny*nx (ndim 1: nx only; 2: ny*nx), in place. */
int fe_nd_f64(int ndim, int64_t nz, int64_t ny, int64_t nx, double *states, int64_t nbatch, double r,
              int64_t steps) {
  const int64_t n = (ndim >= 3 ? nz : 1) * (ndim >= 2 ? ny : 1) * nx;
  double *tmp = (double *)malloc(sizeof(double) * n);
  if (!tmp) return 1;
  for (int64_t b = 0; b < nbatch; ++b) {
    double *a = states + b * n, *x = a, *y = tmp;
    for (int64_t s = 0; s < steps; ++s) {
      fe_f64_step(ndim, nz, ny, nx, x, y, r);
      double *t = x; x = y; y = t;
    }
    if (x != a) memcpy(a, x, sizeof(double) * n);
  }
  free(tmp);
  return 0;
}

int fe_nd_f32(int ndim, int64_t nz, int64_t ny, int64_t nx, float *states, int64_t nbatch, float r,
              int64_t steps) {
  const int64_t n = (ndim >= 3 ? nz : 1) * (ndim >= 2 ? ny : 1) * nx;
  float *tmp = (float *)malloc(sizeof(float) * n);
  if (!tmp) return 1;
  for (int64_t b = 0; b < nbatch; ++b) {
    float *a = states + b * n, *x = a, *y = tmp;
    for (int64_t s = 0; s < steps; ++s) {
      fe_f32_step(ndim, nz, ny, nx, x, y, r);
      float *t = x; x = y; y = t;
    }
    if (x != a) memcpy(a, x, sizeof(float) * n);
  }
  free(tmp);
  return 0;
}

/* Extended precision: double in/out, long double state between steps. */
int fe_nd_ld(int ndim, int64_t nz, int64_t ny, int64_t nx, double *states, int64_t nbatch, double r,
             int64_t steps) {
  const int64_t n = (ndim >= 3 ? nz : 1) * (ndim >= 2 ? ny : 1) * nx;
  long double *x = (long double *)malloc(sizeof(long double) * n);
  long double *y = (long double *)malloc(sizeof(long double) * n);
  if (!x || !y) return 1;
  for (int64_t b = 0; b < nbatch; ++b) {
    double *a = states + b * n;
    for (int64_t i = 0; i < n; ++i) x[i] = a[i];
    long double *p = x, *q = y;
    for (int64_t s = 0; s < steps; ++s) {
      fe_ld_step(ndim, nz, ny, nx, p, q, (long double)r);
      long double *t = p; p = q; q = t;
    }
    for (int64_t i = 0; i < n; ++i) a[i] = (double)p[i];
  }
  free(x);
  free(y);
  return 0;
}
