/* CPU ORACLE (test infrastructure only): extended-precision ground truth for
 * the 1-D implicit step maps of the reference (model.py:172-200), used where
 * fp64 algorithms disagree at the level of the problem's conditioning
 * (SURVEY §7 hard part 1). Arithmetic in long double (x87 80-bit, 64-bit
 * mantissa); inputs/outputs are double.
 *
 *   BE : (D I + E (S+S^T)) x+ = x + f                     (f at the end nodes)
 *   CN : (D I + E (S+S^T)) x+ = ((2-D) I - E (S+S^T)) x + f
 *        i.e. (I - dt/2 A) x+ = (I + dt/2 A) x + dt c with D = 1 - dt/2 a_d,
 *        E = -dt/2 a_o.
 * Thomas elimination without pivoting (K is strictly diagonally dominant).
 */
#include <stdint.h>
#include <stdlib.h>

typedef long double ld;

static void solve(int64_t n, ld D, ld E, const ld *cp, const ld *inv, ld *x) {
  /* forward */
  x[0] = x[0] * inv[0];
  for (int64_t i = 1; i < n; ++i) x[i] = (x[i] - E * x[i - 1]) * inv[i];
  for (int64_t i = n - 2; i >= 0; --i) x[i] = x[i] - cp[i] * x[i + 1];
}

/* states: nbatch x n doubles (in place); steps implicit steps each. */
int thomas_ld_propagate(int64_t n, int64_t nbatch, double *states, double Dd, double Ed, double f_first,
                        double f_last, int64_t steps, int cn, double two_minus_d) {
  ld D = Dd, E = Ed;
  ld *cp = (ld *)malloc(sizeof(ld) * n), *inv = (ld *)malloc(sizeof(ld) * n);
  ld *x = (ld *)malloc(sizeof(ld) * n), *y = (ld *)malloc(sizeof(ld) * n);
  if (!cp || !inv || !x || !y) return 1;
  ld piv = D;
  inv[0] = 1.0L / piv;
  cp[0] = E * inv[0];
  for (int64_t i = 1; i < n; ++i) {
    piv = D - E * cp[i - 1];
    inv[i] = 1.0L / piv;
    cp[i] = E * inv[i];
  }
  /* independent slices: one per OpenMP thread (private work rows) */
  int bad = 0;
#pragma omp parallel reduction(| : bad)
  {
    ld *xt = (ld *)malloc(sizeof(ld) * n), *yt = (ld *)malloc(sizeof(ld) * n);
    if (!xt || !yt) bad = 1;
#pragma omp for schedule(dynamic, 1)
    for (int64_t b = 0; b < nbatch; ++b) {
      if (!xt || !yt) continue;
      double *s = states + b * n;
      for (int64_t i = 0; i < n; ++i) xt[i] = s[i];
      for (int64_t k = 0; k < steps; ++k) {
        if (cn) {
          for (int64_t i = 0; i < n; ++i) {
            ld v = (ld)two_minus_d * xt[i];
            if (i > 0) v -= E * xt[i - 1];
            if (i < n - 1) v -= E * xt[i + 1];
            yt[i] = v;
          }
          for (int64_t i = 0; i < n; ++i) xt[i] = yt[i];
        }
        xt[0] += f_first;
        if (n > 1) xt[n - 1] += f_last;
        solve(n, D, E, cp, inv, xt);
      }
      for (int64_t i = 0; i < n; ++i) s[i] = (double)xt[i];
    }
    free(xt);
    free(yt);
  }
  if (bad) { free(cp); free(inv); free(x); free(y); return 1; }
  free(cp); free(inv); free(x); free(y);
  return 0;
}
