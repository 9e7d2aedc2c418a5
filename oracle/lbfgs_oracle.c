/* lbfgs_oracle.c — TEST INFRASTRUCTURE ONLY (checker / CPU baseline).
 *
 * Float64 restatement of the staged L-BFGS program oracle/programs/lbfgs_m*.msl
 * (BASELINE config C4) as the reference executor evaluates it:
 * every element-wise node is one pass in the node's operand order
 * (reference pkg/src/stagekit/graph/tensor.py:274-287, no FMA contraction),
 * every m.reduce_sum is the reference's left-to-right sum starting at 0.0
 * (tensor.py:335-341), `%` is Python floor-mod (the indices are >= 0 here),
 * `and` in the loop test is the lazy Cond (runtime/dispatch.py:126-146) and
 * the loop is graph/execute.py:218-238.  Bit-exact with the reference on the
 * golden fixtures (tests/test_oracle.py).
 *
 *   oracle_lbfgs(n, m, x0, a, b, tol, max_iter, x_out, margin_out) -> k, or -13
 *   (DivisionByZero when s.y == 0 or y.y == 0).
 *   margin_out = min over evaluated loop tests of |gnorm - tol| / tol: how far
 *   the data-dependent trip count is from flipping.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static double dot(const double* u, const double* v, int64_t n) {
  double acc = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double p = u[i] * v[i];
    acc += p;
  }
  return acc;
}

int64_t oracle_lbfgs(int64_t n, int m, const double* x0, const double* a, const double* b, double tol,
                     int64_t max_iter, double* x_out, double* margin_out) {
  double* x = malloc(n * sizeof(double));
  double* g = malloc(n * sizeof(double));
  double* q = malloc(n * sizeof(double));
  double* r = malloc(n * sizeof(double));
  double* xn = malloc(n * sizeof(double));
  double* gn = malloc(n * sizeof(double));
  double* ss = calloc((size_t)m * n, sizeof(double));
  double* ys = calloc((size_t)m * n, sizeof(double));
  double* rhos = calloc(m, sizeof(double));
  double* alphas = calloc(m, sizeof(double));
  int64_t k = 0, status = 0;
  double margin = INFINITY;
  memcpy(x, x0, n * sizeof(double));
  for (int64_t i = 0; i < n; ++i) { const double t = a[i] * x[i]; g[i] = t - b[i]; }   /* grad */
  double gamma = 1.0;
  double gnorm = dot(g, g, n);
  for (;;) {
    if (!(k < max_iter)) break;
    const double mg = fabs(gnorm - tol) / tol;
    if (mg < margin) margin = mg;
    if (!(gnorm > tol)) break;
    memcpy(q, g, n * sizeof(double));
    for (int j = 0; j < m; ++j) {
      if (!(j < k)) continue;
      const int64_t idx = ((k - 1 - j) % m + m) % m;
      const double* s = ss + idx * n;
      const double* y = ys + idx * n;
      const double al = rhos[idx] * dot(s, q, n);
      alphas[idx] = al;
      for (int64_t i = 0; i < n; ++i) { const double t = al * y[i]; q[i] = q[i] - t; }
    }
    for (int64_t i = 0; i < n; ++i) r[i] = gamma * q[i];
    const int64_t nh = k < m ? k : m;
    for (int j = 0; j < m; ++j) {
      if (!(j < nh)) continue;
      const int64_t idx = ((k - nh + j) % m + m) % m;
      const double* s = ss + idx * n;
      const double* y = ys + idx * n;
      const double be = rhos[idx] * dot(y, r, n);
      const double c = alphas[idx] - be;
      for (int64_t i = 0; i < n; ++i) { const double t = s[i] * c; r[i] = r[i] + t; }
    }
    const int64_t slot = k % m;
    double* s = ss + slot * n;
    double* y = ys + slot * n;
    for (int64_t i = 0; i < n; ++i) {
      xn[i] = x[i] - r[i];
      const double t = a[i] * xn[i];
      gn[i] = t - b[i];
    }
    /* s = xn - x and y = gn - g become the new history entries */
    for (int64_t i = 0; i < n; ++i) { s[i] = xn[i] - x[i]; y[i] = gn[i] - g[i]; }
    const double sy = dot(s, y, n);
    const double yy = dot(y, y, n);
    gnorm = dot(gn, gn, n);
    if (sy == 0.0 || yy == 0.0) { status = -13; break; }
    rhos[slot] = 1.0 / sy;
    gamma = sy / yy;
    double* t;
    t = x; x = xn; xn = t;
    t = g; g = gn; gn = t;
    ++k;
  }
  memcpy(x_out, x, n * sizeof(double));
  if (margin_out) *margin_out = margin;
  free(x); free(g); free(q); free(r); free(xn); free(gn); free(ss); free(ys); free(rhos); free(alphas);
  return status ? status : k;
}
