/*
 * oracle.c — TEST INFRASTRUCTURE ONLY.  A plain-C restatement of the
 * reference's PGD-TO projection (proj/src/projection.cpp) and of the
 * spec-only optimizer step, used as the CPU checker.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library (oracle/liboracle.so); the product path never does.
 *
 * Arithmetic contract (so results are bit-identical to the reference binary
 * compiled with the CMake Release flags, proj/CMakeLists.txt:6-8):
 *   - built with -O2 -ffp-contract=off and no -march (x86-64 SSE2): every
 *     product and sum is separately rounded, no FMA;
 *   - all reductions are sequential, left to right, exactly as the reference
 *     loops are written;
 *   - std::min(a,b) == (b < a ? b : a), std::max(a,b) == (a < b ? b : a).
 *
 * Parity status: the projection restatement is PINNED against the compiled
 * reference (oracle/_ref/libtopt_ref.so, built in place from
 * /root/reference/proj/src/projection.cpp by oracle/Makefile) on the golden
 * fixtures in tests/golden/ and on seeded random instances
 * (tests/test_oracle.py).  The m x m Newton solve (FullPivLU) follows Eigen's
 * published algorithm; Eigen itself is absent, so that boundary is
 * "parity unpinned".  The optimizer step (BB / PR+ /
 * fallback / rho_tilde) has no reference code; it restates SPEC.md and is
 * pinned only by the SPEC known-answer examples.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

static double clip(double v, double lo, double hi) { /* projection.cpp:15-17 */
  return v < lo ? lo : (v > hi ? hi : v);
}
static double dmin(double a, double b) { return (b < a) ? b : a; }
static double dmax(double a, double b) { return (a < b) ? b : a; }

static const double kGradFloor = 1e-300; /* projection.cpp:19 */

/* ---- decision trace (tests read it to measure rounding margins) ---- */
static double* g_trace = NULL;
static int64_t g_trace_cap = 0, g_trace_len = 0;
void orc_trace_set(double* buf, int64_t cap) {
  g_trace = buf;
  g_trace_cap = cap;
  g_trace_len = 0;
}
int64_t orc_trace_len(void) { return g_trace_len; }
static void trace_push(double row, double y, double r, double abs_sum) {
  if (!g_trace || g_trace_len + 4 > g_trace_cap) return;
  g_trace[g_trace_len++] = row;
  g_trace[g_trace_len++] = y;
  g_trace[g_trace_len++] = r;
  g_trace[g_trace_len++] = abs_sum;
}

/* r_j(y) = -ghat_j + sum_i a_i clip(y a_i, l - rho_i, u - rho_i)
 * projection.cpp:25-38 (sequential over all i or over the subset order). */
static double row_residual(const double* a, const double* rho, int64_t n, const int32_t* sub,
                           int64_t nsub, double lower, double upper, double yj, double ghat,
                           int row) {
  double r = -ghat, abs_sum = fabs(ghat);
  if (sub) {
    for (int64_t k = 0; k < nsub; ++k) {
      const int32_t i = sub[k];
      const double t = a[i] * clip(yj * a[i], lower - rho[i], upper - rho[i]);
      r += t;
      abs_sum += fabs(t);
    }
  } else {
    for (int64_t i = 0; i < n; ++i) {
      const double t = a[i] * clip(yj * a[i], lower - rho[i], upper - rho[i]);
      r += t;
      abs_sum += fabs(t);
    }
  }
  trace_push((double)row, yj, r, abs_sum);
  return r;
}

/* Algorithm-1 bisection, projection.cpp:48-110.  Returns 0 or ORC_INFEASIBLE. */
int orc_binary_search_row(const double* a, const double* rho, int64_t n, const int32_t* sub,
                          int64_t nsub, double lower, double upper, double ghat, int equality,
                          double tol_b, int maxiter, int row, double* y_out,
                          double* residual_out, int* iters_out) {
  const double r0 = row_residual(a, rho, n, sub, nsub, lower, upper, 0.0, ghat, row);
  *iters_out = 0;
  if (!equality && r0 <= 0.0) {
    *y_out = 0.0;
    *residual_out = dmax(r0, 0.0);
    return 0;
  }
  if (equality && r0 == 0.0) {
    *y_out = 0.0;
    *residual_out = 0.0;
    return 0;
  }
  double bp_lo = 0.0, bp_hi = 0.0;
  int any = 0;
  const int64_t cnt = sub ? nsub : n;
  for (int64_t k = 0; k < cnt; ++k) { /* projection.cpp:60-73 */
    const int64_t i = sub ? sub[k] : k;
    const double ai = a[i];
    if (fabs(ai) < kGradFloor) continue;
    any = 1;
    const double c1 = (lower - rho[i]) / ai;
    const double c2 = (upper - rho[i]) / ai;
    bp_lo = dmin(bp_lo, dmin(c1, c2));
    bp_hi = dmax(bp_hi, dmax(c1, c2));
  }
  if (!any) return ORC_INFEASIBLE;
  double y_lo, y_hi;
  if (r0 > 0.0) {
    y_lo = bp_lo;
    y_hi = 0.0;
    if (row_residual(a, rho, n, sub, nsub, lower, upper, y_lo, ghat, row) > 0.0)
      return ORC_INFEASIBLE;
  } else {
    y_lo = 0.0;
    y_hi = bp_hi;
    if (row_residual(a, rho, n, sub, nsub, lower, upper, y_hi, ghat, row) < 0.0)
      return ORC_INFEASIBLE;
  }
  int iters = 0;
  double ym = 0.5 * (y_lo + y_hi);
  while ((y_hi - y_lo) > tol_b && iters < maxiter) { /* projection.cpp:97-106 */
    const double rm = row_residual(a, rho, n, sub, nsub, lower, upper, ym, ghat, row);
    if (rm > 0.0)
      y_hi = ym;
    else
      y_lo = ym;
    ym = 0.5 * (y_lo + y_hi);
    ++iters;
  }
  *y_out = ym;
  *residual_out = fabs(row_residual(a, rho, n, sub, nsub, lower, upper, ym, ghat, row));
  *iters_out = iters;
  return 0;
}

/* ConstraintLinearization::build's g_hat, projection.cpp:139-145. */
void orc_build_ghat(int64_t n, int64_t m, const double* grad, const double* g_values,
                    const double* bounds_g, const double* gd_step, double* ghat) {
  for (int64_t j = 0; j < m; ++j) {
    double dot = 0.0;
    const double* a = grad + j * n;
    for (int64_t i = 0; i < n; ++i) dot += gd_step[i] * a[i];
    ghat[j] = bounds_g[j] - g_values[j] + dot;
  }
}

/* ConstraintLinearization::validate, projection.cpp:150-181. */
int orc_validate(int64_t n, int64_t m, const double* grad, const double* g_values,
                 const double* bounds_g, const double* gd_step, const double* ghat,
                 const int64_t* off, const int32_t* idx) {
  for (int64_t j = 0; j < m; ++j) {
    double dot = 0.0;
    const double* a = grad + j * n;
    for (int64_t i = 0; i < n; ++i) dot += gd_step[i] * a[i];
    const double expect = bounds_g[j] - g_values[j] + dot;
    const double scale = dmax(dmax(1.0, fabs(expect)), fabs(ghat[j]));
    if (fabs(ghat[j] - expect) > 1e-14 * scale) return ORC_DOMAIN;
  }
  if (!off) return 0;
  uint8_t* owner = (uint8_t*)calloc((size_t)n, 1);
  int rc = 0;
  for (int64_t j = 0; j < m && !rc; ++j)
    for (int64_t k = off[j]; k < off[j + 1]; ++k) {
      const int32_t i = idx[k];
      if (i < 0 || i >= n) { rc = ORC_DOMAIN; break; }
      if (owner[i]++) { rc = ORC_DOMAIN; break; }
    }
  for (int64_t j = 0; j < m && !rc; ++j) {
    memset(owner, 0, (size_t)n);
    for (int64_t k = off[j]; k < off[j + 1]; ++k) owner[idx[k]] = 1;
    const double* a = grad + j * n;
    for (int64_t i = 0; i < n; ++i)
      if (!owner[i] && a[i] != 0.0) { rc = ORC_DOMAIN; break; }
  }
  free(owner);
  return rc;
}

/* delta_of_y, projection.cpp:192-209. */
void orc_delta_of_y(int64_t n, int64_t m, const double* y, const double* grad,
                    const double* rho, double lower, double upper, double* z) {
  for (int64_t i = 0; i < n; ++i) z[i] = 0.0;
  for (int64_t j = 0; j < m; ++j) {
    const double yj = y[j];
    if (yj == 0.0) continue;
    const double* a = grad + j * n;
    for (int64_t i = 0; i < n; ++i) z[i] += yj * a[i];
  }
  for (int64_t i = 0; i < n; ++i) z[i] = clip(z[i], lower - rho[i], upper - rho[i]);
}

/* constraint_residual_h, projection.cpp:253-267. */
int orc_residual_h(int64_t n, int64_t m, const double* y, const double* grad,
                   const double* ghat, const double* rho, double lower, double upper,
                   double c, double* h) {
  if (!(c > 0.0)) return ORC_PARAMETER;
  double* delta = (double*)malloc(sizeof(double) * (size_t)n);
  orc_delta_of_y(n, m, y, grad, rho, lower, upper, delta);
  for (int64_t j = 0; j < m; ++j) {
    const double* a = grad + j * n;
    double dot = 0.0;
    for (int64_t i = 0; i < n; ++i) dot += a[i] * delta[i];
    h[j] = dot + y[j] / c - ghat[j];
  }
  free(delta);
  return 0;
}

/* eval_phi, projection.cpp:279-298. */
static double eval_phi(int64_t n, int64_t m, const double* y, const double* grad,
                       const double* ghat, const uint8_t* is_eq, const double* rho,
                       double lower, double upper, double c, double* delta, double* h,
                       double* phi) {
  orc_delta_of_y(n, m, y, grad, rho, lower, upper, delta);
  for (int64_t j = 0; j < m; ++j) {
    const double* a = grad + j * n;
    double dot = 0.0;
    for (int64_t i = 0; i < n; ++i) dot += a[i] * delta[i];
    h[j] = dot + y[j] / c - ghat[j];
    phi[j] = is_eq[j] ? h[j] : dmin(-y[j], -h[j]);
  }
  double sq = 0.0;
  for (int64_t j = 0; j < m; ++j) sq += phi[j] * phi[j];
  return 0.5 * sq;
}

static double linf(const double* v, int64_t m) {
  double r = 0.0;
  for (int64_t j = 0; j < m; ++j) r = dmax(r, fabs(v[j]));
  return r;
}

/* Full-pivot LU + solve, mirroring the shim / Eigen::FullPivLU (projection.cpp:401-407).
 * a is m x m column-major and is overwritten.  Returns 0, or ORC_NUMERICAL when
 * the matrix is not invertible (rank < m at threshold eps*m*|maxpivot|). */
int orc_fullpiv_solve(int64_t m, double* a, const double* b, double* x) {
  int64_t rowperm[64], colperm[64];
  if (m > 64) return ORC_DOMAIN;
#define A(i, j) a[(j) * m + (i)]
  for (int64_t i = 0; i < m; ++i) rowperm[i] = colperm[i] = i;
  int64_t nz = m;
  double maxpivot = 0.0;
  for (int64_t k = 0; k < m; ++k) {
    double biggest = -1.0;
    int64_t br = k, bc = k;
    for (int64_t j = k; j < m; ++j)
      for (int64_t i = k; i < m; ++i) {
        const double v = fabs(A(i, j));
        if (v > biggest) { biggest = v; br = i; bc = j; }
      }
    if (biggest == 0.0) { nz = k; break; }
    if (biggest > maxpivot) maxpivot = biggest;
    if (br != k) {
      for (int64_t j = 0; j < m; ++j) { double t = A(k, j); A(k, j) = A(br, j); A(br, j) = t; }
      int64_t t = rowperm[k]; rowperm[k] = rowperm[br]; rowperm[br] = t;
    }
    if (bc != k) {
      for (int64_t i = 0; i < m; ++i) { double t = A(i, k); A(i, k) = A(i, bc); A(i, bc) = t; }
      int64_t t = colperm[k]; colperm[k] = colperm[bc]; colperm[bc] = t;
    }
    const double piv = A(k, k);
    for (int64_t i = k + 1; i < m; ++i) A(i, k) /= piv;
    for (int64_t j = k + 1; j < m; ++j)
      for (int64_t i = k + 1; i < m; ++i) A(i, j) -= A(i, k) * A(k, j);
  }
  const double thr = fabs(maxpivot) * 2.220446049250313e-16 * (double)m;
  int64_t rank = 0;
  for (int64_t i = 0; i < nz; ++i) rank += (fabs(A(i, i)) > thr);
  if (rank != m) return ORC_NUMERICAL;
  double c[64];
  for (int64_t i = 0; i < m; ++i) c[i] = b[rowperm[i]];
  for (int64_t i = 0; i < m; ++i) {
    double s = c[i];
    for (int64_t k = 0; k < i; ++k) s -= A(i, k) * c[k];
    c[i] = s;
  }
  for (int64_t i = nz - 1; i >= 0; --i) {
    double s = c[i];
    for (int64_t k = i + 1; k < nz; ++k) s -= A(i, k) * c[k];
    c[i] = s / A(i, i);
  }
  for (int64_t i = 0; i < m; ++i) x[colperm[i]] = (i < nz) ? c[i] : 0.0;
#undef A
  return 0;
}

static void fill_result_zero(int64_t m, double* y, double* slacks) {
  for (int64_t j = 0; j < m; ++j) { y[j] = 0.0; slacks[j] = 0.0; }
}

/* project_general_newton, projection.cpp:302-438. */
int orc_project_newton(int64_t n, int64_t m, const double* rho, const double* grad,
                       const double* ghat, const uint8_t* is_eq, double lower, double upper,
                       const orc_opts* o, double* delta, double* y_out, double* slacks,
                       orc_meta* meta) {
  if (m < 1) return ORC_DOMAIN;
  if (m > 64) return ORC_DOMAIN;
  double ytrial[64];
  /* Stage 1 (projection.cpp:312-343) */
  for (int64_t j = 0; j < m; ++j) {
    double yj, res;
    int it;
    if (orc_binary_search_row(grad + j * n, rho, n, NULL, 0, lower, upper, ghat[j], is_eq[j],
                              o->tol_b, o->binary_maxiter, (int)j, &yj, &res, &it))
      continue;
    for (int64_t k = 0; k < m; ++k) ytrial[k] = 0.0;
    ytrial[j] = yj;
    orc_delta_of_y(n, m, ytrial, grad, rho, lower, upper, delta);
    int feasible = 1;
    double worst = 0.0;
    for (int64_t k = 0; k < m && feasible; ++k) {
      const double* a = grad + k * n;
      double dot = 0.0;
      for (int64_t i = 0; i < n; ++i) dot += a[i] * delta[i];
      const double v = dot - ghat[k];
      const double viol = is_eq[k] ? fabs(v) : v;
      feasible = viol <= o->tol_n;
      worst = dmax(worst, fabs(v));
    }
    if (feasible) {
      fill_result_zero(m, y_out, slacks);
      y_out[j] = yj;
      meta->path = ORC_PATH_SINGLE;
      meta->newton_iters = 0;
      meta->converged = 1;
      meta->curvature_violations = 0;
      meta->residual = worst;
      meta->stage1_row = (int)j;
      return 0;
    }
  }
  /* Stage 2 (projection.cpp:345-437) */
  double* z = (double*)malloc(sizeof(double) * (size_t)n);
  double* tdelta = (double*)malloc(sizeof(double) * (size_t)n);
  double y[64], h[64], phi[64], th[64], tphi[64], step[64], jh[64 * 64], jphi[64 * 64],
      lu[64 * 64];
  for (int64_t j = 0; j < m; ++j) y[j] = 0.0;
  double merit = eval_phi(n, m, y, grad, ghat, is_eq, rho, lower, upper, o->c, delta, h, phi);
  int iters = 0, curv_viol = 0, have_prev = 0, rc = 0;
  double prev_phi_sq = 0.0;
#define JH(i, j) jh[(j) * m + (i)]
#define JP(i, j) jphi[(j) * m + (i)]
  while (linf(phi, m) > o->tol_n && iters < o->newton_maxiter) {
    for (int64_t k = 0; k < m * m; ++k) jh[k] = 0.0;
    for (int64_t i = 0; i < n; ++i) z[i] = 0.0;
    for (int64_t j = 0; j < m; ++j) {
      if (y[j] == 0.0) continue;
      const double* a = grad + j * n;
      for (int64_t i = 0; i < n; ++i) z[i] += y[j] * a[i];
    }
    for (int64_t i = 0; i < n; ++i) {
      if (z[i] < lower - rho[i] || z[i] > upper - rho[i]) continue;
      for (int64_t j = 0; j < m; ++j) {
        const double aji = grad[j * n + i];
        if (aji == 0.0) continue;
        for (int64_t k = j; k < m; ++k) JH(j, k) += aji * grad[k * n + i];
      }
    }
    for (int64_t j = 0; j < m; ++j) {
      for (int64_t k = j + 1; k < m; ++k) JH(k, j) = JH(j, k);
      JH(j, j) += 1.0 / o->c;
    }
    for (int64_t j = 0; j < m; ++j) {
      if (is_eq[j]) {
        for (int64_t k = 0; k < m; ++k) JP(j, k) = JH(j, k);
      } else if (-y[j] <= -h[j]) {
        for (int64_t k = 0; k < m; ++k) JP(j, k) = 0.0;
        JP(j, j) = -1.0;
      } else {
        for (int64_t k = 0; k < m; ++k) JP(j, k) = -JH(j, k);
      }
    }
    if (have_prev) { /* projection.cpp:396-399 */
      double curv = 0.0;
      for (int64_t j = 0; j < m; ++j) {
        double s = 0.0;
        for (int64_t k = 0; k < m; ++k) s += JP(j, k) * step[k];
        curv += phi[j] * s;
      }
      if (curv > 0.9 * prev_phi_sq) ++curv_viol;
    }
    memcpy(lu, jphi, sizeof(double) * (size_t)(m * m));
    if (orc_fullpiv_solve(m, lu, phi, step)) { rc = ORC_NUMERICAL; break; }
    int finite = 1;
    for (int64_t j = 0; j < m; ++j) finite &= isfinite(step[j]) ? 1 : 0;
    if (!finite) { rc = ORC_NUMERICAL; break; }
    double phi_sq = 0.0;
    for (int64_t j = 0; j < m; ++j) phi_sq += phi[j] * phi[j];
    const double merit0 = merit;
    const double c1 = 1e-4;
    double gamma = 1.0, tmerit;
    for (;;) { /* Armijo, projection.cpp:418-422 */
      for (int64_t j = 0; j < m; ++j) ytrial[j] = y[j] - gamma * step[j];
      tmerit = eval_phi(n, m, ytrial, grad, ghat, is_eq, rho, lower, upper, o->c, tdelta, th,
                        tphi);
      if (tmerit <= merit0 - c1 * gamma * phi_sq || gamma < 1e-16) break;
      gamma *= 0.5;
    }
    for (int64_t j = 0; j < m; ++j) y[j] -= gamma * step[j];
    for (int64_t j = 0; j < m; ++j) step[j] *= gamma;
    prev_phi_sq = gamma * phi_sq;
    have_prev = 1;
    memcpy(delta, tdelta, sizeof(double) * (size_t)n);
    memcpy(h, th, sizeof(double) * (size_t)m);
    memcpy(phi, tphi, sizeof(double) * (size_t)m);
    merit = tmerit;
    ++iters;
    if (meta->iter_trace) {
      meta->iter_trace[iters - 1] = gamma;
      if (iters - 1 < 64) meta->iter_trace[64 + iters - 1] = linf(phi, m);
    }
  }
#undef JH
#undef JP
  free(z);
  free(tdelta);
  if (rc) return rc;
  meta->residual = linf(phi, m);
  meta->converged = meta->residual <= o->tol_n;
  meta->path = ORC_PATH_NEWTON;
  meta->newton_iters = iters;
  meta->curvature_violations = curv_viol;
  meta->stage1_row = -1;
  for (int64_t j = 0; j < m; ++j) {
    y_out[j] = y[j];
    slacks[j] = -y[j] / o->c;
  }
  return 0;
}

/* project_single_binary_search, projection.cpp:211-227. */
int orc_project_single(int64_t n, int64_t m, const double* rho, const double* grad,
                       const double* ghat, const uint8_t* is_eq, double lower, double upper,
                       double tol_b, int maxiter, double* delta, double* y, double* slacks,
                       orc_meta* meta) {
  if (m != 1) return ORC_DOMAIN;
  double yj, res;
  int it;
  int rc = orc_binary_search_row(grad, rho, n, NULL, 0, lower, upper, ghat[0], is_eq[0], tol_b,
                                 maxiter, 0, &yj, &res, &it);
  if (rc) return rc;
  y[0] = yj;
  slacks[0] = 0.0;
  orc_delta_of_y(n, 1, y, grad, rho, lower, upper, delta);
  meta->path = ORC_PATH_SINGLE;
  meta->residual = res;
  meta->newton_iters = 0;
  meta->converged = 1;
  meta->curvature_violations = 0;
  meta->bisect_iters[0] = it;
  meta->stage1_row = -1;
  return 0;
}

/* project_independent, projection.cpp:229-251 (validate() included). */
int orc_project_independent(int64_t n, int64_t m, const double* rho, const double* grad,
                            const double* g_values, const double* bounds_g,
                            const double* gd_step, const double* ghat, const uint8_t* is_eq,
                            const int64_t* off, const int32_t* idx, double lower, double upper,
                            double tol_b, int maxiter, double* delta, double* y, double* slacks,
                            orc_meta* meta) {
  if (!off) return ORC_DOMAIN;
  int rc = orc_validate(n, m, grad, g_values, bounds_g, gd_step, ghat, off, idx);
  if (rc) return rc;
  double worst = 0.0;
  for (int64_t j = 0; j < m; ++j) {
    double yj, res;
    int it;
    rc = orc_binary_search_row(grad + j * n, rho, n, idx + off[j], off[j + 1] - off[j], lower,
                               upper, ghat[j], is_eq[j], tol_b, maxiter, (int)j, &yj, &res, &it);
    if (rc) return rc;
    y[j] = yj;
    slacks[j] = 0.0;
    worst = dmax(worst, res);
    if (j < ORC_MAX_TRACE_ROWS) meta->bisect_iters[j] = it;
  }
  orc_delta_of_y(n, m, y, grad, rho, lower, upper, delta);
  meta->path = ORC_PATH_INDEPENDENT;
  meta->residual = worst;
  meta->newton_iters = 0;
  meta->converged = 1;
  meta->curvature_violations = 0;
  meta->stage1_row = -1;
  return 0;
}

/* project dispatch, projection.cpp:440-460. */
int orc_project(int64_t n, int64_t m, const double* rho, const double* grad,
                const double* g_values, const double* bounds_g, const double* gd_step,
                const double* ghat, const uint8_t* is_eq, const int64_t* off,
                const int32_t* idx, double lower, double upper, const orc_opts* o,
                double* delta, double* y, double* slacks, orc_meta* meta) {
  int rc;
  if (m == 1) {
    rc = orc_project_single(n, m, rho, grad, ghat, is_eq, lower, upper, o->tol_b,
                            o->binary_maxiter, delta, y, slacks, meta);
    if (rc != ORC_INFEASIBLE) return rc;
    return orc_project_newton(n, m, rho, grad, ghat, is_eq, lower, upper, o, delta, y, slacks,
                              meta);
  }
  if (off) {
    rc = orc_project_independent(n, m, rho, grad, g_values, bounds_g, gd_step, ghat, is_eq, off,
                                 idx, lower, upper, o->tol_b, o->binary_maxiter, delta, y,
                                 slacks, meta);
    if (rc != ORC_INFEASIBLE) return rc;
  }
  return orc_project_newton(n, m, rho, grad, ghat, is_eq, lower, upper, o, delta, y, slacks,
                            meta);
}

/* ------------------------------------------------------------------------
 * Optimizer step (spec-only in the reference: SPEC.md:272-358)
 * ---------------------------------------------------------------------- */

/* spectral_step_size, SPEC.md:287-295 (Eq. 13). */
double orc_spectral_step_size(int64_t n, const double* x, const double* x_prev,
                              const double* g, const double* g_prev, double alpha_max,
                              double eps_alpha) {
  double ss = 0.0, sy = 0.0, yy = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double s = x[i] - x_prev[i];
    const double y = g[i] - g_prev[i];
    ss += s * s;
    sy += s * y;
    yy += y * y;
  }
  return orc_spectral_from_sums(ss, sy, yy, alpha_max, eps_alpha);
}

double orc_spectral_from_sums(double ss, double sy, double yy, double alpha_max,
                              double eps_alpha) {
  if (yy == 0.0) return alpha_max;
  const double ns = sqrt(ss), ny = sqrt(yy);
  if (sy <= eps_alpha) return dmin(ns / ny, alpha_max);
  return dmin(dmin(ss / sy, 2.0 * ns / ny), alpha_max);
}

/* PR+ coefficient, SPEC.md:296-304 (Eq. 14). */
double orc_pr_beta(int64_t n, const double* g, const double* g_prev) {
  double num = 0.0, den = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    num += g[i] * (g[i] - g_prev[i]);
    den += g_prev[i] * g_prev[i];
  }
  return orc_pr_beta_from_sums(num, den);
}

double orc_pr_beta_from_sums(double num, double den) {
  if (den == 0.0) return 0.0;
  return dmax(num / den, 0.0);
}

/* pgd_step's pre-projection half, SPEC.md:305-313 / PAPER.md Alg. 3 lines 2-9:
 *   fallback  = t == 0 || (t >= t_warmup && violation > tol_N)
 *   alpha     = fallback ? min(alpha_max, alpha_fallback / ||g||_inf) : spectral
 *   d         = fallback ? g : g + beta * d_prev        (CG memory reset on fallback)
 *   gd_step   = (omega * alpha) * d ;  rho_tilde = x - gd_step
 * Writes d, gd_step, rho_tilde; returns alpha/beta/fallback in *st. */
void orc_step_direction(int64_t n, const double* x, const double* x_prev, const double* g,
                        const double* g_prev, const double* d_prev, int t, double violation,
                        const orc_pgd_settings* s, double* d, double* gd_step,
                        double* rho_tilde, orc_step_info* st) {
  const int fallback = (t == 0) || (t >= s->t_warmup && violation > s->tol_n);
  double alpha, beta = 0.0;
  if (fallback) {
    double ginf = 0.0;
    for (int64_t i = 0; i < n; ++i) ginf = dmax(ginf, fabs(g[i]));
    alpha = dmin(s->alpha_max, s->alpha_fallback / ginf);
  } else {
    alpha = orc_spectral_step_size(n, x, x_prev, g, g_prev, s->alpha_max, s->eps_alpha);
    beta = orc_pr_beta(n, g, g_prev);
  }
  const double wa = s->omega * alpha;
  for (int64_t i = 0; i < n; ++i) {
    d[i] = fallback ? g[i] : g[i] + beta * d_prev[i];
    gd_step[i] = wa * d[i];
    rho_tilde[i] = x[i] - gd_step[i];
  }
  st->alpha = alpha;
  st->beta = beta;
  st->fallback = fallback;
}
