/* TEST INFRASTRUCTURE ONLY — the enumeration oracle of the reference's spec
 * (reference_projection_oracle; not
 * implemented in the reference).  Exact projection of rho_tilde onto
 *     { delta : l - rho <= delta <= u - rho,  a_j . delta <= ghat_j (j ineq),
 *                                             a_j . delta  = ghat_j (j eq) }
 * minimising 1/2 ||delta||^2, by enumerating all 3^N box-activity patterns
 * (lower / free / upper) x 2^m constraint-activity patterns (equality rows
 * always active), solving each equality-constrained least-squares candidate
 *     delta_F = A_JF^T mu,  (A_JF A_JF^T) mu = ghat_J - A_JB delta_B,
 * and keeping the candidates that satisfy the KKT sign conditions
 * ("filtering by KKT signs, returning the feasible candidate with
 * minimum ||delta||").  Sign convention of the reference:
 * mu = y <= 0 on active inequality rows, delta = clip(A^T mu, l - rho, u - rho).
 * Limits: N <= 12, m <= 3.  Used by tests/ only.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

enum { ENUM_OK = 0, ENUM_INFEASIBLE = 1, ENUM_TOO_LARGE = 2 };

/* Solve the k x k SPD-ish system M x = b (k <= 3) by Gaussian elimination with
 * partial pivoting; returns 0 if (numerically) singular. */
static int solve_small(int k, double M[3][3], double b[3], double x[3]) {
  int piv[3] = {0, 1, 2};
  double a[3][3], r[3];
  double scale = 0.0;
  for (int i = 0; i < k; ++i) {
    r[i] = b[i];
    for (int j = 0; j < k; ++j) {
      a[i][j] = M[i][j];
      if (fabs(a[i][j]) > scale) scale = fabs(a[i][j]);
    }
  }
  (void)piv;
  for (int c = 0; c < k; ++c) {
    int p = c;
    for (int i = c + 1; i < k; ++i)
      if (fabs(a[i][c]) > fabs(a[p][c])) p = i;
    if (!(fabs(a[p][c]) > 1e-13 * (scale > 0 ? scale : 1.0))) return 0;
    if (p != c) {
      for (int j = 0; j < k; ++j) { double t = a[c][j]; a[c][j] = a[p][j]; a[p][j] = t; }
      double t = r[c]; r[c] = r[p]; r[p] = t;
    }
    for (int i = c + 1; i < k; ++i) {
      const double f = a[i][c] / a[c][c];
      for (int j = c; j < k; ++j) a[i][j] -= f * a[c][j];
      r[i] -= f * r[c];
    }
  }
  for (int i = k - 1; i >= 0; --i) {
    double s = r[i];
    for (int j = i + 1; j < k; ++j) s -= a[i][j] * x[j];
    x[i] = s / a[i][i];
  }
  return 1;
}

/* Returns ENUM_OK (delta_out, y_out = mu filled), ENUM_INFEASIBLE, or
 * ENUM_TOO_LARGE.  tol: relative KKT tolerance (1e-10 is plenty for
 * well-conditioned random instances). */
int orc_enum_project(int n, int m, const double* rho, const double* A, const double* ghat,
                     const uint8_t* is_eq, double lower, double upper, double tol,
                     double* delta_out, double* y_out) {
  if (n > 12 || m > 3 || n < 0 || m < 0) return ENUM_TOO_LARGE;
  int64_t npat = 1;
  for (int i = 0; i < n; ++i) npat *= 3;
  double best = INFINITY;
  double lo[12], hi[12], d[12], mu_full[3];
  double scale = 1.0;
  for (int i = 0; i < n; ++i) {
    lo[i] = lower - rho[i];
    hi[i] = upper - rho[i];
    scale = fmax(scale, fmax(fabs(lo[i]), fabs(hi[i])));
  }
  for (int j = 0; j < m; ++j) scale = fmax(scale, fabs(ghat[j]));
  const double eps = tol * scale;
  for (int cm = 0; cm < (1 << m); ++cm) {
    int J[3], k = 0, ok_mask = 1;
    for (int j = 0; j < m; ++j) {
      const int act = (cm >> j) & 1;
      if (is_eq && is_eq[j] && !act) { ok_mask = 0; break; }   /* equality rows always active */
      if (act) J[k++] = j;
    }
    if (!ok_mask) continue;
    for (int64_t p = 0; p < npat; ++p) {
      int st[12];
      int64_t q = p;
      for (int i = 0; i < n; ++i) { st[i] = (int)(q % 3); q /= 3; }   /* 0 free, 1 lower, 2 upper */
      double M[3][3] = {{0}}, b[3] = {0}, mu[3] = {0};
      for (int a = 0; a < k; ++a) {
        const double* ra = A + (int64_t)J[a] * n;
        b[a] = ghat[J[a]];
        for (int i = 0; i < n; ++i) {
          if (st[i] == 1) b[a] -= ra[i] * lo[i];
          else if (st[i] == 2) b[a] -= ra[i] * hi[i];
        }
        for (int c = 0; c < k; ++c) {
          const double* rc = A + (int64_t)J[c] * n;
          double s = 0.0;
          for (int i = 0; i < n; ++i)
            if (st[i] == 0) s += ra[i] * rc[i];
          M[a][c] = s;
        }
      }
      if (k > 0 && !solve_small(k, M, b, mu)) continue;
      /* candidate delta and KKT checks */
      int ok = 1;
      for (int i = 0; i < n && ok; ++i) {
        double z = 0.0;
        for (int a = 0; a < k; ++a) z += A[(int64_t)J[a] * n + i] * mu[a];
        if (st[i] == 0) {
          d[i] = z;
          ok = (z >= lo[i] - eps) && (z <= hi[i] + eps);
        } else if (st[i] == 1) {
          d[i] = lo[i];
          ok = z <= lo[i] + eps;     /* bound multiplier >= 0 */
        } else {
          d[i] = hi[i];
          ok = z >= hi[i] - eps;
        }
      }
      if (!ok) continue;
      for (int a = 0; a < k && ok; ++a)   /* inequality multipliers: y = mu <= 0 */
        if (!(is_eq && is_eq[J[a]])) ok = mu[a] <= eps;
      for (int j = 0; j < m && ok; ++j) {   /* every row satisfied */
        double s = 0.0;
        for (int i = 0; i < n; ++i) s += A[(int64_t)j * n + i] * d[i];
        if (is_eq && is_eq[j]) ok = fabs(s - ghat[j]) <= eps * 10;
        else ok = s <= ghat[j] + eps * 10;
      }
      if (!ok) continue;
      double nrm = 0.0;
      for (int i = 0; i < n; ++i) nrm += d[i] * d[i];
      if (nrm < best) {
        best = nrm;
        memcpy(delta_out, d, sizeof(double) * (size_t)n);
        for (int j = 0; j < m; ++j) mu_full[j] = 0.0;
        for (int a = 0; a < k; ++a) mu_full[J[a]] = mu[a];
        if (y_out) memcpy(y_out, mu_full, sizeof(double) * (size_t)m);
      }
    }
  }
  return isfinite(best) ? ENUM_OK : ENUM_INFEASIBLE;
}
