/* TEST INFRASTRUCTURE ONLY — CPU restatements of the producers upstream of
 * the optimizer step, each following the
 * reference function it cites line by line, sequential, no FMA:
 *   orc_filter_csr        build_filter                  filter.cpp:10-43
 *   orc_filter_apply      apply_filter / filter_chain_rule  filter.cpp:45-69
 *   orc_interpolate       interpolate_stiffness         material.cpp:19-46
 *   orc_element_q4        element_stiffness_q4          fea.cpp:20-58
 *   orc_energy_gradient   element energies + gradient   fea.cpp:162-181
 * filter.cpp and material.cpp also compile in place (oracle/_ref); fea.cpp
 * needs Eigen's sparse module (absent), so its two loops are restated here
 * only.  Used by tests/ only.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* build_filter: CSR of the row-normalized hat kernel on an nx x ny grid.
 * Returns nnz; row_ptr / col / weight may be NULL (count only). */
int64_t orc_filter_csr(int nx, int ny, double radius, int32_t* row_ptr, int32_t* col,
                       double* weight) {
  if (!(radius > 0.0)) return -1;                                 /* filter.cpp:11 */
  int reach = (int)ceil(radius) - 1;                              /* filter.cpp:20 */
  if (reach < 0) reach = 0;
  int64_t k = 0;
  if (row_ptr) row_ptr[0] = 0;
  for (int ey = 0; ey < ny; ++ey)
    for (int ex = 0; ex < nx; ++ex) {
      const int64_t begin = k;
      double total = 0.0;
      for (int dy = -reach; dy <= reach; ++dy) {
        const int iy = ey + dy;
        if (iy < 0 || iy >= ny) continue;
        for (int dx = -reach; dx <= reach; ++dx) {
          const int ix = ex + dx;
          if (ix < 0 || ix >= nx) continue;
          const double w = radius - hypot((double)dx, (double)dy);   /* filter.cpp:33 */
          if (w <= 0.0) continue;
          if (col) { col[k] = iy * nx + ix; weight[k] = w; }
          total += w;
          ++k;
        }
      }
      if (weight)
        for (int64_t i = begin; i < k; ++i) weight[i] /= total;     /* filter.cpp:38-39 */
      if (row_ptr) row_ptr[(int64_t)ey * nx + ex + 1] = (int32_t)k;
    }
  return k;
}

/* transpose = 0: out = W raw (filter.cpp:45-56); 1: out = W^T g (:58-69). */
int orc_filter_apply(int nx, int ny, double radius, int transpose, const double* in, double* out) {
  const int64_t n = (int64_t)nx * ny;
  const int64_t nnz = orc_filter_csr(nx, ny, radius, NULL, NULL, NULL);
  if (nnz < 0) return 1;
  int32_t* rp = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
  int32_t* col = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nnz ? nnz : 1));
  double* w = (double*)malloc(sizeof(double) * (size_t)(nnz ? nnz : 1));
  orc_filter_csr(nx, ny, radius, rp, col, w);
  if (!transpose) {
    for (int64_t e = 0; e < n; ++e) {
      double acc = 0.0;
      for (int32_t i = rp[e]; i < rp[e + 1]; ++i) acc += w[i] * in[col[i]];
      out[e] = acc;
    }
  } else {
    for (int64_t e = 0; e < n; ++e) out[e] = 0.0;
    for (int64_t e = 0; e < n; ++e) {
      const double g = in[e];
      for (int32_t i = rp[e]; i < rp[e + 1]; ++i) out[col[i]] += w[i] * g;
    }
  }
  free(rp); free(col); free(w);
  return 0;
}

/* interpolate_stiffness (material.cpp:19-46): densities N*K channel-major. */
int orc_interpolate(int64_t n, int k, const double* young, double e_min, double penalty,
                    const double* dens, double* moduli, double* der) {
  for (int64_t i = 0; i < n * k; ++i)                              /* material.cpp:25-29 */
    if (!(dens[i] >= -1e-12 && dens[i] <= 1.0 + 1e-12)) return 2;
  for (int64_t e = 0; e < n; ++e) moduli[e] = e_min;
  const double p = penalty;
  for (int j = 0; j < k; ++j) {
    const double scale = young[j] - e_min;
    for (int64_t e = 0; e < n; ++e) {
      double r = dens[(int64_t)j * n + e];
      r = r > 0.0 ? r : 0.0;                                       /* std::max(0.0, r) */
      r = r < 1.0 ? r : 1.0;                                       /* std::min(1.0, .) */
      moduli[e] += pow(r, p) * scale;
      der[(int64_t)j * n + e] = p * pow(r, p - 1.0) * scale;
    }
  }
  return 0;
}

/* element_stiffness_q4 (fea.cpp:20-58), row-major 8 x 8. */
int orc_element_q4(double poisson, double h, double* ke) {
  static const double xin[4] = {-1.0, 1.0, 1.0, -1.0}, etan[4] = {-1.0, -1.0, 1.0, 1.0};
  if (!(poisson > 0.0 && poisson < 0.5) || !(h > 0.0)) return 1;
  const double nu = poisson;
  const double d11 = 1.0 / (1.0 - nu * nu), d12 = nu * d11, d33 = 0.5 * (1.0 - nu) * d11;
  for (int i = 0; i < 64; ++i) ke[i] = 0.0;
  const double gp = 1.0 / sqrt(3.0);
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b) {
      const double xi = a == 0 ? -gp : gp, eta = b == 0 ? -gp : gp;
      double dndx[4], dndy[4];
      for (int q = 0; q < 4; ++q) {
        dndx[q] = 0.25 * xin[q] * (1.0 + eta * etan[q]) * (2.0 / h);
        dndy[q] = 0.25 * etan[q] * (1.0 + xi * xin[q]) * (2.0 / h);
      }
      const double w = h * h / 4.0;
      for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) {
          ke[(2 * i) * 8 + 2 * j] += w * (d11 * dndx[i] * dndx[j] + d33 * dndy[i] * dndy[j]);
          ke[(2 * i) * 8 + 2 * j + 1] += w * (d12 * dndx[i] * dndy[j] + d33 * dndy[i] * dndx[j]);
          ke[(2 * i + 1) * 8 + 2 * j] += w * (d12 * dndy[i] * dndx[j] + d33 * dndx[i] * dndy[j]);
          ke[(2 * i + 1) * 8 + 2 * j + 1] +=
              w * (d11 * dndy[i] * dndy[j] + d33 * dndx[i] * dndx[j]);
        }
    }
  return 0;
}

/* Element energies u_e^T k0 u_e and gradient -der * energy (fea.cpp:162-181),
 * dofs of element e per grid.cpp:15-24. */
int orc_energy_gradient(int nx, int ny, double h, double poisson, const double* u, int k,
                        const double* der, double* energy, double* grad) {
  double ke[64];
  if (orc_element_q4(poisson, h, ke)) return 1;
  const int64_t n = (int64_t)nx * ny;
  for (int64_t e = 0; e < n; ++e) {
    const int ex = (int)(e % nx), ey = (int)(e / nx);
    const int64_t n1 = (int64_t)ey * (nx + 1) + ex, n2 = n1 + 1;
    const int64_t n3 = (int64_t)(ey + 1) * (nx + 1) + ex + 1, n4 = n3 - 1;
    const int64_t dofs[8] = {2 * n1, 2 * n1 + 1, 2 * n2, 2 * n2 + 1,
                             2 * n3, 2 * n3 + 1, 2 * n4, 2 * n4 + 1};
    double ue[8];
    for (int i = 0; i < 8; ++i) ue[i] = u[dofs[i]];
    double acc = 0.0;
    for (int i = 0; i < 8; ++i) {
      double row = 0.0;
      for (int j = 0; j < 8; ++j) row += ke[i * 8 + j] * ue[j];
      acc += ue[i] * row;
    }
    energy[e] = acc;
  }
  for (int j = 0; j < k; ++j)
    for (int64_t e = 0; e < n; ++e) grad[(int64_t)j * n + e] = -der[(int64_t)j * n + e] * energy[e];
  return 0;
}
