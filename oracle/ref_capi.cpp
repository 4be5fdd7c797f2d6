// TEST INFRASTRUCTURE ONLY — C wrapper around the UNMODIFIED reference
// projection code (/root/reference/proj/src/projection.cpp), compiled in place
// by oracle/Makefile into oracle/_ref/libtopt_ref.so.  Used by tests/ (as the
// checker), by bench.py's cpu_baseline / --impl reference arm, and by
// tests/golden/make_golden.py.  Never linked into the product.
//
// Every entry point mirrors one reference function:
//   ref_build_ghat        -> ConstraintLinearization::build   (projection.cpp:119-148)
//   ref_validate          -> ConstraintLinearization::validate (projection.cpp:150-181)
//   ref_delta_of_y        -> delta_of_y                        (projection.cpp:192-209)
//   ref_residual_h        -> constraint_residual_h             (projection.cpp:253-267)
//   ref_filter_csr        -> build_filter                      (filter.cpp:10-43)
//   ref_filter_apply      -> apply_filter / filter_chain_rule  (filter.cpp:45-69)
//   ref_interpolate       -> interpolate_stiffness             (material.cpp:19-46)
//   ref_project           -> project / project_single_binary_search /
//                            project_independent / project_general_newton
//                                                               (projection.cpp:211-460)
// Error codes follow include/topt_b200.h (TOPT_ERR_*), one per errors.hpp type.
#include <cstdint>
#include <cstring>
#include <exception>
#include <optional>
#include <span>
#include <string>
#include <vector>

#include "topt/errors.hpp"
#include "topt/filter.hpp"
#include "topt/grid.hpp"
#include "topt/material.hpp"
#include "topt/projection.hpp"

namespace {

void put_err(char* err, std::size_t len, const char* msg) {
  if (!err || len == 0) return;
  std::strncpy(err, msg, len - 1);
  err[len - 1] = '\0';
}

template <class F>
int guarded(char* err, std::size_t len, F&& f) {
  try {
    f();
    return 0;
  } catch (const topt::ParameterError& e) {
    put_err(err, len, e.what());
    return 1;
  } catch (const topt::DomainError& e) {
    put_err(err, len, e.what());
    return 2;
  } catch (const topt::SingularSystemError& e) {
    put_err(err, len, e.what());
    return 3;
  } catch (const topt::InfeasibleLinearization& e) {
    put_err(err, len, e.what());
    return 4;
  } catch (const topt::NumericalError& e) {
    put_err(err, len, e.what());
    return 5;
  } catch (const topt::UnsupportedProblem& e) {
    put_err(err, len, e.what());
    return 6;
  } catch (const std::exception& e) {
    put_err(err, len, e.what());
    return 99;
  }
}

std::optional<std::vector<std::vector<int>>> make_partition(std::size_t m,
                                                            const int64_t* off,
                                                            const int32_t* idx) {
  if (!off) return std::nullopt;
  std::vector<std::vector<int>> p(m);
  for (std::size_t j = 0; j < m; ++j)
    p[j].assign(idx + off[j], idx + off[j + 1]);
  return p;
}

topt::ConstraintLinearization make_lin(std::size_t n, std::size_t m, const double* grad,
                                       const double* g_values, const double* bounds_g,
                                       const double* gd_step, const uint8_t* is_eq,
                                       const int64_t* off, const int32_t* idx) {
  return topt::ConstraintLinearization::build(
      m, n, std::vector<double>(grad, grad + m * n),
      std::vector<double>(g_values, g_values + m),
      std::vector<double>(bounds_g, bounds_g + m),
      std::vector<double>(gd_step, gd_step + n),
      is_eq ? std::vector<std::uint8_t>(is_eq, is_eq + m) : std::vector<std::uint8_t>{},
      make_partition(m, off, idx));
}

}  // namespace

extern "C" {

int ref_build_ghat(std::size_t n, std::size_t m, const double* grad, const double* g_values,
                   const double* bounds_g, const double* gd_step, const uint8_t* is_eq,
                   const int64_t* part_off, const int32_t* part_idx, double* ghat_out,
                   char* err, std::size_t errlen) {
  return guarded(err, errlen, [&] {
    auto lin = make_lin(n, m, grad, g_values, bounds_g, gd_step, is_eq, part_off, part_idx);
    for (std::size_t j = 0; j < m; ++j) ghat_out[j] = lin.g_hat[j];
  });
}

// Calls validate() on a linearization whose g_hat was overwritten by the
// caller (exercises the 1e-14 consistency check, projection.cpp:151-159).
int ref_validate(std::size_t n, std::size_t m, const double* grad, const double* g_values,
                 const double* bounds_g, const double* gd_step, const double* ghat_override,
                 const int64_t* part_off, const int32_t* part_idx, char* err,
                 std::size_t errlen) {
  return guarded(err, errlen, [&] {
    auto lin = make_lin(n, m, grad, g_values, bounds_g, gd_step, nullptr, nullptr, nullptr);
    lin.partition = make_partition(m, part_off, part_idx);
    if (ghat_override)
      for (std::size_t j = 0; j < m; ++j) lin.g_hat[j] = ghat_override[j];
    lin.validate();
  });
}

int ref_delta_of_y(std::size_t n, std::size_t m, const double* y, const double* grad,
                   const double* rho, double lower, double upper, double* delta_out,
                   char* err, std::size_t errlen) {
  return guarded(err, errlen, [&] {
    std::vector<double> zeros_m(m, 0.0), zeros_n(n, 0.0);
    auto lin = make_lin(n, m, grad, zeros_m.data(), zeros_m.data(), zeros_n.data(), nullptr,
                        nullptr, nullptr);
    auto d = topt::delta_of_y(std::span<const double>(y, m), lin,
                              std::span<const double>(rho, n), lower, upper);
    std::memcpy(delta_out, d.data(), n * sizeof(double));
  });
}

int ref_residual_h(std::size_t n, std::size_t m, const double* y, const double* grad,
                   const double* g_values, const double* bounds_g, const double* gd_step,
                   const double* rho, double lower, double upper, double c, double* h_out,
                   char* err, std::size_t errlen) {
  return guarded(err, errlen, [&] {
    auto lin = make_lin(n, m, grad, g_values, bounds_g, gd_step, nullptr, nullptr, nullptr);
    auto h = topt::constraint_residual_h(std::span<const double>(y, m), lin,
                                         std::span<const double>(rho, n), lower, upper, c);
    std::memcpy(h_out, h.data(), m * sizeof(double));
  });
}

// which: 0 = project (dispatch), 1 = project_single_binary_search,
//        2 = project_independent, 3 = project_general_newton.
int ref_project(int which, std::size_t n, std::size_t m, const double* rho,
                const double* grad, const double* g_values, const double* bounds_g,
                const double* gd_step, const uint8_t* is_eq, const int64_t* part_off,
                const int32_t* part_idx, double lower, double upper, double c, double tol_b,
                double tol_n, int newton_maxiter, int binary_maxiter, double* delta_out,
                double* y_out, double* slacks_out, int32_t* meta_i /* path, newton_iters,
                converged, curvature_violations */, double* residual_out, double* ghat_out,
                char* err, std::size_t errlen) {
  return guarded(err, errlen, [&] {
    auto lin = make_lin(n, m, grad, g_values, bounds_g, gd_step, is_eq, part_off, part_idx);
    if (ghat_out)
      for (std::size_t j = 0; j < m; ++j) ghat_out[j] = lin.g_hat[j];
    topt::ProjectionOptions o;
    o.c = c;
    o.tol_b = tol_b;
    o.tol_n = tol_n;
    o.newton_maxiter = newton_maxiter;
    o.binary_maxiter = binary_maxiter;
    std::span<const double> r(rho, n);
    topt::ProjectionResult res;
    switch (which) {
      case 1: res = topt::project_single_binary_search(r, lin, lower, upper, tol_b, binary_maxiter); break;
      case 2: res = topt::project_independent(r, lin, lower, upper, tol_b, binary_maxiter); break;
      case 3: res = topt::project_general_newton(r, lin, lower, upper, o); break;
      default: res = topt::project(r, lin, lower, upper, o); break;
    }
    std::memcpy(delta_out, res.delta.data(), n * sizeof(double));
    std::memcpy(y_out, res.y.data(), m * sizeof(double));
    std::memcpy(slacks_out, res.slacks.data(), m * sizeof(double));
    meta_i[0] = static_cast<int32_t>(res.path);
    meta_i[1] = res.newton_iters;
    meta_i[2] = res.converged ? 1 : 0;
    meta_i[3] = res.curvature_violations;
    *residual_out = res.residual;
  });
}

// build_filter's CSR (filter.cpp:10-43).  nnz_io: in = capacity of col /
// weight (0: query only), out = nnz.
int ref_filter_csr(int nx, int ny, double radius, int32_t* row_ptr, int32_t* col, double* weight,
                   int64_t* nnz_io, char* err, std::size_t errlen) {
  return guarded(err, errlen, [&] {
    const topt::StructuredGrid grid(nx, ny);
    const topt::FilterKernel k = topt::build_filter(grid, radius);
    const int64_t cap = *nnz_io;
    *nnz_io = (int64_t)k.col.size();
    if (cap <= 0) return;
    for (std::size_t e = 0; e <= k.size; ++e) row_ptr[e] = k.row_ptr[e];
    for (std::size_t i = 0; i < k.col.size() && (int64_t)i < cap; ++i) {
      col[i] = k.col[i];
      weight[i] = k.weight[i];
    }
  });
}

// apply_filter (transpose = 0, filter.cpp:45-56) / filter_chain_rule
// (transpose = 1, filter.cpp:58-69) with the kernel build_filter makes.
int ref_filter_apply(int nx, int ny, double radius, int transpose, const double* in, double* out,
                     char* err, std::size_t errlen) {
  return guarded(err, errlen, [&] {
    const topt::StructuredGrid grid(nx, ny);
    const topt::FilterKernel k = topt::build_filter(grid, radius);
    const std::span<const double> v(in, k.size);
    const std::vector<double> r =
        transpose ? topt::filter_chain_rule(k, v) : topt::apply_filter(k, v);
    std::memcpy(out, r.data(), r.size() * sizeof(double));
  });
}

// interpolate_stiffness (material.cpp:19-46): moduli (N) and derivative (N*K).
int ref_interpolate(std::size_t n, std::size_t k, const double* young, double e_min,
                    double poisson, double penalty, const double* densities, double* moduli,
                    double* derivative, char* err, std::size_t errlen) {
  return guarded(err, errlen, [&] {
    topt::MaterialModel mm;
    mm.young_moduli.assign(young, young + k);
    mm.e_min = e_min;
    mm.poisson = poisson;
    mm.penalty = penalty;
    const auto r = topt::interpolate_stiffness(std::span<const double>(densities, n * k), n, mm);
    std::memcpy(moduli, r.moduli.data(), n * sizeof(double));
    std::memcpy(derivative, r.derivative.data(), n * k * sizeof(double));
  });
}

}  // extern "C"
