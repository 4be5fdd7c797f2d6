// dropin.cpp — the reference's C++ projection / optimizer API (namespace topt)
// implemented on top of the C-ABI.  Status codes become the reference's
// exception types (errors.hpp); every computation runs on the GPU.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>

#include "topt/errors.hpp"
#include "topt/optimizer.hpp"
#include "topt/projection.hpp"
#include "topt_b200.h"

namespace topt {
namespace {

topt_b200_ctx* ctx() {
  static std::once_flag once;
  static topt_b200_ctx* c = nullptr;
  std::call_once(once, [] {
    int dev = 0;
    if (const char* e = std::getenv("TOPT_B200_DEVICE")) dev = std::atoi(e);
    if (topt_b200_ctx_create(dev, &c) != TOPT_OK) c = nullptr;
  });
  if (!c) throw std::runtime_error("topt_b200: no CUDA device (the library has no CPU path)");
  return c;
}

// One process-wide context holds mutable per-call state (plan, staging,
// streams, last error), so calls through it are serialized: the reference's
// functions are safe to call concurrently, and so are these.
std::mutex& ctx_mutex() {
  static std::mutex mu;
  return mu;
}
std::unique_lock<std::mutex> lock_ctx() { return std::unique_lock<std::mutex>(ctx_mutex()); }

[[noreturn]] void raise(int rc, const char* where) {
  std::string msg = std::string(where) + ": " + topt_b200_last_error(ctx());
  switch (rc) {
    case TOPT_ERR_PARAMETER: throw ParameterError(msg);
    case TOPT_ERR_DOMAIN: throw DomainError(msg);
    case TOPT_ERR_SINGULAR: throw SingularSystemError(msg);
    case TOPT_ERR_INFEASIBLE: throw InfeasibleLinearization(msg);
    case TOPT_ERR_NUMERICAL: throw NumericalError(msg);
    case TOPT_ERR_UNSUPPORTED: throw UnsupportedProblem(msg);
    default: throw std::runtime_error(msg);
  }
}

struct CsrPartition {
  std::vector<int64_t> off;
  std::vector<int32_t> idx;
};

CsrPartition to_csr(const std::optional<std::vector<std::vector<int>>>& p, std::size_t m) {
  CsrPartition c;
  if (!p) return c;
  if (p->size() != m) throw DomainError("ConstraintLinearization: partition size != m");
  c.off.assign(m + 1, 0);
  for (std::size_t j = 0; j < m; ++j) c.off[j + 1] = c.off[j] + (int64_t)(*p)[j].size();
  c.idx.reserve((std::size_t)c.off[m]);
  for (const auto& s : *p) c.idx.insert(c.idx.end(), s.begin(), s.end());
  return c;
}

topt_linearization view(const ConstraintLinearization& lin, const CsrPartition& part,
                        bool with_gd) {
  topt_linearization v;
  std::memset(&v, 0, sizeof(v));
  v.num_constraints = lin.num_constraints;
  v.num_vars = lin.num_vars;
  v.grad = lin.grad.data();
  v.g_values = lin.g_values.data();
  v.bounds_g = lin.bounds_g.data();
  v.gd_step = with_gd && !lin.gd_step.empty() ? lin.gd_step.data() : nullptr;
  v.g_hat = lin.g_hat.data();
  v.g_hat_err = lin.g_hat_err.size() == lin.num_constraints ? lin.g_hat_err.data() : nullptr;
  v.is_equality = lin.is_equality.empty() ? nullptr : lin.is_equality.data();
  v.part_offsets = part.off.empty() ? nullptr : part.off.data();
  v.part_indices = part.idx.empty() ? nullptr : part.idx.data();
  return v;
}

void check_rho(const ConstraintLinearization& lin, std::span<const double> rho) {
  if (rho.size() != lin.num_vars)
    throw DomainError("projection: rho_tilde size does not match linearization");
}

ProjectionResult run_project(int which, std::span<const double> rho,
                             const ConstraintLinearization& lin, double lower, double upper,
                             const ProjectionOptions& o) {
  const auto lk = lock_ctx();
  check_rho(lin, rho);
  const CsrPartition part = to_csr(lin.partition, lin.num_constraints);
  const topt_linearization v = view(lin, part, true);
  topt_proj_options co{o.c, o.tol_b, o.tol_n, o.newton_maxiter, o.binary_maxiter};
  ProjectionResult r;
  r.delta.resize(lin.num_vars);
  r.y.resize(lin.num_constraints);
  r.slacks.resize(lin.num_constraints);
  topt_proj_meta meta;
  const int rc = topt_b200_project(ctx(), which, rho.data(), &v, lower, upper, &co,
                                   r.delta.data(), r.y.data(), r.slacks.data(), &meta);
  if (rc != TOPT_OK) raise(rc, "project");
  r.path = static_cast<ProjectionPath>(meta.path);
  r.newton_iters = meta.newton_iters;
  r.residual = meta.residual;
  r.converged = meta.converged != 0;
  r.curvature_violations = meta.curvature_violations;
  return r;
}

}  // namespace

ConstraintLinearization ConstraintLinearization::build(
    std::size_t m, std::size_t n, std::vector<double> grad, std::vector<double> g_values,
    std::vector<double> bounds_g, std::vector<double> gd_step,
    std::vector<std::uint8_t> is_equality,
    std::optional<std::vector<std::vector<int>>> partition) {
  const auto lk = lock_ctx();
  ConstraintLinearization lin;
  lin.num_constraints = m;
  lin.num_vars = n;
  lin.grad = std::move(grad);
  lin.g_values = std::move(g_values);
  lin.bounds_g = std::move(bounds_g);
  lin.gd_step = std::move(gd_step);
  lin.is_equality = is_equality.empty() ? std::vector<std::uint8_t>(m, 0) : std::move(is_equality);
  lin.partition = std::move(partition);
  if (lin.grad.size() != m * n || lin.g_values.size() != m || lin.bounds_g.size() != m ||
      lin.gd_step.size() != n || lin.is_equality.size() != m)
    throw DomainError("ConstraintLinearization: inconsistent dimensions");
  lin.g_hat.assign(m, 0.0);
  lin.g_hat_err.assign(m, 0.0);
  const CsrPartition part = to_csr(lin.partition, m);
  const topt_linearization v = view(lin, part, true);
  const int rc = topt_b200_build(ctx(), &v, lin.g_hat.data(), lin.g_hat_err.data());
  if (rc != TOPT_OK) raise(rc, "ConstraintLinearization::build");
  return lin;
}

void ConstraintLinearization::validate() const {
  const ConstraintLinearization fresh =
      build(num_constraints, num_vars, grad, g_values, bounds_g, gd_step, is_equality, partition);
  for (std::size_t j = 0; j < num_constraints; ++j) {
    const double expect = fresh.g_hat[j];
    const double scale = std::max({1.0, std::abs(expect), std::abs(g_hat[j])});
    if (std::abs(g_hat[j] - expect) > 1e-14 * scale + fresh.g_hat_err[j])
      throw DomainError("ConstraintLinearization: g_hat inconsistent with fields");
  }
}

const char* to_string(ProjectionPath path) {
  switch (path) {
    case ProjectionPath::single_binary: return "single_binary";
    case ProjectionPath::independent_binary: return "independent_binary";
    case ProjectionPath::newton: return "newton";
  }
  return "unknown";
}

std::vector<double> delta_of_y(std::span<const double> y, const ConstraintLinearization& lin,
                               std::span<const double> rho_tilde, double lower, double upper) {
  const auto lk = lock_ctx();
  check_rho(lin, rho_tilde);
  if (y.size() != lin.num_constraints)
    throw DomainError("delta_of_y: dual size does not match linearization");
  const CsrPartition none;
  const topt_linearization v = view(lin, none, false);
  std::vector<double> out(lin.num_vars);
  const int rc = topt_b200_delta_of_y(ctx(), y.data(), &v, rho_tilde.data(), lower, upper,
                                      out.data());
  if (rc != TOPT_OK) raise(rc, "delta_of_y");
  return out;
}

std::vector<double> constraint_residual_h(std::span<const double> y,
                                          const ConstraintLinearization& lin,
                                          std::span<const double> rho_tilde, double lower,
                                          double upper, double c) {
  const auto lk = lock_ctx();
  if (!(c > 0.0)) throw ParameterError("constraint_residual_h: c must be > 0");
  check_rho(lin, rho_tilde);
  const CsrPartition none;
  const topt_linearization v = view(lin, none, false);
  std::vector<double> h(lin.num_constraints);
  const int rc = topt_b200_constraint_residual_h(ctx(), y.data(), &v, rho_tilde.data(), lower,
                                                 upper, c, h.data());
  if (rc != TOPT_OK) raise(rc, "constraint_residual_h");
  return h;
}

ProjectionResult project_single_binary_search(std::span<const double> rho_tilde,
                                              const ConstraintLinearization& lin,
                                              double lower, double upper, double tol_b,
                                              int binary_maxiter) {
  ProjectionOptions o;
  o.tol_b = tol_b;
  o.binary_maxiter = binary_maxiter;
  return run_project(TOPT_PROJECT_SINGLE, rho_tilde, lin, lower, upper, o);
}

ProjectionResult project_independent(std::span<const double> rho_tilde,
                                     const ConstraintLinearization& lin, double lower,
                                     double upper, double tol_b, int binary_maxiter) {
  ProjectionOptions o;
  o.tol_b = tol_b;
  o.binary_maxiter = binary_maxiter;
  if (!lin.partition) throw DomainError("project_independent: linearization has no partition");
  return run_project(TOPT_PROJECT_INDEPENDENT, rho_tilde, lin, lower, upper, o);
}

ProjectionResult project_general_newton(std::span<const double> rho_tilde,
                                        const ConstraintLinearization& lin, double lower,
                                        double upper, const ProjectionOptions& options) {
  return run_project(TOPT_PROJECT_NEWTON, rho_tilde, lin, lower, upper, options);
}

ProjectionResult project(std::span<const double> rho_tilde, const ConstraintLinearization& lin,
                         double lower, double upper, const ProjectionOptions& options) {
  return run_project(TOPT_PROJECT_AUTO, rho_tilde, lin, lower, upper, options);
}

// ---- optimizer -------------------------------------------
namespace {
topt_pgd_settings to_c(const PgdSettings& s) {
  return topt_pgd_settings{s.alpha_max, s.alpha_fallback, s.omega, s.eps_alpha, s.tol_N,
                           s.t_warmup};
}
}  // namespace

double spectral_step_size(const OptimizerState& st, const PgdSettings& s) {
  const auto lk = lock_ctx();
  const std::size_t n = st.rho.size();
  std::vector<double> d(n), rt(n);
  double alpha = 0.0, beta = 0.0;
  int32_t fb = 0;
  const topt_pgd_settings cs = to_c(s);
  // t = 1, no violation: the spectral branch (Eq. 13) is taken.
  const int rc = topt_b200_step_direction(ctx(), (int64_t)n, st.rho.data(), st.rho_prev.data(),
                                          st.grad.data(), st.grad_prev.data(),
                                          st.direction_prev.empty() ? st.grad_prev.data()
                                                                    : st.direction_prev.data(),
                                          1, 0.0, &cs, d.data(), rt.data(), &alpha, &beta, &fb);
  if (rc != TOPT_OK) raise(rc, "spectral_step_size");
  return alpha;
}

std::vector<double> cg_direction(const OptimizerState& st) {
  const auto lk = lock_ctx();
  if (st.iteration == 0 || st.grad_prev.empty()) return st.grad;   // d_0 = grad f_0
  const std::size_t n = st.rho.size();
  std::vector<double> d(n), rt(n);
  double alpha = 0.0, beta = 0.0;
  int32_t fb = 0;
  const topt_pgd_settings cs = to_c(PgdSettings{});
  const int rc = topt_b200_step_direction(ctx(), (int64_t)n, st.rho.data(), st.rho_prev.data(),
                                          st.grad.data(), st.grad_prev.data(),
                                          st.direction_prev.data(), 1, 0.0, &cs, d.data(),
                                          rt.data(), &alpha, &beta, &fb);
  if (rc != TOPT_OK) raise(rc, "cg_direction");
  return d;
}

StepRecord pgd_step(OptimizerState& st, const ConstraintBundle& cons, double lower, double upper,
                    const PgdSettings& s) {
  const auto lk = lock_ctx();
  const std::size_t n = st.rho.size(), m = cons.m;
  if (cons.grad.size() != m * n || cons.values.size() != m || cons.bounds.size() != m)
    throw DomainError("pgd_step: inconsistent constraint bundle");
  const bool first = st.iteration == 0 || st.rho_prev.empty();
  const std::vector<double>& xp = first ? st.rho : st.rho_prev;
  const std::vector<double>& gp = first ? st.grad : st.grad_prev;
  const std::vector<double>& dp = st.direction_prev.empty() ? gp : st.direction_prev;
  double viol = 0.0;
  for (double v : st.last_violation) viol = std::max(viol, v);
  const CsrPartition part = to_csr(cons.partition, m);
  topt_step_problem pr;
  std::memset(&pr, 0, sizeof(pr));
  pr.n = (int64_t)n; pr.m = (int32_t)m; pr.t = st.iteration; pr.violation = viol;
  pr.lower = lower; pr.upper = upper;
  pr.x = st.rho.data(); pr.x_prev = xp.data(); pr.g = st.grad.data(); pr.g_prev = gp.data();
  pr.d_prev = dp.data(); pr.grad = cons.grad.data();
  pr.g_values = cons.values.data(); pr.bounds_g = cons.bounds.data();
  pr.is_equality = cons.is_equality.empty() ? nullptr : cons.is_equality.data();
  pr.part_offsets = part.off.empty() ? nullptr : part.off.data();
  pr.part_indices = part.idx.empty() ? nullptr : part.idx.data();
  StepRecord rec;
  std::vector<double> x_new(n), d(n), rt(n), delta(n);
  rec.projection.y.resize(m);
  rec.projection.slacks.resize(m);
  rec.g_hat.resize(m);
  topt_step_outputs out;
  std::memset(&out, 0, sizeof(out));
  out.x_new = x_new.data(); out.d = d.data(); out.rho_tilde = rt.data(); out.delta = delta.data();
  out.y = rec.projection.y.data(); out.slacks = rec.projection.slacks.data();
  out.g_hat = rec.g_hat.data();
  const topt_pgd_settings cs = to_c(s);
  topt_proj_options co{s.C, s.tol_B, s.tol_N, 50, 200};
  topt_proj_meta meta;
  const int rc = topt_b200_pgd_step(ctx(), &pr, &cs, &co, &out, &meta);
  if (rc != TOPT_OK) raise(rc, "pgd_step");
  rec.alpha = meta.alpha;
  rec.beta = meta.beta;
  rec.fallback = meta.fallback != 0;
  rec.projection.delta = std::move(delta);
  rec.projection.path = static_cast<ProjectionPath>(meta.path);
  rec.projection.newton_iters = meta.newton_iters;
  rec.projection.residual = meta.residual;
  rec.projection.converged = meta.converged != 0;
  rec.projection.curvature_violations = meta.curvature_violations;
  st.rho_prev = st.rho;
  st.rho = std::move(x_new);
  st.grad_prev = st.grad;
  st.direction_prev = std::move(d);
  st.alpha = meta.alpha;
  st.iteration += 1;
  return rec;
}

}  // namespace topt
