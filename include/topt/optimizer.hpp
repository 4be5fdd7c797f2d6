// topt/optimizer.hpp — the optimizer-step interface.  The reference lists
// src/optimizer.cpp (proj/CMakeLists.txt:21) but ships neither it nor a
// header; these declarations follow its spec (OptimizerState,
// PgdSettings, spectral_step_size, cg_direction, pgd_step) with the problem
// evaluators replaced by an explicit constraint bundle (the FE solve and the
// filter are outside this library).
#ifndef TOPT_B200_DROPIN_OPTIMIZER_HPP
#define TOPT_B200_DROPIN_OPTIMIZER_HPP

#include <cstdint>
#include <optional>
#include <vector>

#include "topt/projection.hpp"

namespace topt {

struct OptimizerState {
  std::vector<double> rho, rho_prev, grad, grad_prev, direction_prev;
  double alpha = 0.0;
  int iteration = 0;
  std::vector<double> last_violation;
};

struct PgdSettings {
  double alpha_max = 1e2;
  double alpha_fallback = 0.2;
  int t_warmup = 50;
  double omega = 1.0;
  double eps_alpha = 1e-6;
  double tol = 0.0;
  int K_max = 300;
  double C = 1e12;
  double tol_B = 1e-8;
  double tol_N = 1e-6;
};

// Constraint values/gradients at rho_t (what the problem evaluators return).
struct ConstraintBundle {
  std::size_t m = 0;
  std::vector<double> values, bounds, grad;  // grad: m x N row-major
  std::vector<std::uint8_t> is_equality;
  std::optional<std::vector<std::vector<int>>> partition;
};

struct StepRecord {
  double alpha = 0.0, beta = 0.0;
  bool fallback = false;
  std::vector<double> g_hat;
  ProjectionResult projection;
};

double spectral_step_size(const OptimizerState& state, const PgdSettings& settings);
std::vector<double> cg_direction(const OptimizerState& state);
// One PGD-TO step (Alg. 3 lines 2-15).  Updates state in place: rho_prev <- rho,
// rho <- rho_tilde + delta, direction_prev <- d, grad_prev <- grad,
// iteration += 1, alpha <- the step used.  The caller refreshes state.grad.
StepRecord pgd_step(OptimizerState& state, const ConstraintBundle& constraints, double lower,
                    double upper, const PgdSettings& settings);

}  // namespace topt

#endif
