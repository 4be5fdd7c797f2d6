// optimizer_test.cpp — the C++ drop-in's optimizer entry points
// (include/topt/optimizer.hpp: spectral_step_size, cg_direction, pgd_step),
// which the reference specifies but does not ship.  Prints
// every result as exact hex floats; tests/test_dropin_cpp.py regenerates the
// same inputs (the same xorshift64*) and compares with the CPU oracle.
#include <cinttypes>
#include <cstdio>
#include <cstring>
#include <vector>

#include "topt/optimizer.hpp"

static uint64_t s = 0x2545F4914F6CDD1Dull;
static double urand() {
  s ^= s >> 12; s ^= s << 25; s ^= s >> 27;
  return (double)((s * 2685821657736338717ull) >> 11) * (1.0 / 9007199254740992.0);
}

static void hexv(const char* tag, const std::vector<double>& v) {
  uint64_t h = 1469598103934665603ull;
  for (double x : v) { uint64_t b; std::memcpy(&b, &x, 8); h = (h ^ b) * 1099511628211ull; }
  std::printf("%s %016" PRIx64 "\n", tag, h);
}

int main() {
  const std::size_t n = 6000, m = 2;
  topt::OptimizerState st;
  st.rho.resize(n); st.rho_prev.resize(n); st.grad.resize(n); st.grad_prev.resize(n);
  for (std::size_t i = 0; i < n; ++i) {
    st.rho[i] = 0.05 + 0.9 * urand();
    st.rho_prev[i] = st.rho[i] + 0.02 * (urand() - 0.5);
    const double e = 0.2 + 3.0 * urand();
    st.grad[i] = -3.0 * st.rho[i] * st.rho[i] * e;
    st.grad_prev[i] = -3.0 * st.rho_prev[i] * st.rho_prev[i] * e;
  }
  st.direction_prev = st.grad_prev;
  st.iteration = 1;
  topt::PgdSettings set;
  std::printf("alpha %a\n", topt::spectral_step_size(st, set));
  hexv("direction", topt::cg_direction(st));
  topt::ConstraintBundle cons;
  cons.m = m;
  cons.grad.assign(m * n, 1.0);
  double sx = 0.0;
  for (std::size_t i = 0; i < n; ++i) {
    sx += st.rho[i];
    cons.grad[n + i] = ((double)(i % 60) + 0.5 - 30.0) / (double)n;
  }
  cons.values = {sx, 0.0};
  cons.bounds = {0.45 * (double)n, 0.01};
  const topt::StepRecord rec = topt::pgd_step(st, cons, 0.0, 1.0, set);
  std::printf("step alpha %a beta %a fallback %d path %s iters %d\n", rec.alpha, rec.beta,
              (int)rec.fallback, topt::to_string(rec.projection.path), rec.projection.newton_iters);
  std::printf("y %a %a\n", rec.projection.y[0], rec.projection.y[1]);
  hexv("x_new", st.rho);
  hexv("d", st.direction_prev);
  return 0;
}
