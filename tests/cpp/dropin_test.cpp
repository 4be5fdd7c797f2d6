// dropin_test.cpp — source-compatibility + parity check of the C++ drop-in.
// The SAME source is compiled twice by tests/cpp/Makefile:
//   dropin_ours : -I include/            linked against libtopt_b200.so (GPU)
//   dropin_ref  : -I reference headers   linked against oracle/_ref/libtopt_ref.so
//                 (the reference's own projection.cpp, CPU)
// and tests/test_dropin_cpp.py checks both print identical results.
#include <cinttypes>
#include <cstdio>
#include <cstring>
#include <vector>

#include "topt/errors.hpp"
#include "topt/projection.hpp"

static uint64_t s = 0x9E3779B97F4A7C15ull;
static double urand() {  // xorshift64*, deterministic
  s ^= s >> 12; s ^= s << 25; s ^= s >> 27;
  return (double)((s * 2685821657736338717ull) >> 11) * (1.0 / 9007199254740992.0);
}

static void print(const char* tag, const topt::ProjectionResult& r) {
  uint64_t hy = 0, hd = 0;
  for (double v : r.y) { uint64_t b; std::memcpy(&b, &v, 8); hy = hy * 1000003u ^ b; }
  for (double v : r.delta) { double w = v + 0.0; uint64_t b; std::memcpy(&b, &w, 8); hd = hd * 1000003u ^ b; }
  double dsum = 0.0;
  for (double v : r.delta) dsum += v;
  std::printf("%s path=%s iters=%d conv=%d yhash=%016" PRIx64 " dhash=%016" PRIx64
              " dsum=%.17g y=", tag, topt::to_string(r.path), r.newton_iters, (int)r.converged,
              hy, hd, dsum);
  for (double v : r.y) std::printf("%.17g,", v);
  std::printf("\n");
}

int main() {
  // SPEC.md:201 halfspace example
  auto lin = topt::ConstraintLinearization::build(1, 2, {0.5, 0.5}, {0.7}, {0.5}, {0.0, 0.0});
  std::vector<double> rho = {0.8, 0.6};
  print("halfspace", topt::project_single_binary_search(rho, lin, 0.0, 1.0, 1e-8));
  // random single dense row (C2-like) and a coupled m = 3 problem
  const std::size_t n = 4096;
  std::vector<double> a(n), r(n), gd(n, 0.0);
  double cl = 0.0;
  for (std::size_t i = 0; i < n; ++i) {
    const double x = 0.05 + 0.9 * urand(), e = 0.2 + 3.0 * urand();
    a[i] = -3.0 * x * x * e;
    r[i] = x - 0.5 * urand();
    cl += -a[i] * x;
  }
  auto lin1 = topt::ConstraintLinearization::build(1, n, a, {cl}, {0.8 * cl}, gd);
  print("dense_row", topt::project(r, lin1, 0.0, 1.0));
  std::vector<double> A(3 * n);
  for (std::size_t i = 0; i < n; ++i) {
    A[i] = 1.0;
    A[n + i] = ((double)(i % 64) + 0.5 - 32.0) / n;
    A[2 * n + i] = -A[n + i];
  }
  double sx = 0.0;
  for (double v : r) sx += v;
  auto lin3 = topt::ConstraintLinearization::build(3, n, A, {sx, 0.0, 0.0},
                                                   {0.35 * n, -0.02, 0.01}, gd);
  print("coupled3", topt::project(r, lin3, 0.0, 1.0));
  // errors map to the reference's exception types
  try {
    topt::project_single_binary_search(r, lin3, 0.0, 1.0, 1e-8);
    std::printf("no-throw\n");
  } catch (const topt::DomainError&) {
    std::printf("DomainError\n");
  }
  try {
    topt::constraint_residual_h(std::vector<double>{0.0}, lin1, r, 0.0, 1.0, 0.0);
    std::printf("no-throw\n");
  } catch (const topt::ParameterError&) {
    std::printf("ParameterError\n");
  }
  auto d = topt::delta_of_y(std::vector<double>{-0.6}, lin, rho, 0.0, 1.0);
  std::printf("delta_of_y %.17g %.17g\n", d[0], d[1]);
  return 0;
}
