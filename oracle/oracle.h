/* oracle.h — TEST INFRASTRUCTURE ONLY (see oracle.c header). */
#ifndef TOPT_ORACLE_H
#define TOPT_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  ORC_OK = 0,
  ORC_PARAMETER = 1,
  ORC_DOMAIN = 2,
  ORC_SINGULAR = 3,
  ORC_INFEASIBLE = 4,
  ORC_NUMERICAL = 5,
  ORC_UNSUPPORTED = 6
};
enum { ORC_PATH_SINGLE = 0, ORC_PATH_INDEPENDENT = 1, ORC_PATH_NEWTON = 2 };
#define ORC_MAX_TRACE_ROWS 64

typedef struct {
  double c, tol_b, tol_n;
  int newton_maxiter, binary_maxiter;
} orc_opts;

typedef struct {
  int path, newton_iters, converged, curvature_violations, stage1_row;
  double residual;
  int bisect_iters[ORC_MAX_TRACE_ROWS];
  double* iter_trace; /* optional: accepted Armijo gamma per Newton iteration */
} orc_meta;

typedef struct {
  double alpha_max, alpha_fallback, omega, eps_alpha, tol_n;
  int t_warmup;
} orc_pgd_settings;

typedef struct {
  double alpha, beta;
  int fallback;
} orc_step_info;

void orc_trace_set(double* buf, int64_t cap);
int64_t orc_trace_len(void);

int orc_binary_search_row(const double* a, const double* rho, int64_t n, const int32_t* sub,
                          int64_t nsub, double lower, double upper, double ghat, int equality,
                          double tol_b, int maxiter, int row, double* y_out,
                          double* residual_out, int* iters_out);
void orc_build_ghat(int64_t n, int64_t m, const double* grad, const double* g_values,
                    const double* bounds_g, const double* gd_step, double* ghat);
int orc_validate(int64_t n, int64_t m, const double* grad, const double* g_values,
                 const double* bounds_g, const double* gd_step, const double* ghat,
                 const int64_t* off, const int32_t* idx);
void orc_delta_of_y(int64_t n, int64_t m, const double* y, const double* grad,
                    const double* rho, double lower, double upper, double* z);
int orc_residual_h(int64_t n, int64_t m, const double* y, const double* grad,
                   const double* ghat, const double* rho, double lower, double upper,
                   double c, double* h);
int orc_fullpiv_solve(int64_t m, double* a, const double* b, double* x);
int orc_project_newton(int64_t n, int64_t m, const double* rho, const double* grad,
                       const double* ghat, const uint8_t* is_eq, double lower, double upper,
                       const orc_opts* o, double* delta, double* y, double* slacks,
                       orc_meta* meta);
int orc_project_single(int64_t n, int64_t m, const double* rho, const double* grad,
                       const double* ghat, const uint8_t* is_eq, double lower, double upper,
                       double tol_b, int maxiter, double* delta, double* y, double* slacks,
                       orc_meta* meta);
int orc_project_independent(int64_t n, int64_t m, const double* rho, const double* grad,
                            const double* g_values, const double* bounds_g,
                            const double* gd_step, const double* ghat, const uint8_t* is_eq,
                            const int64_t* off, const int32_t* idx, double lower, double upper,
                            double tol_b, int maxiter, double* delta, double* y, double* slacks,
                            orc_meta* meta);
int orc_project(int64_t n, int64_t m, const double* rho, const double* grad,
                const double* g_values, const double* bounds_g, const double* gd_step,
                const double* ghat, const uint8_t* is_eq, const int64_t* off,
                const int32_t* idx, double lower, double upper, const orc_opts* o,
                double* delta, double* y, double* slacks, orc_meta* meta);

double orc_spectral_step_size(int64_t n, const double* x, const double* x_prev,
                              const double* g, const double* g_prev, double alpha_max,
                              double eps_alpha);
double orc_spectral_from_sums(double ss, double sy, double yy, double alpha_max,
                              double eps_alpha);
double orc_pr_beta(int64_t n, const double* g, const double* g_prev);
double orc_pr_beta_from_sums(double num, double den);
void orc_step_direction(int64_t n, const double* x, const double* x_prev, const double* g,
                        const double* g_prev, const double* d_prev, int t, double violation,
                        const orc_pgd_settings* s, double* d, double* gd_step,
                        double* rho_tilde, orc_step_info* st);

#ifdef __cplusplus
}
#endif
#endif
