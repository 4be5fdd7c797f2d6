/*
 * topt_b200.h — C-ABI of the B200-native PGD-TO optimizer step.
 *
 * Plain C: POD structs, raw pointers and sizes, int status codes, no
 * exceptions and no torch types across the boundary.  Every entry point
 * replaces one reference interface (file:line in /root/reference/proj/ or the
 * reference's SPEC.md, where the optimizer module exists only as a spec):
 *
 *   topt_b200_build                 <- ConstraintLinearization::build
 *                                      include/topt/projection.hpp:30-35,
 *                                      src/projection.cpp:119-148 (+ validate :150-181)
 *   topt_b200_delta_of_y            <- delta_of_y        projection.hpp:67-70, projection.cpp:192-209
 *   topt_b200_constraint_residual_h <- constraint_residual_h
 *                                      projection.hpp:90-93, projection.cpp:253-267
 *   topt_b200_project (which=...)   <- project / project_single_binary_search /
 *                                      project_independent / project_general_newton
 *                                      projection.hpp:76-109, projection.cpp:211-460
 *   topt_b200_pgd_step              <- pgd_step (spectral_step_size + cg_direction +
 *                                      rho_tilde + project + rho_{t+1})
 *   *_dev variants                  the same calls on device-resident buffers
 *
 * Status codes map 1:1 onto the reference's exception taxonomy
 * (include/topt/errors.hpp:9-42).  A failed call leaves a message in
 * topt_b200_last_error().  Host-pointer calls copy through pinned staging;
 * *_dev calls take device pointers and never touch host memory except the
 * O(m) scalars named as such.
 */
#ifndef TOPT_B200_H
#define TOPT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  TOPT_OK = 0,
  TOPT_ERR_PARAMETER = 1,   /* topt::ParameterError          errors.hpp:11-14 */
  TOPT_ERR_DOMAIN = 2,      /* topt::DomainError             errors.hpp:16-20 */
  TOPT_ERR_SINGULAR = 3,    /* topt::SingularSystemError     errors.hpp:22-25 */
  TOPT_ERR_INFEASIBLE = 4,  /* topt::InfeasibleLinearization errors.hpp:27-32 */
  TOPT_ERR_NUMERICAL = 5,   /* topt::NumericalError          errors.hpp:34-38 */
  TOPT_ERR_UNSUPPORTED = 6, /* topt::UnsupportedProblem      errors.hpp:40-44 */
  TOPT_ERR_CUDA = 7,        /* CUDA runtime failure / no device */
  TOPT_ERR_INTERNAL = 8
};

/* ProjectionPath, projection.hpp:43 */
enum { TOPT_PATH_SINGLE_BINARY = 0, TOPT_PATH_INDEPENDENT_BINARY = 1, TOPT_PATH_NEWTON = 2 };

/* which solver entry point to mirror */
enum {
  TOPT_PROJECT_AUTO = 0,        /* topt::project                       projection.cpp:440 */
  TOPT_PROJECT_SINGLE = 1,      /* topt::project_single_binary_search  projection.cpp:211 */
  TOPT_PROJECT_INDEPENDENT = 2, /* topt::project_independent           projection.cpp:229 */
  TOPT_PROJECT_NEWTON = 3       /* topt::project_general_newton        projection.cpp:302 */
};

#define TOPT_B200_MAX_M 16

/* topt::ProjectionOptions, projection.hpp:58-64 (defaults: 1e12, 1e-8, 1e-6, 50, 200) */
typedef struct {
  double c;
  double tol_b;
  double tol_n;
  int32_t newton_maxiter;
  int32_t binary_maxiter;
} topt_proj_options;

/* PgdSettings, SPEC.md:282 (defaults: 1e2, 0.2, 1.0, 1e-6, 1e-6, 50) */
typedef struct {
  double alpha_max;
  double alpha_fallback;
  double omega;
  double eps_alpha;
  double tol_n;
  int32_t t_warmup;
} topt_pgd_settings;

/* topt::ProjectionResult scalars (projection.hpp:47-56) + diagnostics */
typedef struct {
  int32_t path;                  /* TOPT_PATH_* */
  int32_t newton_iters;
  int32_t converged;
  int32_t curvature_violations;
  double residual;
  /* diagnostics (not in the reference) */
  int32_t passes;                /* O(n) passes executed on the device */
  int32_t sweeps;                /* multi-candidate bisection sweeps */
  int32_t stage1_row;            /* row accepted by Newton stage 1, or -1 */
  int32_t near_ties;             /* directly-evaluated decisions with |r| <= bound */
  double min_margin;             /* min |r| / bound over direct decisions */
  int32_t bisect_iters[TOPT_B200_MAX_M];
  /* pgd_step only */
  double alpha;
  double beta;
  int32_t fallback;
  int32_t local_sweeps;          /* CTA-local sweeps on gathered active elements */
  int32_t gathered;              /* 1 if the active sets were gathered */
  int32_t exact_passes;          /* strict parity: reference-order chain passes run */
  double active;                 /* active elements after the last compacted sweep */
} topt_proj_meta;

/* topt::ConstraintLinearization, projection.hpp:17-41.  grad/gd_step are
 * host pointers for the host API and device pointers for *_dev; the O(m)
 * vectors and the partition are always host pointers. */
typedef struct {
  size_t num_constraints;          /* m */
  size_t num_vars;                 /* n */
  const double* grad;              /* m*n row-major */
  const double* g_values;          /* m */
  const double* bounds_g;          /* m */
  const double* gd_step;           /* n (may be NULL for project calls) */
  const double* g_hat;             /* m (project / delta / residual calls) */
  const double* g_hat_err;         /* m bound on |g_hat - sequential g_hat|, or NULL */
  const uint8_t* is_equality;      /* m, or NULL (all inequality) */
  const int64_t* part_offsets;     /* m+1 CSR offsets, or NULL (no partition) */
  const int32_t* part_indices;     /* partition indices (host) */
  const int8_t* owner;             /* *_dev only: device owner map from topt_b200_owner_map */
} topt_linearization;

/* One optimizer step's state (OptimizerState).  Device
 * pointers for topt_b200_pgd_step_dev, host pointers for topt_b200_pgd_step. */
typedef struct {
  int64_t n;
  int32_t m;
  int32_t t;                       /* iteration index */
  double violation;                /* ||max(g - G, 0)||_inf, fallback trigger */
  double lower, upper;
  const double* x;                 /* rho_t */
  const double* x_prev;            /* rho_{t-1} */
  const double* g;                 /* grad f(rho_t) */
  const double* g_prev;            /* grad f(rho_{t-1}) */
  const double* d_prev;            /* d_{t-1} */
  const double* grad;              /* m*n constraint gradients, row-major */
  const double* g_values;          /* host, m */
  const double* bounds_g;          /* host, m */
  const uint8_t* is_equality;      /* host, m or NULL */
  const int64_t* part_offsets;     /* host CSR partition or NULL */
  const int32_t* part_indices;
  const int8_t* owner;             /* *_dev: device owner map or NULL */
} topt_step_problem;

typedef struct {
  double* x_new;                   /* n: rho_{t+1} = rho_tilde + delta */
  double* d;                       /* n: new direction d_t */
  double* rho_tilde;               /* n: workspace/output (required for *_dev) */
  double* delta;                   /* n or NULL */
  double* y;                       /* host, m duals */
  double* slacks;                  /* host, m */
  double* g_hat;                   /* host, m or NULL */
  uint8_t* mask;                   /* n or NULL: 0 free, 1 lower, 2 upper */
} topt_step_outputs;

typedef struct topt_b200_ctx topt_b200_ctx;

const char* topt_b200_version(void);
int topt_b200_ctx_create(int device, topt_b200_ctx** out);
void topt_b200_ctx_destroy(topt_b200_ctx* ctx);
const char* topt_b200_last_error(const topt_b200_ctx* ctx);
/* Number of device kernels launched by this context so far (bench evidence). */
int64_t topt_b200_kernel_launches(const topt_b200_ctx* ctx);
/* CUDA stream used by the context (cudaStream_t as void*); may be replaced. */
void* topt_b200_get_stream(const topt_b200_ctx* ctx);
int topt_b200_set_stream(topt_b200_ctx* ctx, void* stream);

/* Parity mode of the following calls on this context (default CERTIFIED;
 * environment TOPT_B200_PARITY=strict sets STRICT at context creation).
 *   CERTIFIED  every decision the reference takes on a floating-point sign
 *              (bisection midpoints, stage-1 feasibility, Armijo, the
 *              Newton stop test) is taken on our own tree-summed values; a
 *              bisection / stage-1 decision is PROVEN to equal the
 *              reference's unless our |value| lies within the bound on the
 *              reference's own rounding error (counted in meta.near_ties);
 *              Newton runs on accurately summed h and Gram (it stops at the
 *              true tolerance, where the reference's sequentially summed
 *              ||Phi|| may stall on its own rounding noise).
 *   STRICT     additionally evaluates every such undecided value, every
 *              Newton-stage sum, g_hat's dots, the BB / PR+ sums and the
 *              reported residuals in the reference's own sequential order
 *              (one chain pass: ~8 GPU cycles per element), so every output
 *              is bit-identical to the reference built without FMA
 *              (oracle/_ref).  Single GPU, dense rows, m <= 9.
 * A context is not thread-safe: serialize calls on one context (the C++
 * drop-in does); distinct contexts may run concurrently. */
enum { TOPT_PARITY_CERTIFIED = 0, TOPT_PARITY_STRICT = 1 };
int topt_b200_set_parity(topt_b200_ctx* ctx, int mode);
int topt_b200_get_parity(const topt_b200_ctx* ctx);

/* Structured constraint rows (extension beyond the reference interface;
 * SURVEY.md §8(f) rank 1).  Rows the caller can describe instead of storing:
 *   TOPT_ROW_DENSE     row k of prob->grad (as usual)
 *   TOPT_ROW_CONST     a_i = value                      (volume rows)
 *   TOPT_ROW_CENTROID  a_i = sign * ((c_axis(i) + 0.5) - center) / scale
 * where c_axis(i) is the integer coordinate of global element
 * i + index_offset on the x-fastest grid[0] x grid[1] x grid[2]
 * (grid.hpp:29-33; the centre-of-mass rows of SPEC.md:405).  The values are
 * bit-identical to the dense rows the same formulas produce, and the passes
 * then never read them from memory.  Applies to the following
 * topt_b200_pgd_step_dev / topt_b200_pgd_step_ranks calls on this context
 * (2 <= m <= 8, no partition, even n); rows = NULL clears it. */
enum { TOPT_ROW_DENSE = 0, TOPT_ROW_CONST = 1, TOPT_ROW_CENTROID = 2 };
typedef struct {
  int32_t kind;
  int32_t axis;                    /* CENTROID: 0 x, 1 y, 2 z */
  double value;                    /* CONST */
  double center, scale, sign;      /* CENTROID */
} topt_row_desc;
int topt_b200_set_structured_rows(topt_b200_ctx* ctx, int32_t m, const topt_row_desc* rows,
                                  const int64_t* grid, int64_t index_offset);

/* Per-launch device timing of the pass kernel (CUDA events on the launching
 * stream).  When enabled, every pass launch is bracketed by events; the
 * accumulated device time and launch count are returned (and reset). */
int topt_b200_set_profiling(topt_b200_ctx* ctx, int enabled);
int topt_b200_kernel_time(topt_b200_ctx* ctx, double* total_ms, int64_t* launches,
                          double* max_ms);
/* Whole-job device time under profiling: CUDA events on the context's stream
 * from the plan upload to the results download of each job (step, projection,
 * ...), accumulated and reset on read. */
int topt_b200_step_time(topt_b200_ctx* ctx, double* total_ms, int64_t* jobs, double* max_ms);

/* Debug: per-pass device timestamps of the next persistent launch. */
int topt_b200_debug_trace(topt_b200_ctx* ctx, int enable, unsigned long long* out);

void topt_b200_default_options(topt_proj_options* o);
void topt_b200_default_settings(topt_pgd_settings* s);

/* ConstraintLinearization::build: g_hat_j = (G_j - g_j) + gd_step . grad_j, and
 * validate() of the partition when one is given. */
int topt_b200_build(topt_b200_ctx* ctx, const topt_linearization* lin, double* g_hat_out,
                    double* g_hat_err_out);

int topt_b200_delta_of_y(topt_b200_ctx* ctx, const double* y, const topt_linearization* lin,
                         const double* rho_tilde, double lower, double upper,
                         double* delta_out);

int topt_b200_constraint_residual_h(topt_b200_ctx* ctx, const double* y,
                                    const topt_linearization* lin, const double* rho_tilde,
                                    double lower, double upper, double c, double* h_out);

/* project / project_*: host buffers (rho_tilde, grad, delta_out are n-sized). */
int topt_b200_project(topt_b200_ctx* ctx, int which, const double* rho_tilde,
                      const topt_linearization* lin, double lower, double upper,
                      const topt_proj_options* opts, double* delta_out, double* y_out,
                      double* slacks_out, topt_proj_meta* meta);

/* Same on device buffers (rho_tilde, lin->grad, lin->gd_step, lin->owner,
 * delta_out, mask_out are device pointers; y/slacks/meta are host). */
int topt_b200_project_dev(topt_b200_ctx* ctx, int which, const double* rho_tilde,
                          const topt_linearization* lin, double lower, double upper,
                          const topt_proj_options* opts, double* delta_out, uint8_t* mask_out,
                          double* y_out, double* slacks_out, topt_proj_meta* meta);

/* Device owner map (int8, -1 = in no block) from a host CSR partition; checks
 * index range and overlap like validate() (projection.cpp:163-171). */
int topt_b200_owner_map(topt_b200_ctx* ctx, int64_t n, int32_t m, const int64_t* part_offsets,
                        const int32_t* part_indices, int8_t* owner_dev);

/* Full optimizer step (BB + PR+ + rho_tilde + build + project + rho_{t+1}). */
int topt_b200_pgd_step(topt_b200_ctx* ctx, const topt_step_problem* prob,
                       const topt_pgd_settings* settings, const topt_proj_options* opts,
                       const topt_step_outputs* out, topt_proj_meta* meta);
int topt_b200_pgd_step_dev(topt_b200_ctx* ctx, const topt_step_problem* prob,
                           const topt_pgd_settings* settings, const topt_proj_options* opts,
                           const topt_step_outputs* out, topt_proj_meta* meta);

/* ---- multi-GPU: one process per GPU, element-slab sharding, NCCL ----------
 * Each rank passes its contiguous slab of every n-vector (device pointers,
 * prob->n = slab length); per pass the rank's partial sums are all-gathered
 * over NCCL and combined in rank order on every GPU, so all ranks take the
 * same decisions.  n_global / row_counts: global element / row counts. */
int topt_b200_nccl_unique_id(unsigned char* out, size_t len);   /* 128 bytes */
int topt_b200_ctx_create_ranks(int device, int rank, int world, const unsigned char* nccl_id,
                               topt_b200_ctx** out);
int topt_b200_pgd_step_ranks(topt_b200_ctx* ctx, const topt_step_problem* prob,
                             int64_t n_global, const int64_t* row_counts,
                             const topt_pgd_settings* settings, const topt_proj_options* opts,
                             const topt_step_outputs* out, topt_proj_meta* meta);

/* Single-process lockstep ranks: the same multi-rank data plane (per-rank
 * pass kernels over element slabs, rank-order combine, replicated control)
 * with the per-pass all-gather done as device-to-device copies instead of
 * NCCL -- for one process driving several slabs (or GPUs), and to test the
 * multi-rank code on one device.  Rank r's context comes from
 * topt_b200_ctx_create_lockstep(device, r, world); probs / outs / metas are
 * per-rank arrays (device pointers as for topt_b200_pgd_step_ranks). */
int topt_b200_ctx_create_lockstep(int device, int rank, int world, topt_b200_ctx** out);
int topt_b200_pgd_step_lockstep(int world, topt_b200_ctx* const* ctxs,
                                const topt_step_problem* probs, int64_t n_global,
                                const int64_t* row_counts, const topt_pgd_settings* settings,
                                const topt_proj_options* opts, const topt_step_outputs* outs,
                                topt_proj_meta* metas);

/* spectral_step_size + cg_direction + rho_tilde only, host
 * buffers.  d_out = new direction, rho_tilde_out = x - omega*alpha*d. */
int topt_b200_step_direction(topt_b200_ctx* ctx, int64_t n, const double* x,
                             const double* x_prev, const double* g, const double* g_prev,
                             const double* d_prev, int32_t t, double violation,
                             const topt_pgd_settings* settings, double* d_out,
                             double* rho_tilde_out, double* alpha_out, double* beta_out,
                             int32_t* fallback_out);

/* ---- upstream of the step ---------------------
 * Density filter: the row-normalized linear hat kernel of build_filter on an
 * nx x ny StructuredGrid (element e = ey nx + ex, unit element size;
 * filter.cpp:10-43), applied matrix-free on the GPU with the reference's
 * weights and summation orders: W x (apply_filter, filter.cpp:45-56) and
 * W^T g (filter_chain_rule, filter.cpp:58-69), bit-identical to the CSR code.
 * Status: radius <= 0 or nx, ny < 1 -> TOPT_ERR_PARAMETER (ParameterError). */
typedef struct topt_b200_filter topt_b200_filter;
int topt_b200_filter_create(topt_b200_ctx* ctx, int32_t nx, int32_t ny, double radius,
                            topt_b200_filter** out);
void topt_b200_filter_destroy(topt_b200_filter* f);
int64_t topt_b200_filter_nnz(const topt_b200_filter* f);
/* build_filter's CSR (row_ptr: n + 1, col / weight: nnz entries; host). */
int topt_b200_filter_csr(const topt_b200_filter* f, int32_t* row_ptr, int32_t* col,
                         double* weight);
/* transpose = 0: out = W in ; 1: out = W^T in.  n = nx ny doubles each. */
int topt_b200_filter_apply(topt_b200_ctx* ctx, const topt_b200_filter* f, int transpose,
                           const double* in, double* out);
int topt_b200_filter_apply_dev(topt_b200_ctx* ctx, const topt_b200_filter* f, int transpose,
                               const double* in_dev, double* out_dev);
/* Any CSR filter kernel (a topt::FilterKernel, host arrays): W x / W^T x in
 * the reference's orders. */
int topt_b200_csr_apply(topt_b200_ctx* ctx, int64_t n, const int32_t* row_ptr, const int32_t* col,
                        const double* weight, int transpose, const double* in, double* out);
/* SIMP interpolate_stiffness (material.cpp:19-46), device buffers (densities
 * N*K channel-major; young: K host values).  derivative may be NULL.
 * pow() is CUDA's (<= 2 ulp), every other operation the reference's. */
int topt_b200_interpolate_stiffness_dev(topt_b200_ctx* ctx, int64_t n, int32_t k,
                                        const double* young, double e_min, double poisson,
                                        double penalty, const double* dens_dev,
                                        double* moduli_dev, double* der_dev);
/* element_stiffness_q4 (fea.cpp:20-58): 64 values, row-major, host. */
int topt_b200_element_stiffness_q4(double poisson, double element_size, double* ke64);
/* Element energies u_e^T k0 u_e and the compliance gradient -dE * energy
 * (fea.cpp:162-181) from a displacement field u (2 (nx+1)(ny+1) dofs,
 * grid.cpp:15-24 numbering); device buffers, energy / grad may be NULL. */
int topt_b200_compliance_gradient_dev(topt_b200_ctx* ctx, int32_t nx, int32_t ny,
                                      double element_size, double poisson, const double* u_dev,
                                      int32_t kmat, const double* der_dev, double* energy_dev,
                                      double* grad_dev);

/* FE solve (assemble_and_solve, fea.cpp:60-144):
 * plane-stress Q4 elasticity on an nx x ny grid with element moduli E (device,
 * nx ny), fixed dofs and point loads (host lists, BoundaryConditions of
 * grid.hpp:36-41, validated as grid.cpp:26-38), solved matrix-free by Jacobi-
 * preconditioned CG to ||K u - f|| / ||f|| <= rel_tol in at most 10 N_free
 * iterations (the reference's Eigen ConjugateGradient settings).  u_dev: all
 * 2 (nx+1)(ny+1) dofs, fixed ones 0.  Status: bad BCs -> TOPT_ERR_PARAMETER,
 * no convergence -> TOPT_ERR_SINGULAR (SingularSystemError). */
int topt_b200_fe_solve_dev(topt_b200_ctx* ctx, int32_t nx, int32_t ny, double element_size,
                           double poisson, const double* moduli_dev, const int32_t* fixed_dofs,
                           int64_t n_fixed, const int32_t* load_dofs, const double* load_values,
                           int64_t n_loads, double rel_tol, double* u_dev, int64_t* iterations,
                           double* residual);

#ifdef __cplusplus
}
#endif
#endif
