// topt_core.h — plan/controller state shared by the CUDA passes and the host.
//
// The PGD-TO step is a sequence of full-array PASSES (HBM/L2 sweeps that
// produce a handful of partial sums) separated by tiny scalar CONTROL steps
// (BB/PR+ scalars, the bisection walks, Stage-1 selection, the Newton m x m
// solve).  The controller below is plain C++ compiled for both the device
// (it runs inside the pass kernels, in the block that finishes last, so no
// host round trip sits between passes) and the host (C-ABI controller entry
// points used by the multi-rank tests).  Nothing here allocates.
//
// Reference map (file:line in /root/reference/proj):
//   Walk            <- binary_search_row            src/projection.cpp:48-110
//   stage-1 select  <- project_general_newton       src/projection.cpp:312-343
//   Newton          <- project_general_newton       src/projection.cpp:345-437
//   dispatch        <- project                      src/projection.cpp:440-460
//   step scalars    <- SPEC.md:287-313 (no reference code exists)
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define TOPT_HD __host__ __device__ __forceinline__
#define TOPT_HDN __host__ __device__
#define TOPT_NOINLINE __host__ __device__ __noinline__
#else
#define TOPT_HD inline
#define TOPT_HDN
#define TOPT_NOINLINE inline
#endif

namespace topt_b200 {

constexpr int MAX_M = 16;      // constraint rows
#ifndef TOPT_MAX_K
#define TOPT_MAX_K 16
#endif
constexpr int MAX_K = TOPT_MAX_K;   // bisection candidates per row per sweep
constexpr int MAX_CAND = 64;   // candidates per sweep over all rows
constexpr int MAX_FEAS = MAX_M + 1;
constexpr int PMAX = 512;      // partial-sum slots per pass

enum Phase : int32_t {
  PH_STEP_REDUCE = 0,  // K1: BB / PR+ dot products
  PH_PREP = 1,         // K2: direction + rho_tilde + linearization + r(0) + breakpoints
  PH_SWEEP = 2,        // K3: r_j(y) at up to MAX_CAND candidate duals
  PH_FEAS = 3,         // K4: stage-1 feasibility dots
  PH_NEWTON = 4,       // K5: delta(y), h-dots and A D A^T at one trial dual
  PH_FINAL = 5,        // K7: delta / x_new writes + residual dots
  PH_DONE = 6,
  PH_GATHER = 7,       // copy the (small) active sets to every CTA; later sweeps run CTA-locally
  PH_EXACT = 8         // strict parity: sums in the reference's sequential order (chains)
};

// Strict-parity "chains": one reference-order sequential sum each
// (s = start; for i in the reference's element order: s = fl(s + term_i)).
// A chain pass evaluates up to MAX_EX of them over one element sequence.
constexpr int MAX_EX = 96;
enum ChainKind : int8_t {
  CH_RESID = 0,   // start -g_hat_j; term a_j clip(y a_j, lo, hi)         projection.cpp:30-36
  CH_DOTZ = 1,    // term a_k delta_i, delta = clip(z(cmd.y), lo, hi)     projection.cpp:287-288
  CH_GRAM = 2,    // term a_j a_k over free i of z(cmd.y)                 projection.cpp:368-376
  CH_FEAS = 3,    // term a_k clip(0 + y a_j, lo, hi) (row j < 0: y = 0)  projection.cpp:320-328
  CH_GHAT = 4,    // term gd_i a_j                                        projection.cpp:140-145
  CH_STEP = 5     // BB / PR+ sums of oracle.c (k = 0..4)
};
// What a chain pass's results feed.
enum ExWhat : int32_t {
  EXW_NONE = 0, EXW_STEP, EXW_GHAT, EXW_WALK, EXW_FEAS, EXW_NEWTON, EXW_FINAL, EXW_RESH
};
struct ExChain {
  int8_t kind, j, k, pad_;
  int32_t pad2_;
  double y;       // CH_RESID / CH_FEAS dual
  double start;   // initial value of the sum
};
constexpr int GATHER_CAP = 1024;   // max gathered active elements (all rows; = the trigger)
constexpr int GATHER_BLK = 128;    // per-CTA items a compacted sweep publishes (fused gather)
constexpr int GATHER_TRIGGER = 1024;   // go CTA-local at or below this many active items

enum Status : int32_t {
  ST_OK = 0,
  ST_PARAMETER = 1,     // topt::ParameterError
  ST_DOMAIN = 2,        // topt::DomainError
  ST_SINGULAR = 3,      // topt::SingularSystemError
  ST_INFEASIBLE = 4,    // topt::InfeasibleLinearization
  ST_NUMERICAL = 5,     // topt::NumericalError
  ST_UNSUPPORTED = 6,   // topt::UnsupportedProblem
  ST_CUDA = 7,
  ST_INTERNAL = 8
};

enum Path : int32_t { PATH_SINGLE = 0, PATH_INDEPENDENT = 1, PATH_NEWTON = 2 };
enum Which : int32_t { W_AUTO = 0, W_SINGLE = 1, W_INDEPENDENT = 2, W_NEWTON = 3 };
enum Job : int32_t {
  JOB_PROJECT = 0,    // project / project_* (rho_tilde + linearization given)
  JOB_PGD_STEP = 1,   // full optimizer step from (x, x_prev, g, g_prev, d_prev, A)
  JOB_BUILD = 2,      // ConstraintLinearization::build: g_hat (+ partition validation)
  JOB_DELTA = 3,      // delta_of_y
  JOB_RESIDUAL_H = 4, // constraint_residual_h
  JOB_DIRECTION = 5   // spectral_step_size + cg_direction + rho_tilde only
};
enum Stage : int32_t {
  SG_INIT = 0, SG_SINGLE, SG_INDEP, SG_STAGE1, SG_FEAS, SG_NEWTON, SG_FINAL, SG_DONE
};
enum WalkStatus : int32_t {
  WK_IDLE = 0, WK_NEED = 1, WK_DONE = 2, WK_INFEASIBLE = 3,
  WK_EXACT = 4   // strict parity: a decision needs the reference-order value at ex_y
};

struct ProjOptions {
  double c, tol_b, tol_n;
  int32_t newton_maxiter, binary_maxiter;
};

struct PgdSettings {
  double alpha_max, alpha_fallback, omega, eps_alpha, tol_n;
  int32_t t_warmup;
};

// One reference bisection (binary_search_row) replayed from evaluations.
struct Walk {
  int32_t status, eq, up, feas_done;
  int32_t iters, pad_, near_ties, n_direct;
  double ghat, E, r0, S0, bp_lo, bp_hi, count;
  double lo, hi, ym, y, residual, min_margin;
  int32_t hasL, hasH, hasA, hasB;
  double yL, yH;                    // certified: R(yL) < -E, R(yH) > E
  double ya, Ra, Sa, yb, Rb, Sb;    // nearest evaluated points with R<=0 / R>0
  double hy, hs;                    // root estimate from the PREP sketch (if hok)
  int32_t hok, pad2_;
  // strict parity: reference-order evaluations are certificates with E = 0;
  // r(yL0) == 0 exactly (so r <= 0 below it, not r < 0)
  int32_t hasL0, ex_state;          // ex_state: 1 exact r(ex_y) pending, 2 exact r(0) pending
  double yL0, ex_y, any_;
};

struct Newton {
  double y[MAX_M], step[MAX_M], h[MAX_M], phi[MAX_M];
  double gram[MAX_M * (MAX_M + 1) / 2];   // A D A^T at the accepted y (upper, packed)
  double ty[MAX_M];                        // trial dual
  double merit, merit0, phi_sq, prev_phi_sq, gamma;
  int32_t iters, curv_viol, have_prev, in_linesearch;
};

// The command the next pass executes (read by every CTA).
struct Cmd {
  int32_t phase;
  int32_t nslots;
  // PH_PREP
  int32_t compute_dir, use_dprev, compute_dot, validate_part;
  double beta, wa;
  // PH_SWEEP: candidates grouped by row
  int32_t ncand;
  int32_t row_start[MAX_M + 1];
  double cand_y[MAX_CAND];
  // PH_FEAS: distinct stage-1 candidate duals (row < 0 -> all-zero dual)
  int32_t nfeas;
  int32_t feas_row[MAX_FEAS];
  double feas_y[MAX_FEAS];
  // PH_NEWTON / PH_FINAL: dual vector
  double y[MAX_M];
  int32_t want_gram;
  int32_t resid_rows;            // PH_FINAL: accumulate a_j . delta for all rows
  int32_t write_delta, write_x, write_mask;
  // PH_SWEEP active-set compaction: every candidate of row j lies in the
  // walk interval [wlo_j, whi_j]; elements whose clip region is the same at
  // both ends are folded into per-CTA fixed sums and dropped from the list.
  int32_t pat_hint;              // PH_PREP: the two-sweep pattern PREP (Problem::pat_hint)
  int32_t feas_gram0;            // PH_FEAS: also return Newton's first evaluation (y = 0):
                                 // m h-dots and the packed free-set Gram after the nfeas * m dots
  int32_t compact, local;        // local: sweep runs on the gathered items in each CTA
  int32_t load_fused;            // the items were published by the last global sweep:
                                 // every CTA loads them before the first local sweep
  int32_t sample;                // > 0: a SKETCH sweep over every 2^sample-th step of each
                                 // thread's elements; its sums only steer the candidates
  double wlo[MAX_M], whi[MAX_M];
  // PH_EXACT (strict parity)
  int32_t ex_n;                  // chains
  int32_t ex_seq;                // -1: elements 0..n-1; j: row j's partition sequence
  int32_t ex_what;               // ExWhat
  int32_t ex_row;                // EXW_FINAL: first row of this batch
  ExChain ex[MAX_EX];
};

// Problem description (device pointers are filled by the host).
struct Problem {
  int64_t n;          // local element count (this rank's slab)
  int64_t n_global;   // global element count (error bounds)
  int32_t m;
  int32_t job, which, has_part, t;
  double lower, upper, violation;
  ProjOptions opt;
  PgdSettings set;
  // device arrays
  const double* x;
  const double* x_prev;
  const double* g;
  const double* g_prev;
  const double* d_prev;
  const double* grad;      // m x ld row-major
  int64_t ld;              // row stride of grad
  const double* gd_step;   // JOB_PROJECT / JOB_BUILD
  const int8_t* owner;     // partition owner map (-1 = none) or null
  double* rho;             // rho_tilde (read in PROJECT, written in PGD_STEP)
  double* d_out;           // new direction (PGD_STEP)
  double* delta_out;       // optional
  double* x_out;           // optional x_{t+1}
  uint8_t* mask_out;       // optional 0 free, 1 lower, 2 upper
  // host-provided scalars
  double G_minus_g[MAX_M];      // bounds_g - g_values (rounded as the reference does)
  double ghat_in[MAX_M];        // JOB_PROJECT: lin.g_hat
  double ghat_err_in[MAX_M];    // bound on |ghat_in - reference ghat| (0 if exact)
  double y_in[MAX_M];           // JOB_DELTA / JOB_RESIDUAL_H
  int32_t is_eq[MAX_M];
  double row_count[MAX_M];      // terms summed by the reference per row
  double ours_len;              // bound on our summation depth (error bound)
  int32_t compact_cap;          // per-warp active-list capacity (0: no compaction)
  int32_t pad0_;
  // Host-buffer streaming (persistent kernel, host C-ABI entry only): the
  // inputs arrive in `nchunk` element chunks of `chunk` elements while the
  // kernel runs.  Chunk c of x, x_prev, g, g_prev is resident once
  // in_flags[c] has reached `epoch`, chunk c of d_prev and every grad row
  // once in_flags[nchunk + c] has.  The kernel sets *out_flag = epoch once d
  // is final (after PREP), so its device->host copy overlaps the bisection.
  const unsigned* in_flags;
  unsigned* out_flag;
  int64_t chunk;                // 0: inputs already resident
  uint32_t epoch;
  int32_t nchunk;
  // Partition whose every set is a contiguous ascending index range (e.g.
  // the channel-major material blocks of C3): set j = [row_lo[j], row_hi[j]).
  // The passes then visit each row's own range instead of all n elements.
  int32_t part_ranges;
  int32_t structured;           // some rows are generated (row_kind != RK_DENSE)
  int64_t row_lo[MAX_M], row_hi[MAX_M];
  // Structured constraint rows: a row is dense
  // (grad + k*ld), a constant (volume rows: a_i = row_c[k]) or a centroid
  // row a_i = sign * ((coord_axis(i) + 0.5) - center) / scale of an
  // x-fastest grid (grid.hpp:29-33), read from a per-launch shared-memory
  // table tab[row_tab[k] + coord] built with the same IEEE operations.
  int32_t row_kind[MAX_M];
  int32_t row_axis[MAX_M];
  int32_t row_tab[MAX_M];       // table offset (doubles) of a centroid row
  int32_t n_tab;                // table entries in all
  double row_c[MAX_M];          // constant value / center
  double row_scale[MAX_M];
  double row_sign[MAX_M];
  int64_t grid_n[3];            // nx, ny, nz
  int64_t idx_off;              // global index of local element 0 (slabs)
  int32_t axis_tab[3];          // the one table of each axis (-1: none / several)
  int32_t axis_fast;            // every centroid row uses its axis' one table,
  int32_t const_tab;            // ... and the constant rows share one value (entry)
  // strict parity (PH_EXACT): reference-order sums for every decision the
  // certificates cannot settle and for every Newton-stage sum
  int32_t strict;
  int32_t ex_nst;               // ring stages of the chain consumer (16 KB each)
  int32_t ex_smem;              // byte offset of the chain ring in dynamic shared memory
  int32_t ex_debug;             // print each chain pass's first results (TOPT_B200_EXDEBUG)
  int32_t ms_smem;              // byte offset of the fused-sweep area (0: none)
  int32_t pad4_;
  double* ex_buf;               // 2 x ex_seg x MAX_EX doubles (term staging)
  int64_t ex_seg;               // elements per staged segment
  const int32_t* part_idx;      // device partition indices (CSR; for subset chains)
  int64_t part_off[MAX_M + 1];  // host-copied CSR offsets
  // row structure found by PREP (controller-written; the passes after PREP
  // read each distinct row once): AK_CONST rows a_i = alias_c, AK_NEG rows
  // a_i = -a_{k-1,i}; pat7: the volume + 3 paired centre-of-mass layout
  int8_t alias_kind[MAX_M];
  int32_t n_alias, pat7;
  double alias_c[MAX_M];
  // root sketch (controller.h: consume_sketch): problems with at least this
  // many elements run sampled sweeps before the first full sweep (0: never)
  int64_t sketch_min_n;
  // the previous step on these same buffers found pat7: PREP reads the rows
  // in two sweeps and only VERIFIES rows 2, 4, 6 against -row 1, 3, 5 (their
  // sums follow by exact sign flips); a failed verification re-runs the
  // general PREP
  int32_t pat_hint;
  int32_t first_k;   // > 0: candidates per row in a walk's first full sweep (after the sketch)
};
enum RowKind { RK_DENSE = 0, RK_CONST = 1, RK_CENTROID = 2 };
// Row structure detected in the data by PREP (dense rows, single rank).
enum AliasKind { AK_DENSE = 0, AK_CONST = 1, AK_NEG = 2 };
constexpr int MAX_TAB = 8192;   // centroid table entries (shared memory, 64 KB)

// Controller-visible result.
struct Result {
  int32_t status, path, newton_iters, converged, curvature_violations;
  int32_t passes, sweeps, stage1_row, near_ties, fallback;
  int32_t local_sweeps, gathered;
  int32_t pat7, pad_res_;             // PREP found the volume + 3 paired rows layout (Problem::pat7)
  int32_t final_phase, exact_passes;  // cmd.phase when the persistent kernel returned;
                                      // chain passes (strict parity)
  double active;            // active elements after the last compacted sweep
  int32_t bisect_iters[MAX_M];
  double residual, alpha, beta, min_margin;
  double y[MAX_M], slacks[MAX_M], ghat[MAX_M], ghat_err[MAX_M], h[MAX_M];
  double step_sums[6];
};

// Controller scratch (kept in the Plan so device threads carry no big stack).
constexpr int CAND_CAP = 64;
struct Scratch {
  double np[CAND_CAP], nlo[CAND_CAP], nhi[CAND_CAP], nym[CAND_CAP];
  double jh[MAX_M * MAX_M], jp[MAX_M * MAX_M];
};

struct Plan {
  Problem P;
  Cmd cmd;
  int32_t stage;
  int32_t dot_mode;    // 1: ghat computed in-pass (errors include dot bound)
  Walk w[MAX_M];
  Newton nt;
  Result res;
  int32_t feas_map[MAX_M];
  // root sketch from the PREP pass (candidate choice only, never a decision)
  double hint_y[MAX_M], hint_sig[MAX_M];
  int32_t hint_ok[MAX_M];
  int32_t sketch_left, pad_sk_;       // sampled sweeps still to run before the full ones
  double sk_T[MAX_M];                 // PREP's sum |a_i| max(|lo_i|, |hi_i|) (sampling-noise scale)
  // strict parity
  int32_t ghat_ex_ok;                 // g_hat dots below are reference-order exact
  int32_t nglobal;                    // grid-synchronized passes so far (partials buffer parity)
  double ghat_dot_ex[MAX_M];
  double prep_save[MAX_M * 12];       // PREP totals held across the g_hat chain pass
  double step_save[6];
  Scratch sc;
};

}  // namespace topt_b200
