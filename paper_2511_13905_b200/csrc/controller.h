// controller.h — the scalar control logic between passes (host + device).
//
// consume(plan, totals) takes the reduced partial sums of the pass described
// by plan.cmd and writes the next command.  Every decision that the
// reference takes on a floating-point sign (bisection `rm > 0.0`, stage-1
// `viol <= tol_n`, Armijo) is taken here, in the reference's order.
//
// Bisection parity (projection.cpp:96-109).  The reference walks dyadic
// midpoints ym = 0.5*(lo+hi) one O(n) pass at a time.  Here a sweep
// evaluates up to MAX_K midpoints of the walk's decision tree per row in ONE
// pass, and the walk is then replayed exactly:
//   * a midpoint that was evaluated is decided by the evaluated sign
//     (R^ > 0.0), exactly like the reference;
//   * a midpoint that was not evaluated is decided only when monotonicity of
//     r(y) (PAPER.md Eq. (Delta); each rounded term a*clip(fl(y a)) is itself
//     monotone) CERTIFIES the reference's own sign: an evaluated point
//     y_c <= ym with R^(y_c) > E forces r_ref(ym) > 0, and y_c >= ym with
//     R^(y_c) < -E forces r_ref(ym) <= 0.  E bounds the reference's
//     sequential-summation error, the g_hat discrepancy and our own
//     summation error (gamma_k bounds, Higham Thm 4.4).
// The walk therefore visits the reference's midpoints in the reference's
// order and returns the reference's final midpoint; it differs from the
// reference only if a DIRECTLY evaluated midpoint has |r| below the
// reference's own rounding noise (counted in Result::near_ties).
#pragma once
#include <math.h>
#include <string.h>

#include "topt_core.h"

namespace topt_b200 {

constexpr double kUnit = 1.1102230246251565e-16;  // 2^-53

// Optional device-side timeline marks (debug builds of the trace only).
#if defined(__CUDACC__)
__device__ unsigned long long* g_ctl_marks = nullptr;
// Debug progress words in mapped host memory (TOPT_B200_PROGRESS=1): a
// watchdog thread prints them while a launch is stuck.
__device__ unsigned long long* g_progress = nullptr;
__device__ __forceinline__ void progress_mark(int slot, unsigned long long v) {
  if (g_progress) {
    if (blockIdx.x == 0 && threadIdx.x == 0) g_progress[slot] = v;
    if (threadIdx.x == 0) atomicAdd_system(g_progress + 16 + slot, 1ull);
    __threadfence_system();
  }
}
#if defined(TOPT_CTL_MARK_SMEM)   // microbenchmark builds: clock64 into shared memory
__device__ __forceinline__ unsigned long long* ctl_marks_smem() {
  __shared__ unsigned long long m[16];
  return m;
}
#endif
__host__ __device__ __forceinline__ void ctl_mark(int k) {
#if defined(__CUDA_ARCH__) && defined(TOPT_CTL_MARK_SMEM)
  ctl_marks_smem()[k] = clock64();
#elif defined(__CUDA_ARCH__)
  if (g_ctl_marks && blockIdx.x == 0) {
    unsigned long long t;
#if defined(TOPT_CTL_MARK_CLOCK)
    t = clock64();
#else
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
#endif
    g_ctl_marks[k] = t;
  }
#else
  (void)k;
#endif
}
#else
inline void ctl_mark(int) {}
#endif
constexpr double kGradFloor = 1e-300;              // projection.cpp:19

TOPT_HD double gamma_k(double k) { return k * kUnit / (1.0 - k * kUnit); }
TOPT_HD double dmin_(double a, double b) { return (b < a) ? b : a; }  // std::min
TOPT_HD double dmax_(double a, double b) { return (a < b) ? b : a; }  // std::max

// Number of PREP slots per row and their meaning (kernels write these).
enum PrepSlot {
  PS_DOT = 0,      // sum gd_i a_i
  PS_DABS = 1,     // sum |gd_i a_i|
  PS_S0 = 2,       // sum a_i clip(0, lo_i, hi_i)
  PS_SLOPE0 = 3,   // sum over free-at-0 of a_i^2
  PS_T = 4,        // sum |a_i| max(|lo_i|, |hi_i|)      (bounds every |term|)
  PS_NZOUT = 5,    // count of a_ji != 0 outside the partition block
  PS_BPLO = 6,     // min breakpoint (min-reduced)
  PS_BPHI = 7,     // max breakpoint (max-reduced)
  PS_ANY = 8,      // count of |a_i| >= 1e-300
  // row-structure detection (single rank, dense rows; 1.0 = not examined):
  PS_NCONST = 9,   // count of a_i != a_0            (a constant row: volume)
  PS_AREF = 10,    // a_0 (one contributor)
  PS_NNEG = 11,    // count of a_i != -a_{j-1,i}      (the +- rows of a two-sided constraint)
  PREP_SLOTS = 12
};

static_assert(sizeof(((Plan*)0)->prep_save) == sizeof(double) * MAX_M * PREP_SLOTS,
              "prep_save holds one PREP pass");

// Reduction operator of a slot: 0 sum, 1 min, 2 max.
TOPT_HD int slot_op(int phase, int slot) {
  if (phase == PH_STEP_REDUCE) return slot == 5 ? 2 : 0;
  if (phase == PH_PREP) {
    const int s = slot % PREP_SLOTS;
    return s == PS_BPLO ? 1 : (s == PS_BPHI ? 2 : 0);
  }
  return 0;
}

// ---------------------------------------------------------------------------
// m x m full-pivot LU + solve (mirrors Eigen::FullPivLU as used at
// projection.cpp:401-407; same algorithm as oracle.c's orc_fullpiv_solve).
// a is column-major m x m and is destroyed.  Returns false if not invertible.
TOPT_NOINLINE bool fullpiv_solve(int m, double* a, const double* b, double* x) {
  int rowperm[MAX_M], colperm[MAX_M];
#define A_(i, j) a[(j) * m + (i)]
  for (int i = 0; i < m; ++i) rowperm[i] = colperm[i] = i;
  int nz = m;
  double maxpivot = 0.0;
  for (int k = 0; k < m; ++k) {
    double biggest = -1.0;
    int br = k, bc = k;
    for (int j = k; j < m; ++j)
      for (int i = k; i < m; ++i) {
        const double v = fabs(A_(i, j));
        if (v > biggest) { biggest = v; br = i; bc = j; }
      }
    if (biggest == 0.0) { nz = k; break; }
    if (biggest > maxpivot) maxpivot = biggest;
    if (br != k) {
      for (int j = 0; j < m; ++j) { const double t = A_(k, j); A_(k, j) = A_(br, j); A_(br, j) = t; }
      const int t = rowperm[k]; rowperm[k] = rowperm[br]; rowperm[br] = t;
    }
    if (bc != k) {
      for (int i = 0; i < m; ++i) { const double t = A_(i, k); A_(i, k) = A_(i, bc); A_(i, bc) = t; }
      const int t = colperm[k]; colperm[k] = colperm[bc]; colperm[bc] = t;
    }
    const double piv = A_(k, k);
    for (int i = k + 1; i < m; ++i) A_(i, k) = A_(i, k) / piv;
    for (int j = k + 1; j < m; ++j)
      for (int i = k + 1; i < m; ++i) A_(i, j) = A_(i, j) - A_(i, k) * A_(k, j);
  }
  const double thr = fabs(maxpivot) * 2.220446049250313e-16 * (double)m;
  int rank = 0;
  for (int i = 0; i < nz; ++i) rank += (fabs(A_(i, i)) > thr) ? 1 : 0;
  if (rank != m) return false;
  double c[MAX_M];
  for (int i = 0; i < m; ++i) c[i] = b[rowperm[i]];
  for (int i = 0; i < m; ++i) {
    double s = c[i];
    for (int k = 0; k < i; ++k) s = s - A_(i, k) * c[k];
    c[i] = s;
  }
  for (int i = nz - 1; i >= 0; --i) {
    double s = c[i];
    for (int k = i + 1; k < nz; ++k) s = s - A_(i, k) * c[k];
    c[i] = s / A_(i, i);
  }
  for (int i = 0; i < m; ++i) x[colperm[i]] = (i < nz) ? c[i] : 0.0;
#undef A_
  return true;
}

// ---------------------------------------------------------------------------
// Bisection walk

// This sweep's evaluations for one row: candidate duals cy[k] and the
// partial slots t2[2k] (sum of terms, not yet offset by -ghat), t2[2k+1] (slope).
struct Evals {
  const double* cy;
  const double* t2;
  int nc;
};

// Candidates are mostly consumed in generation order (the predicted path),
// so the search starts just after the previous hit.
TOPT_HD bool evals_lookup(const Evals& ev, double ghat, double y, double* R, int* hint) {
  const int nc = ev.nc;
  int k = *hint;
  for (int c = 0; c < nc; ++c) {
    if (k >= nc) k = 0;
    if (ev.cy[k] == y) { *R = ev.t2[2 * k] - ghat; *hint = k + 1; return true; }
    ++k;
  }
  return false;
}

// Fold this sweep's evaluations into the walk's knowledge (brackets).
TOPT_HD void walk_ingest(Walk& w, const Evals& ev) {
  for (int k = 0; k < ev.nc; ++k) {
    const double y = ev.cy[k], R = ev.t2[2 * k] - w.ghat, S = ev.t2[2 * k + 1];
    if (R <= 0.0 && (!w.hasA || y > w.ya)) { w.hasA = 1; w.ya = y; w.Ra = R; w.Sa = S; }
    if (R > 0.0 && (!w.hasB || y < w.yb)) { w.hasB = 1; w.yb = y; w.Rb = R; w.Sb = S; }
    if (R < -w.E && (!w.hasL || y > w.yL)) { w.hasL = 1; w.yL = y; }
    if (R > w.E && (!w.hasH || y < w.yH)) { w.hasH = 1; w.yH = y; }
  }
}

// Replay the reference walk as far as evaluations/certificates allow.
TOPT_HD void walk_advance(Walk& w, const ProjOptions& o, const Evals& ev, bool strict = false) {
  if (w.status == WK_DONE || w.status == WK_INFEASIBLE || w.status == WK_IDLE ||
      w.status == WK_EXACT)
    return;
  const bool hasL = w.hasL, hasH = w.hasH, hasL0 = w.hasL0;
  const double yL = w.yL, yH = w.yH, yL0 = w.yL0, E = w.E, ghat = w.ghat;
  int near = 0, direct = 0, hint = 0;
  double minm = w.min_margin;
  if (!w.feas_done) {
    // projection.cpp:80-94: r(y_lo) > 0 (down) / r(y_hi) < 0 (up) => infeasible.
    // Certificates first (proofs); a direct evaluation otherwise.
    const double yb = w.up ? w.bp_hi : w.bp_lo;
    double R;
    int infeasible;
    if (hasH && yH <= yb) {
      infeasible = w.up ? 0 : 1;
    } else if (hasL && yL >= yb) {
      infeasible = w.up ? 1 : 0;
    } else if (hasL0 && (w.up ? yL0 == yb : yL0 >= yb)) {
      infeasible = 0;   // r(yb) <= 0 (down), r(yb) == 0 (up)
    } else if (evals_lookup(ev, ghat, yb, &R, &hint)) {
      if (strict && fabs(R) <= E) {   // undecidable from our sum: reference-order value
        w.status = WK_EXACT; w.ex_state = 1; w.ex_y = yb;
        return;
      }
      infeasible = w.up ? (R < 0.0) : (R > 0.0);
      minm = dmin_(minm, fabs(R) / E);
      near += (fabs(R) <= E);
    } else {
      w.status = WK_NEED;
      return;
    }
    w.near_ties += near;
    w.min_margin = minm;
    near = 0;
    if (infeasible) { w.status = WK_INFEASIBLE; return; }
    w.feas_done = 1;
  }
  double lo = w.lo, hi = w.hi, ym = w.ym;
  int it = w.iters;
  const double tol_b = o.tol_b;
  const int maxit = o.binary_maxiter;
  int status = WK_DONE;
  while ((hi - lo) > tol_b && it < maxit) {
    int d;
    if (hasH && yH <= ym) {
      d = 1;
    } else if ((hasL && yL >= ym) || (hasL0 && yL0 >= ym)) {
      d = -1;
    } else {
      double R;
      if (!evals_lookup(ev, ghat, ym, &R, &hint)) { status = WK_NEED; break; }
      if (strict && fabs(R) <= E) { status = WK_EXACT; w.ex_state = 1; w.ex_y = ym; break; }
      minm = dmin_(minm, fabs(R) / E);
      near += (fabs(R) <= E);
      ++direct;
      d = R > 0.0 ? 1 : -1;
    }
    if (d > 0) hi = ym; else lo = ym;
    ym = 0.5 * (lo + hi);
    ++it;
  }
  w.lo = lo; w.hi = hi; w.ym = ym; w.iters = it;
  w.near_ties += near;
  w.n_direct += direct;
  w.min_margin = minm;
  w.status = status;
  if (status == WK_DONE) w.y = ym;
}

// Cheap, host/device-identical approximations used ONLY to rank speculative
// midpoints (erfc/log cost ~1000 dependent cycles each on one GPU thread).
TOPT_HD double approx_log2(double x) {
  uint64_t b;
  memcpy(&b, &x, sizeof(b));
  const int64_t e = (int64_t)((b >> 52) & 0x7ff) - 1023;
  const double m = (double)(b & 0xfffffffffffffull) * 2.220446049250313e-16;  // [0,1)
  return (double)e + m;
}
#if defined(__CUDA_ARCH__)
#define TOPT_FDIV(a, b) __fdividef((a), (b))
#else
#define TOPT_FDIV(a, b) ((a) / (b))
#endif
TOPT_HD double approx_ncdf_upper(double t) {  // ~ P(Z > t), monotone, in (0, 1)
  float u = (float)(2.5 * t);
  if (!(u == u)) u = 0.0f;
  if (u > 1e30f) u = 1e30f;
  if (u < -1e30f) u = -1e30f;
  return (double)(0.5f - 0.5f * TOPT_FDIV(u, 1.0f + fabsf(u)));
}

// Root estimate used to choose speculative midpoints (never a decision).
struct RootEst {
  int kind;        // 0: gaussian(ye, sig) ; 1: log-uniform prior below 0 ; 2: above 0
  double ye, sig, L, inv_sig;
  double sl, E;    // slope scale near the root (0 if unknown) and the walk's bound
  double thr;      // est_certain distance: max(6 sig, 16 E / sl)
};

// Division for estimates only (never a decision): reciprocal estimate + one
// Newton step on the device, IEEE on the host.
TOPT_HDN inline double est_div(double a, double b) {
#if defined(__CUDA_ARCH__)
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(b));
  r = __fma_rn(r, __fma_rn(-b, r, 1.0), r);
  return a * r;
#else
  return a / b;
#endif
}

TOPT_HD RootEst walk_estimate_(const Walk& w);
TOPT_NOINLINE RootEst walk_estimate(const Walk& w) {
  RootEst e = walk_estimate_(w);
  e.inv_sig = est_div(1.0, e.sig);
  e.thr = dmax_(6.0 * e.sig, (e.sl > 0.0) ? est_div(16.0 * e.E, e.sl) : 0.0);
  return e;
}
TOPT_HD RootEst walk_estimate_(const Walk& w) {
  RootEst e;
  e.kind = 0; e.ye = 0.0; e.sig = 1.0; e.L = 0.0; e.inv_sig = 1.0;
  e.sl = dmax_(w.hasA ? w.Sa : 0.0, w.hasB ? w.Sb : 0.0);
  e.E = w.E;
  // the PREP sketch, while it lies in the walk interval
  const bool hint = w.hok && w.hy >= w.lo && w.hy <= w.hi && w.hs > 0.0;
  if (w.hasA && w.hasB && w.ya < w.yb) {
    const double ya = w.ya, yb = w.yb;
    double sec = ya - est_div(w.Ra * (yb - ya), w.Rb - w.Ra);
    if (!(sec >= ya)) sec = ya;
    if (!(sec <= yb)) sec = yb;
    // Newton from the bracket end closer to the root (smaller |R|); its error
    // is ~ curvature * step^2 / (2 slope), the curvature taken from the two
    // end slopes.  Without a usable slope: the secant, its spread as sigma.
    const bool na = w.Sa > 0.0, nb = w.Sb > 0.0;
    const double Na = na ? dmin_(dmax_(ya - est_div(w.Ra, w.Sa), ya), yb) : sec;
    const double Nb = nb ? dmin_(dmax_(yb - est_div(w.Rb, w.Sb), ya), yb) : sec;
    double ye = sec, sig;
    if (na && nb) {
      const bool use_a = fabs(w.Ra) <= fabs(w.Rb);
      ye = use_a ? Na : Nb;
      const double S = use_a ? w.Sa : w.Sb, d = ye - (use_a ? ya : yb);
      const double curv = est_div(fabs(w.Sb - w.Sa), yb - ya);
      sig = 2.0 * curv * est_div(d * d, S);
      sig = dmax_(sig, 1e-3 * fabs(Na - Nb));
    } else if (na || nb) {   // one slope: Newton from that end, a quarter of
      ye = na ? Na : Nb;      // its distance to the secant as sigma
      sig = 0.25 * fabs(ye - sec);
    } else {
      sig = 0.5 * (yb - ya);
    }
    sig = dmax_(sig, (yb - ya) * 1e-6);
    sig = dmax_(sig, fabs(ye) * 1e-15);
    e.ye = ye;
    e.sig = dmax_(sig, 1e-300);
    if (hint && w.hy > ya && w.hy < yb && w.hs < e.sig) { e.ye = w.hy; e.sig = w.hs; }
    return e;
  }
  if (hint) { e.ye = w.hy; e.sig = w.hs; return e; }
  if (!w.up) {  // root in [bp_lo, 0], r(0) > 0 known
    if (w.hasB && w.Sb > 0.0) {
      e.ye = dmax_(w.yb - est_div(w.Rb, w.Sb), w.lo);
      e.sig = dmax_(0.5 * fabs(e.ye), 1e-300);
      return e;
    }
    e.kind = 1;
    e.L = approx_log2(fabs(w.lo) + 1e-300);
    return e;
  }
  if (w.hasA && w.Sa > 0.0) {  // root in [0, bp_hi], r(0) < 0 known
    e.ye = dmin_(w.ya - est_div(w.Ra, w.Sa), w.hi);
    e.sig = dmax_(0.5 * fabs(e.ye), 1e-300);
    return e;
  }
  e.kind = 2;
  e.L = approx_log2(fabs(w.hi) + 1e-300);
  return e;
}

TOPT_HDN inline bool est_certain(const RootEst& e, double y) {
  // 6 sigma away, and far enough that |r| there should clear the bound E
  return e.kind == 0 && fabs(y - e.ye) >= e.thr;
}

// Probability that the root lies above y.
TOPT_HDN inline double est_p_above(const RootEst& e, double y) {
  if (e.kind == 0) return approx_ncdf_upper((y - e.ye) * e.inv_sig);
  const double ay = fabs(y);
  if (!(ay > 0.0)) return e.kind == 1 ? 0.0 : 1.0;
  double p = (approx_log2(ay) - (e.L - 66.0)) * (1.0 / 66.0);  // P(|root| < |y|), log-uniform prior
  p = dmin_(dmax_(p, 0.0), 1.0);
  return e.kind == 1 ? p : 1.0 - p;
}

// The part of the walk interval where evaluations can still matter: midpoints
// outside the certified bounds (yL, yH) are decided without evaluation.  Every
// candidate of a sweep lies in this window, so it also bounds the compacted
// sweeps (elements of constant clip region over it are folded).
TOPT_HDN inline void walk_window(const Walk& w, double* clo, double* chi) {
  double a = w.lo, b = w.hi;
  if (w.feas_done) {   // before that, the infeasibility probe sits at an interval end
    if (w.hasL && w.yL > a) a = w.yL;
    if (w.hasL0 && w.yL0 > a) a = w.yL0;
    if (w.hasH && w.yH < b) b = w.yH;
  }
  *clo = a; *chi = b;
}

// A level whose midpoint lies more than kCertainSig standard deviations from
// a point estimate is predicted with near certainty (the ranking CDF above has
// heavy tails on purpose and is not used for this).
TOPT_HDN inline bool est_certain(const RootEst& e, double y);

// Choose up to K midpoints of the walk's remaining decision tree to evaluate
// next: the predicted path (most probable branch at every uncertain level),
// plus first-level alternatives ("hedges") at its least certain levels,
// ranked by the probability of being visited.  O(K + certain levels), all
// state in registers.
constexpr int MAX_HEDGE = 4;
constexpr int kMaxPathLevels = 64;               // uncertain + certain levels walked
// Predicted path (most probable branch at every uncertain level) plus the
// MAX_HEDGE most probable first-level alternatives, merged by probability of
// being visited.  Per-level work is a few register operations (the hedge
// set is kept in registers; only the path is written to local memory).
TOPT_HD int walk_candidates(const Walk& w, const ProjOptions& o, int K, double* out,
                            Scratch& scr) {
  (void)scr;
  int n = 0;
  if (w.status != WK_NEED || K <= 0) return 0;
  if (!w.feas_done) out[n++] = w.up ? w.bp_hi : w.bp_lo;
  ctl_mark(4);
  const RootEst e = walk_estimate(w);
  ctl_mark(5);
  double py[MAX_K], pp[MAX_K];
  double hy[MAX_HEDGE], hp[MAX_HEDGE];
#pragma unroll
  for (int k = 0; k < MAX_HEDGE; ++k) { hy[k] = 0.0; hp[k] = -1.0; }
  double hpmin = -1.0;      // smallest kept hedge probability
  int np = 0;
  double lo = w.lo, hi = w.hi, ym = w.ym, p = 1.0;
  int it = w.iters;
  const bool hasL = w.hasL, hasH = w.hasH;
  const double yL = w.yL, yH = w.yH;
  const int Kp = K - n;
  // levels whose branch is near-certain are not evaluated themselves: one
  // evaluation at the innermost of them per direction (cert_lo / cert_hi)
  // certifies the whole run by monotonicity.
  double cert_lo = 0.0, cert_hi = 0.0;
  bool has_cl = false, has_ch = false;
  int lev = 0;
  double clo, chi;
  walk_window(w, &clo, &chi);
  const int Kpath = Kp;
  while (np < Kpath && lev < kMaxPathLevels && (hi - lo) > o.tol_b && it < o.binary_maxiter) {
    if (hasH && yH <= ym) {
      hi = ym;
    } else if (hasL && yL >= ym) {
      lo = ym;
    } else {
      const double pa = est_p_above(e, ym);   // root above ym -> r(ym) <= 0 -> lo = ym
      bool right;   // p_above >= 0.5, as one comparison (as walk_candidates_warp)
      if (e.kind == 0) right = ym <= e.ye;
      else if (e.kind == 1) right = approx_log2(fabs(ym)) >= e.L - 33.0;
      else right = approx_log2(fabs(ym)) <= e.L - 33.0;
      ++lev;
      if (lev > 1 && est_certain(e, ym)) {   // the walk's next midpoint is always taken
        if (right) { cert_lo = ym; has_cl = true; } else { cert_hi = ym; has_ch = true; }
      } else {
        py[np] = ym;
        pp[np] = p;
        ++np;
        const double palt = p * (right ? 1.0 - pa : pa);
        const double alt = right ? 0.5 * (lo + ym) : 0.5 * (ym + hi);
        if (palt > 1e-12 && palt > hpmin && alt > clo && alt < chi) {
          bool done = false;   // replace the first slot holding the minimum
#pragma unroll
          for (int k = 0; k < MAX_HEDGE; ++k)
            if (!done && hp[k] == hpmin) { hp[k] = palt; hy[k] = alt; done = true; }
          hpmin = hp[0];
#pragma unroll
          for (int k = 1; k < MAX_HEDGE; ++k) hpmin = dmin_(hpmin, hp[k]);
        }
        p = p * (right ? pa : 1.0 - pa);
      }
      if (right) lo = ym; else hi = ym;
    }
    ym = 0.5 * (lo + hi);
    ++it;
  }
  if (has_cl && n < K) out[n++] = cert_lo;
  if (has_ch && n < K) out[n++] = cert_hi;
  ctl_mark(6);
  // merge (path nodes are ordered by decreasing probability; a hedge is
  // taken when more probable than the next path node -- its parent, being
  // more probable still, has then already been taken).
  int ip = 0;
  while (n < K) {
    double hbest = hp[0];
#pragma unroll
    for (int k = 1; k < MAX_HEDGE; ++k) hbest = dmax_(hbest, hp[k]);
    if (ip < np && pp[ip] >= hbest) {
      out[n++] = py[ip++];
    } else if (hbest > 0.0) {
      bool done = false;
#pragma unroll
      for (int k = 0; k < MAX_HEDGE; ++k)
        if (!done && hp[k] == hbest) { out[n++] = hy[k]; hp[k] = -1.0; done = true; }
    } else {
      break;
    }
  }
  ctl_mark(7);
  return n;
}

// Initialise a walk from the PREP totals (projection.cpp:53-97).  r0_exact:
// r0 is the reference-order r(0) (strict parity); otherwise, in strict mode,
// an r0 within the error bound E of a decision asks for it first.
TOPT_NOINLINE void walk_init(Walk& w, int eq, double ghat, double E, double r0, double S0,
                             double bp_lo, double bp_hi, double any, double count,
                             bool strict = false, bool r0_exact = false) {
  Walk z = {};
  w = z;
  w.eq = eq; w.ghat = ghat; w.E = E; w.r0 = r0; w.S0 = S0;
  w.bp_lo = bp_lo; w.bp_hi = bp_hi; w.count = count; w.any_ = any;
  w.min_margin = 1e300;
  if (strict && !r0_exact && fabs(r0) <= E) {
    w.status = WK_EXACT; w.ex_state = 2; w.ex_y = 0.0;
    return;
  }
  const double Ec = r0_exact ? 0.0 : E;   // certificate margin at y = 0
  if (!eq && r0 <= 0.0) {             // inactive: y = 0, residual = max(r0, 0)
    w.status = WK_DONE; w.y = 0.0; w.residual = dmax_(r0, 0.0);
    if (!r0_exact && fabs(r0) <= E) { w.near_ties++; }
    w.min_margin = r0_exact ? 1e300 : fabs(r0) / E;
    return;
  }
  if (eq && r0 == 0.0) { w.status = WK_DONE; w.y = 0.0; w.residual = 0.0; return; }
  if (!(any > 0.0)) { w.status = WK_INFEASIBLE; return; }
  if (r0 > 0.0) {
    w.up = 0; w.lo = bp_lo; w.hi = 0.0;
    w.hasB = 1; w.yb = 0.0; w.Rb = r0; w.Sb = S0;
    if (r0 > Ec) { w.hasH = 1; w.yH = 0.0; }
  } else {
    w.up = 1; w.lo = 0.0; w.hi = bp_hi;
    w.hasA = 1; w.ya = 0.0; w.Ra = r0; w.Sa = S0;
    if (r0 < -Ec) { w.hasL = 1; w.yL = 0.0; }
  }
  w.ym = 0.5 * (w.lo + w.hi);
  w.iters = 0;
  w.status = WK_NEED;
  w.residual = -1.0;   // filled by the FINAL pass (|r(ym)|)
}

// A reference-order value r(y) (strict parity) as a certificate: r is
// monotone in y for the reference's own rounding too (every rounded term is
// monotone, and so is a sequential floating-point sum), so r(y) > 0 decides
// every midpoint >= y and r(y) <= 0 every midpoint <= y.
TOPT_HD void walk_exact_value(Walk& w, double y, double r) {
  if (r > 0.0) {
    if (!w.hasH || y < w.yH) { w.hasH = 1; w.yH = y; }
    if (!w.hasB || y < w.yb) { w.hasB = 1; w.yb = y; w.Rb = r; w.Sb = 0.0; }
  } else {
    if (r < 0.0) {
      if (!w.hasL || y > w.yL) { w.hasL = 1; w.yL = y; }
    } else if (!w.hasL0 || y > w.yL0) {
      w.hasL0 = 1; w.yL0 = y;
    }
    if (!w.hasA || y > w.ya) { w.hasA = 1; w.ya = y; w.Ra = r; w.Sa = 0.0; }
  }
}

// ---------------------------------------------------------------------------
// Plan-level control

TOPT_HD int gram_idx(int m, int j, int k) {  // packed upper triangle, j <= k
  return j * m - j * (j - 1) / 2 + (k - j);
}

TOPT_HDN inline void set_error(Plan& pl, int st) {
  pl.res.status = st;
  pl.stage = SG_DONE;
  pl.cmd.phase = PH_DONE;
  pl.cmd.nslots = 0;
}

// ---- strict parity: chain passes (PH_EXACT) ------------------------------
TOPT_HDN inline void ex_begin(Plan& pl, int what, int seq) {
  Cmd& c = pl.cmd;
  c.phase = PH_EXACT;
  c.ex_n = 0;
  c.ex_seq = seq;
  c.ex_what = what;
  c.nslots = 0;
}
TOPT_HDN inline void ex_add(Plan& pl, int kind, int j, int k, double y, double start) {
  Cmd& c = pl.cmd;
  if (c.ex_n >= MAX_EX) return;
  ExChain& e = c.ex[c.ex_n++];
  e.kind = (int8_t)kind; e.j = (int8_t)j; e.k = (int8_t)k; e.pad_ = 0; e.pad2_ = 0;
  e.y = y; e.start = start;
  c.nslots = c.ex_n;
}
// Element sequence the reference sums a walk of row j over: its partition
// set on the independent path (projection.cpp:242-248), all of 0..n-1 else.
TOPT_HD int walk_seq(const Plan& pl, int j) {
  const bool indep = pl.stage == SG_INDEP ||
                     (pl.stage == SG_FINAL && pl.res.path == PATH_INDEPENDENT);
  return (indep && pl.P.has_part) ? j : -1;
}

TOPT_HDN inline void cmd_final(Plan& pl, const double* y, int resid_rows) {
  Cmd& c = pl.cmd;
  c.phase = PH_FINAL;
  c.local = 0;
  for (int j = 0; j < MAX_M; ++j) c.y[j] = (j < pl.P.m) ? y[j] : 0.0;
  c.resid_rows = resid_rows;
  c.nslots = resid_rows ? pl.P.m : 0;
  c.write_delta = pl.P.delta_out != nullptr;
  c.write_x = pl.P.x_out != nullptr;
  c.write_mask = pl.P.mask_out != nullptr;
  pl.stage = SG_FINAL;
}

TOPT_HDN inline void cmd_newton(Plan& pl) {
  Cmd& c = pl.cmd;
  const int m = pl.P.m;
  if (pl.P.strict) {   // h-dots and the Gram in the reference's order: chains
    ex_begin(pl, EXW_NEWTON, -1);
    for (int j = 0; j < MAX_M; ++j) c.y[j] = (j < m) ? pl.nt.ty[j] : 0.0;
    for (int k = 0; k < m; ++k) ex_add(pl, CH_DOTZ, 0, k, 0.0, 0.0);
    for (int j = 0; j < m; ++j)
      for (int k = j; k < m; ++k) ex_add(pl, CH_GRAM, j, k, 0.0, 0.0);
    pl.stage = SG_NEWTON;
    return;
  }
  c.phase = PH_NEWTON;
  c.local = 0;
  for (int j = 0; j < MAX_M; ++j) c.y[j] = (j < m) ? pl.nt.ty[j] : 0.0;
  c.want_gram = 1;
  c.nslots = m + m * (m + 1) / 2;
  pl.stage = SG_NEWTON;
}

TOPT_HDN inline void start_newton(Plan& pl) {
  Newton& nt = pl.nt;
  Newton z = {};
  nt = z;
  for (int j = 0; j < pl.P.m; ++j) nt.ty[j] = 0.0;
  nt.in_linesearch = 0;
  cmd_newton(pl);
}

// Walks waiting for reference-order values -> one chain pass: the pending
// point, and (lanes are free) the walk's next midpoints breadth-first, so one
// pass settles several near-tie levels.  Rows of different element sequences
// (partition sets) go in separate passes.
TOPT_NOINLINE bool schedule_exact_walks(Plan& pl) {
  const int m = pl.P.m;
  int rows[MAX_M], nr = 0, seq = -2;
  for (int j = 0; j < m; ++j) {
    if (pl.w[j].status != WK_EXACT) continue;
    const int sq = walk_seq(pl, j);
    if (seq == -2) seq = sq;
    if (sq == seq) rows[nr++] = j;
  }
  if (!nr) return false;
  ex_begin(pl, EXW_WALK, seq);
  const int budget = MAX_EX / nr;
  double* qlo = pl.sc.nlo;
  double* qhi = pl.sc.nhi;
  for (int r = 0; r < nr; ++r) {
    const Walk& w = pl.w[rows[r]];
    const double start = -w.ghat;
    if (w.ex_state == 2 || !w.feas_done) {
      ex_add(pl, CH_RESID, rows[r], 0, w.ex_y, start);
      continue;
    }
    int head = 0, tail = 1, cnt = 0;
    qlo[0] = w.lo; qhi[0] = w.hi;
    while (cnt < budget && head < tail) {
      const double l = qlo[head], h = qhi[head];
      ++head;
      const double y = 0.5 * (l + h);
      ex_add(pl, CH_RESID, rows[r], 0, y, start);
      ++cnt;
      if (tail + 2 <= CAND_CAP) {
        qlo[tail] = l; qhi[tail] = y; ++tail;
        qlo[tail] = y; qhi[tail] = h; ++tail;
      }
    }
  }
  return true;
}

// ---- root sketch ------------------------------------------------------------
// Before the first full sweep of a large problem, SKETCH_PASSES sampled sweeps
// (cmd.sample = s: every 2^s-th step of each thread's element loop, about
// n / 2^s elements spread over the whole index range) evaluate the walks'
// candidates approximately.  Their sums are never evidence -- no bracket, no
// certificate, no walk decision uses them: they only place the root estimate
// (Walk::hy, hs) the candidate choice starts from.  The first full sweep's
// candidates, and with them the window [y_first, y_last] outside which an
// element costs three running sums instead of a per-candidate loop, are then
// already narrow (C5 first sweep: 7.9 ms with the r(0) Newton estimate).
constexpr int SKETCH_PASSES = 4;   // at most; the sketch stops at its sampling-noise floor
TOPT_HD int sketch_shift(const Plan& pl) {   // 1/16 of the elements, 1/64 from 2^28 on
  const int64_t n = pl.P.n_global;
  return 4 + (n >= ((int64_t)1 << 26) ? 1 : 0) + (n >= ((int64_t)1 << 28) ? 1 : 0);
}

TOPT_HD bool sketch_wanted(const Plan& pl) {
  const Problem& P = pl.P;
  return P.sketch_min_n > 0 && P.n_global >= P.sketch_min_n && !P.strict && !P.has_part;
}

// A sketch command = the sweep command just built, run over the sample; one
// extra slot returns the number of elements visited.
TOPT_HDN inline void sketch_command(Plan& pl) {
  Cmd& c = pl.cmd;
  c.sample = 0;
  if (pl.sketch_left > 0 && !c.local && c.phase == PH_SWEEP) {
    c.sample = sketch_shift(pl);
    c.compact = 0;
    c.nslots = 2 * c.ncand + 1 + pl.P.m;   // + elements visited + each row's sampled r(0) sum
    pl.res.sweeps--;   // not a sweep of the walk (the first full sweep is still "first")
  }
}

TOPT_NOINLINE void consume_sketch(Plan& pl, const double* t) {
  const int m = pl.P.m;
  Cmd& c = pl.cmd;
  const double visited = t[2 * c.ncand];
  const double scale = visited > 0.0 ? (double)pl.P.n_global / visited : 0.0;
  bool refine = false;   // some row's bracket is still wider than its sampling noise
  for (int j = 0; j < m; ++j) {
    const int b = c.row_start[j], e = c.row_start[j + 1];
    if (e <= b || !(scale > 0.0)) continue;
    Walk& w = pl.w[j];
    // nearest points on either side of the sampled root, seeded with what the
    // walk knows exactly (r(0) from PREP)
    bool ha = w.hasA != 0, hb = w.hasB != 0;
    double ya = w.ya, Ra = w.Ra, yb = w.yb, Rb = w.Rb;
    double smax = dmax_(ha ? w.Sa : 0.0, hb ? w.Sb : 0.0);
    // r(y) ~ r(0) [exact, from PREP] + scale (sampled sum at y - sampled sum
    // at 0): only the terms that change between 0 and y carry sampling
    // noise (the clipped constants of the centre-of-mass rows, which cancel
    // to a small r over the whole vector but not over a sample, drop out)
    const double R0s = t[2 * c.ncand + 1 + j];
    double dmax = 0.0;
    for (int k = b; k < e; ++k) {
      const double y = c.cand_y[k], D = scale * (t[2 * k] - R0s), R = w.r0 + D;
      const double S = scale * t[2 * k + 1];
      smax = dmax_(smax, S);
      if (fabs(R) <= fabs(w.r0)) dmax = dmax_(dmax, fabs(D));   // |difference| near the root
      if (R <= 0.0 && (!ha || y > ya)) { ha = true; ya = y; Ra = R; }
      if (R > 0.0 && (!hb || y < yb)) { hb = true; yb = y; Rb = R; }
    }
    if (!(ha && hb)) continue;   // no sign change among the points: keep the earlier estimate
    double hy;
    if (ya < yb) {
      hy = ya - est_div(Ra * (yb - ya), Rb - Ra);
      if (!(hy >= ya)) hy = ya;
      if (!(hy <= yb)) hy = yb;
    } else {   // sampling noise crossed the two sides: the middle of the span
      const double tmp = ya; ya = yb; yb = tmp;
      hy = 0.5 * (ya + yb);
    }
    // sampling noise of the scaled difference, ~ 6 |difference| / sqrt(visited)
    // (coefficient of variation of the changed terms taken as <= 6), in units of y
    const double noise = smax > 0.0 ? est_div(6.0 * dmax_(dmax, fabs(w.r0)), sqrt(visited) * smax) : 0.0;
    const double width = 0.125 * (yb - ya);
    refine = refine || width > noise;
    const double hs = dmax_(dmax_(width, noise), 1e-300);
    w.hok = 1; w.hy = hy; w.hs = hs;
  }
  pl.sketch_left = refine ? pl.sketch_left - 1 : 0;
  c.sample = 0;
}

// Build the next sweep over all walks that need evaluations; if none do,
// advance the stage.  Returns true if a sweep was scheduled.
TOPT_HDN inline int schedule_per(const Plan& pl, int need) {
  int per = MAX_CAND / need;
  if (per > MAX_K) per = MAX_K;
  // a walk's first full sweep has a wide window (the per-candidate loop runs
  // for a large share of the elements): with a sketched root estimate fewer
  // candidates place the next bracket almost as well
  if (pl.P.first_k > 0 && pl.res.sweeps == 0 && pl.sketch_left == 0 && !pl.cmd.local &&
      sketch_wanted(pl) && per > pl.P.first_k)
    per = pl.P.first_k;
  return per;
}

TOPT_NOINLINE bool schedule_sweep(Plan& pl) {
  if (schedule_exact_walks(pl)) return true;
  const int m = pl.P.m;
  int need = 0;
  for (int j = 0; j < m; ++j) need += (pl.w[j].status == WK_NEED);
  if (!need) return false;
  const int per = schedule_per(pl, need);
  Cmd& c = pl.cmd;
  c.phase = PH_SWEEP;
  int tot = 0;
  for (int j = 0; j < m; ++j) {
    c.row_start[j] = tot;
    if (pl.w[j].status == WK_NEED) {
      const Walk w = pl.w[j];
      const int nc = walk_candidates(w, pl.P.opt, per, c.cand_y + tot, pl.sc);
      double* cy = c.cand_y + tot;   // the sweeps want each row's candidates ascending
      for (int a = 1; a < nc; ++a) {
        const double v = cy[a];
        int b = a - 1;
        while (b >= 0 && cy[b] > v) { cy[b + 1] = cy[b]; --b; }
        cy[b + 1] = v;
      }
      tot += nc;
    }
  }
  for (int j = m; j <= MAX_M; ++j) c.row_start[j] = tot;
  c.compact = (pl.P.compact_cap > 0 && (m == 1 || pl.P.has_part) &&
               (c.local || pl.res.sweeps > 0)) ? 1 : 0;   // see schedule_sweep_warp
  for (int j = 0; j < m; ++j) walk_window(pl.w[j], &c.wlo[j], &c.whi[j]);
  c.ncand = tot;
  // compacted global sweeps append two slots: the active elements left and
  // the CTAs holding more than GATHER_BLK of them
  c.nslots = 2 * tot + ((c.compact && !c.local) ? 2 : 0);
  if (c.local) pl.res.local_sweeps++; else pl.res.sweeps++;
  sketch_command(pl);
  return true;
}

TOPT_NOINLINE void after_walks(Plan& pl);

// finish_newton_or_loop in two halves around the m x m solve, so that the
// device can run the solve on a whole warp: _pre builds J_Phi (sc.jp) and
// returns 1 when a solve J_Phi step = Phi is pending; _post consumes it.
TOPT_NOINLINE int finish_newton_pre(Plan& pl) {
  Newton& nt = pl.nt;
  const Problem& P = pl.P;
  const int m = P.m;
  double linf = 0.0;
  for (int j = 0; j < m; ++j) linf = dmax_(linf, fabs(nt.phi[j]));
  if (linf > P.opt.tol_n && nt.iters < P.opt.newton_maxiter) {
    double* jh = pl.sc.jh;
    double* jp = pl.sc.jp;
    for (int j = 0; j < m; ++j)
      for (int k = j; k < m; ++k) {
        const double v = nt.gram[gram_idx(m, j, k)];
        jh[k * m + j] = v;
        jh[j * m + k] = v;
      }
    for (int j = 0; j < m; ++j) jh[j * m + j] = jh[j * m + j] + 1.0 / P.opt.c;
    for (int j = 0; j < m; ++j) {           // projection.cpp:382-392
      if (P.is_eq[j]) {
        for (int k = 0; k < m; ++k) jp[k * m + j] = jh[k * m + j];
      } else if (-nt.y[j] <= -nt.h[j]) {
        for (int k = 0; k < m; ++k) jp[k * m + j] = 0.0;
        jp[j * m + j] = -1.0;
      } else {
        for (int k = 0; k < m; ++k) jp[k * m + j] = -jh[k * m + j];
      }
    }
    if (nt.have_prev) {                     // projection.cpp:396-399
      double curv = 0.0;
      for (int j = 0; j < m; ++j) {
        double s = 0.0;
        for (int k = 0; k < m; ++k) s = s + jp[k * m + j] * nt.step[k];
        curv = curv + nt.phi[j] * s;
      }
      if (curv > 0.9 * nt.prev_phi_sq) nt.curv_viol++;
    }
    return 1;
  }
  Result& r = pl.res;
  r.path = PATH_NEWTON;
  r.newton_iters = nt.iters;
  r.residual = linf;
  r.converged = linf <= P.opt.tol_n;
  r.curvature_violations = nt.curv_viol;
  r.stage1_row = -1;
  for (int j = 0; j < m; ++j) {
    r.y[j] = nt.y[j];
    r.slacks[j] = -nt.y[j] / P.opt.c;
    r.h[j] = nt.h[j];
  }
  cmd_final(pl, nt.y, 0);
  return 0;
}

TOPT_NOINLINE void finish_newton_post(Plan& pl, bool solved) {
  Newton& nt = pl.nt;
  const int m = pl.P.m;
  if (!solved) { set_error(pl, ST_NUMERICAL); return; }
  for (int j = 0; j < m; ++j)
    if (!isfinite(nt.step[j])) { set_error(pl, ST_NUMERICAL); return; }
  double sq = 0.0;
  for (int j = 0; j < m; ++j) sq = sq + nt.phi[j] * nt.phi[j];
  nt.phi_sq = sq;
  nt.merit0 = nt.merit;
  nt.gamma = 1.0;
  for (int j = 0; j < m; ++j) nt.ty[j] = nt.y[j] - nt.gamma * nt.step[j];
  nt.in_linesearch = 1;
  cmd_newton(pl);
}



// consume_newton up to the pending solve (returns finish_newton_pre's flag).
TOPT_NOINLINE int consume_newton_core(Plan& pl, const double* t) {
  Newton& nt = pl.nt;
  const Problem& P = pl.P;
  const int m = P.m;
  double th[MAX_M], tphi[MAX_M];
  double sq = 0.0;
  for (int j = 0; j < m; ++j) {           // eval_phi, projection.cpp:287-296
    th[j] = t[j] + nt.ty[j] / P.opt.c - pl.res.ghat[j];
    tphi[j] = P.is_eq[j] ? th[j] : dmin_(-nt.ty[j], -th[j]);
    sq = sq + tphi[j] * tphi[j];
  }
  const double tmerit = 0.5 * sq;
  const int ng = m * (m + 1) / 2;
  if (!nt.in_linesearch) {                // initial evaluation at y = 0
    for (int j = 0; j < m; ++j) { nt.y[j] = nt.ty[j]; nt.h[j] = th[j]; nt.phi[j] = tphi[j]; }
    for (int k = 0; k < ng; ++k) nt.gram[k] = t[m + k];
    nt.merit = tmerit;
    return finish_newton_pre(pl);
  }
  const double c1 = 1e-4;                 // projection.cpp:415-422
  if (tmerit <= nt.merit0 - c1 * nt.gamma * nt.phi_sq || nt.gamma < 1e-16) {
    for (int j = 0; j < m; ++j) {
      nt.y[j] = nt.ty[j];
      nt.step[j] = nt.step[j] * nt.gamma;
      nt.h[j] = th[j];
      nt.phi[j] = tphi[j];
    }
    nt.prev_phi_sq = nt.gamma * nt.phi_sq;
    nt.have_prev = 1;
    nt.merit = tmerit;
    for (int k = 0; k < ng; ++k) nt.gram[k] = t[m + k];
    nt.iters++;
    nt.in_linesearch = 0;
    return finish_newton_pre(pl);
  }
  nt.gamma = nt.gamma * 0.5;
  for (int j = 0; j < m; ++j) nt.ty[j] = nt.y[j] - nt.gamma * nt.step[j];
  cmd_newton(pl);
  return 0;
}

TOPT_NOINLINE void consume_newton(Plan& pl, const double* t) {
  if (consume_newton_core(pl, t))
    finish_newton_post(pl, fullpiv_solve(pl.P.m, pl.sc.jp, pl.nt.phi, pl.nt.step));
}



// Stage-1 feasibility (projection.cpp:320-342) over every row whose bisection
// succeeded, evaluated in one pass; first feasible row by index wins.
TOPT_HDN inline void schedule_feas(Plan& pl) {
  const int m = pl.P.m;
  Cmd& c = pl.cmd;
  c.phase = PH_FEAS;
  c.local = 0;
  int nf = 0, zero_idx = -1;
  for (int j = 0; j < m; ++j) {
    Walk& w = pl.w[j];
    pl.feas_map[j] = -1;
    if (w.status != WK_DONE) continue;
    if (w.y == 0.0) {
      if (zero_idx < 0) { zero_idx = nf; c.feas_row[nf] = -1; c.feas_y[nf] = 0.0; ++nf; }
      pl.feas_map[j] = zero_idx;
    } else {
      c.feas_row[nf] = j; c.feas_y[nf] = w.y; pl.feas_map[j] = nf; ++nf;
    }
  }
  c.nfeas = nf;
  c.nslots = nf * m;
  // The FEAS pass of the detected C4/C5 row layout reads exactly what
  // Newton's first evaluation (y = 0, projection.cpp:345-357) reads: it
  // returns that evaluation too, and a Newton solve that follows starts from
  // it without a pass of its own.
  c.feas_gram0 = (pl.P.pat7 && !pl.P.strict && nf > 0) ? 1 : 0;
  if (c.feas_gram0) c.nslots += m + m * (m + 1) / 2;
  pl.stage = SG_FEAS;
  if (nf == 0) start_newton(pl);
}

TOPT_NOINLINE void consume_feas(Plan& pl, const double* t) {
  const Problem& P = pl.P;
  const int m = P.m;
  if (P.strict && pl.cmd.phase == PH_FEAS) {   // every stage-1 dot in the reference's order
    ex_begin(pl, EXW_FEAS, -1);
    for (int f = 0; f < pl.cmd.nfeas; ++f)
      for (int k = 0; k < m; ++k)
        ex_add(pl, CH_FEAS, pl.cmd.feas_row[f], k, pl.cmd.feas_y[f], 0.0);
    return;
  }
  for (int j = 0; j < m; ++j) {
    const int f = pl.feas_map[j];
    if (f < 0) continue;
    bool feasible = true;
    double worst = 0.0;
    for (int k = 0; k < m && feasible; ++k) {
      const double v = t[f * m + k] - pl.res.ghat[k];
      const double viol = P.is_eq[k] ? fabs(v) : v;
      feasible = viol <= P.opt.tol_n;
      worst = dmax_(worst, fabs(v));
    }
    if (feasible) {
      Result& r = pl.res;
      double y[MAX_M];
      for (int k = 0; k < m; ++k) { y[k] = 0.0; r.slacks[k] = 0.0; }
      y[j] = pl.w[j].y;
      for (int k = 0; k < m; ++k) r.y[k] = y[k];
      r.path = PATH_SINGLE;
      r.residual = worst;
      r.newton_iters = 0;
      r.converged = 1;
      r.curvature_violations = 0;
      r.stage1_row = j;
      cmd_final(pl, y, 0);
      return;
    }
  }
  if (pl.cmd.feas_gram0 && pl.cmd.phase == PH_FEAS) {
    // Newton's evaluation at y = 0 came with the FEAS pass: consume it as if
    // a PH_NEWTON pass had returned it (scalar m x m solve: same pivots and
    // arithmetic as the warp version)
    const double* t0 = t + pl.cmd.nfeas * m;
    Newton& nt = pl.nt;
    Newton z = {};
    nt = z;
    nt.in_linesearch = 0;
    pl.stage = SG_NEWTON;
    pl.cmd.feas_gram0 = 0;
    consume_newton(pl, t0);
    return;
  }
  start_newton(pl);
}

TOPT_NOINLINE void after_walks(Plan& pl) {
  const Problem& P = pl.P;
  const int m = P.m;
  Result& r = pl.res;
  int infeasible = 0;
  for (int j = 0; j < m; ++j) {
    infeasible += (pl.w[j].status == WK_INFEASIBLE);
    r.bisect_iters[j] = pl.w[j].iters;
    r.near_ties += pl.w[j].near_ties;
    r.min_margin = dmin_(r.min_margin, pl.w[j].min_margin);
  }
  if (pl.stage == SG_SINGLE || pl.stage == SG_INDEP) {
    if (infeasible) {
      if (P.which != W_AUTO) { set_error(pl, ST_INFEASIBLE); return; }
      if (pl.stage == SG_SINGLE) { start_newton(pl); return; }  // stage 1 would skip row 0
      pl.stage = SG_STAGE1;  // subset walks == full-row walks (zeros contribute nothing)
      schedule_feas(pl);
      return;
    }
    double y[MAX_M];
    for (int j = 0; j < m; ++j) { y[j] = pl.w[j].y; r.y[j] = y[j]; r.slacks[j] = 0.0; }
    r.path = pl.stage == SG_SINGLE ? PATH_SINGLE : PATH_INDEPENDENT;
    r.newton_iters = 0;
    r.converged = 1;
    r.curvature_violations = 0;
    r.stage1_row = -1;
    cmd_final(pl, y, 1);
    return;
  }
  // SG_STAGE1
  schedule_feas(pl);
}

// PREP totals -> g_hat, error bounds, walks, path dispatch.
TOPT_NOINLINE void consume_prep_core(Plan& pl, const double* t) {
  Problem& P = pl.P;
  const int m = P.m;
  Result& r = pl.res;
  if (pl.cmd.pat_hint) {
    // the pattern PREP derived rows 2, 4, 6 from rows 1, 3, 5: valid only if
    // every element verified as the exact negation -- else the general PREP
    // runs again (cmd.phase stays PH_PREP, d and rho_tilde are rewritten alike)
    bool bad = false;
    for (int j = 2; j < m; j += 2) bad = bad || t[j * PREP_SLOTS + PS_NNEG] != 0.0;
    if (bad) { pl.cmd.pat_hint = 0; return; }
  }
  for (int j = 0; j < m; ++j) {
    const double* s = t + j * PREP_SLOTS;
    double ghat, gerr;
    const double cnt = P.row_count[j];
    const double ours = P.ours_len;
    const bool ex = pl.ghat_ex_ok != 0;     // reference-order dot (strict parity)
    const double dot = ex ? pl.ghat_dot_ex[j] : s[PS_DOT];
    if (pl.dot_mode) {  // projection.cpp:139-145: (G - g) + dot
      ghat = P.G_minus_g[j] + dot;
      gerr = ex ? 0.0
                : (gamma_k((double)P.n_global + 2.0) + gamma_k(ours)) * s[PS_DABS] +
                      2.0 * kUnit * fabs(ghat);
    } else {
      ghat = P.ghat_in[j];
      gerr = P.ghat_err_in[j];
      if (pl.cmd.validate_part && P.gd_step) {  // validate(): 1e-14 consistency
        const double expect = P.G_minus_g[j] + dot;
        const double scale = dmax_(dmax_(1.0, fabs(expect)), fabs(ghat));
        if (fabs(ghat - expect) > 1e-14 * scale) { set_error(pl, ST_DOMAIN); return; }
      }
    }
    r.ghat[j] = ghat;
    r.ghat_err[j] = (ex && pl.dot_mode) ? 0.0
                    : (gamma_k((double)P.n_global + 2.0) + gamma_k(ours)) * s[PS_DABS];
    if (pl.cmd.validate_part && s[PS_NZOUT] > 0.0) { set_error(pl, ST_DOMAIN); return; }
    // + 16u T: sweeps sum free terms as y * sum(a^2) instead of
    // sum fl(fl(y a) a), and classify regions by breakpoints (passes.cuh).
    const double E = 1.0625 * (gamma_k(cnt + 2.0) * (fabs(ghat) + s[PS_T]) + gerr +
                               gamma_k(ours) * (fabs(ghat) + s[PS_T]) +
                               16.0 * kUnit * s[PS_T]) + 1e-300;
    const double r0 = s[PS_S0] - ghat;
    walk_init(pl.w[j], P.is_eq[j], ghat, E, r0, s[PS_SLOPE0], s[PS_BPLO], s[PS_BPHI],
              s[PS_ANY], cnt, P.strict != 0);
    if (pl.hint_ok[j]) { pl.w[j].hok = 1; pl.w[j].hy = pl.hint_y[j]; pl.w[j].hs = pl.hint_sig[j]; }
    pl.sk_T[j] = s[PS_T];
  }
  pl.sketch_left = sketch_wanted(pl) ? SKETCH_PASSES : 0;
  // Row structure seen by PREP (every row was read once): constant rows and
  // rows that are the exact negation of their predecessor.  The later passes
  // then read each distinct row once and derive the others bit for bit
  // (negation and a constant are exact), so results do not change.
  P.n_alias = 0;
  P.pat7 = 0;
  for (int j = 0; j < MAX_M; ++j) { P.alias_kind[j] = AK_DENSE; P.alias_c[j] = 0.0; }
  if (!P.structured && !P.owner && P.n_global == P.n && m >= 2 && m <= 8) {
    for (int j = 0; j < m; ++j) {
      const double* sj = t + j * PREP_SLOTS;
      if (sj[PS_NCONST] == 0.0) {
        P.alias_kind[j] = AK_CONST; P.alias_c[j] = sj[PS_AREF]; P.n_alias++;
      } else if (j >= 1 && sj[PS_NNEG] == 0.0 && P.alias_kind[j - 1] == AK_DENSE) {
        P.alias_kind[j] = AK_NEG; P.n_alias++;
      }
    }
    P.pat7 = (m == 7 && P.alias_kind[0] == AK_CONST && P.alias_kind[1] == AK_DENSE &&
              P.alias_kind[2] == AK_NEG && P.alias_kind[3] == AK_DENSE &&
              P.alias_kind[4] == AK_NEG && P.alias_kind[5] == AK_DENSE &&
              P.alias_kind[6] == AK_NEG) ? 1 : 0;
  }
  r.pat7 = P.pat7;
  if (P.job == JOB_BUILD || P.job == JOB_DIRECTION) { set_error(pl, ST_OK); return; }
  if (m < 1) { set_error(pl, ST_DOMAIN); return; }
  // Path dispatch, projection.cpp:440-460
  if (P.which == W_NEWTON) {
    pl.stage = SG_STAGE1;
  } else if (P.which == W_SINGLE || (P.which == W_AUTO && m == 1)) {
    if (m != 1) { set_error(pl, ST_DOMAIN); return; }
    pl.stage = SG_SINGLE;
  } else if (P.which == W_INDEPENDENT || (P.which == W_AUTO && P.has_part)) {
    if (!P.has_part) { set_error(pl, ST_DOMAIN); return; }
    pl.stage = SG_INDEP;
  } else {
    pl.stage = SG_STAGE1;
  }
  const Evals none = {nullptr, nullptr, 0};
  for (int j = 0; j < m; ++j) walk_advance(pl.w[j], P.opt, none, P.strict != 0);
  pl.cmd.phase = PH_SWEEP;   // marker: the caller schedules the first sweep
  pl.cmd.nslots = -1;
}

// Strict parity: g_hat's dot (ConstraintLinearization::build / validate,
// projection.cpp:140-145, :151-155) in the reference's order before any
// decision uses it; the PREP totals wait in the plan meanwhile.
TOPT_HD bool prep_needs_exact(const Plan& pl) {
  return pl.P.strict && !pl.ghat_ex_ok && pl.P.m > 0 &&
         (pl.dot_mode || (pl.cmd.validate_part && pl.P.gd_step != nullptr));
}
TOPT_NOINLINE void schedule_exact_ghat(Plan& pl, const double* t) {
  const int m = pl.P.m;
  for (int k = 0; k < m * PREP_SLOTS; ++k) pl.prep_save[k] = t[k];
  ex_begin(pl, EXW_GHAT, -1);
  for (int j = 0; j < m; ++j) ex_add(pl, CH_GHAT, j, 0, 0.0, 0.0);
}

// (returns with cmd.nslots == -1 when the walks need their first sweep)
TOPT_NOINLINE void consume_prep(Plan& pl, const double* t) {
  if (prep_needs_exact(pl)) { schedule_exact_ghat(pl, t); return; }
  consume_prep_core(pl, t);
  if (pl.cmd.phase == PH_SWEEP && pl.cmd.nslots == -1)
    if (!schedule_sweep(pl)) after_walks(pl);
}

TOPT_NOINLINE void consume_sweep(Plan& pl, const double* t) {
  const int m = pl.P.m;
  Cmd& c = pl.cmd;
  ctl_mark(0);
  if (c.sample) {   // a sketch: steer the candidates, decide nothing
    consume_sketch(pl, t);
    if (!schedule_sweep(pl)) after_walks(pl);
    return;
  }
  const bool was_global_compact = c.compact && !c.local;
  if (was_global_compact) pl.res.active = t[2 * c.ncand];
  for (int j = 0; j < m; ++j) {
    const int b = c.row_start[j], e = c.row_start[j + 1];
    if (e <= b) continue;
    Walk w = pl.w[j];                      // registers for the replay
    const Evals ev = {c.cand_y + b, t + 2 * b, e - b};
    walk_ingest(w, ev);
    ctl_mark(1);
    walk_advance(w, pl.P.opt, ev, pl.P.strict != 0);
    ctl_mark(2);
    pl.w[j] = w;
  }
  // few active elements left: gather them into every CTA and finish the
  // walks CTA-locally (no grid barrier per sweep)
  int need = 0;
  for (int j = 0; j < m; ++j) need += (pl.w[j].status == WK_NEED);
  if (need && was_global_compact && pl.res.active <= (double)GATHER_TRIGGER) {
    if (t[2 * c.ncand + 1] == 0.0) {   // every CTA published its items (fused gather)
      c.local = 1;
      c.load_fused = 1;
      pl.res.gathered = 1;
      if (!schedule_sweep(pl)) after_walks(pl);
      ctl_mark(3);
      return;
    }
    c.phase = PH_GATHER;
    c.nslots = 0;
    ctl_mark(3);
    return;
  }
  if (!schedule_sweep(pl)) after_walks(pl);
  ctl_mark(3);
}


TOPT_NOINLINE void consume_gather(Plan& pl) {
  pl.cmd.local = 1;
  pl.res.gathered = 1;
  if (!schedule_sweep(pl)) after_walks(pl);
}

// Strict parity: |r(y)| of the walked rows in the reference's order
// (projection.cpp:108), one element sequence per pass.  Returns false when
// no row is pending.
TOPT_NOINLINE bool schedule_exact_final(Plan& pl) {
  const int m = pl.P.m;
  int seq = -2;
  for (int j = 0; j < m; ++j) {
    const Walk& w = pl.w[j];
    if (!(w.residual < 0.0)) continue;
    const int sq = walk_seq(pl, j);
    if (seq == -2) { seq = sq; ex_begin(pl, EXW_FINAL, seq); }
    if (sq == seq) ex_add(pl, CH_RESID, j, 0, w.y, -w.ghat);
  }
  return seq != -2;
}

TOPT_NOINLINE void finish_final(Plan& pl) {
  Result& r = pl.res;
  pl.stage = SG_DONE;
  pl.cmd.phase = PH_DONE;
  pl.cmd.nslots = 0;
  r.status = ST_OK;
}

TOPT_NOINLINE void consume_final(Plan& pl, const double* t) {
  Problem& P = pl.P;
  Result& r = pl.res;
  const int m = P.m;
  if (P.strict && pl.cmd.phase == PH_FINAL) {
    if (P.job == JOB_RESIDUAL_H) {          // the h-dots as chains (cmd.y = the dual)
      ex_begin(pl, EXW_RESH, -1);
      for (int k = 0; k < m; ++k) ex_add(pl, CH_DOTZ, 0, k, 0.0, 0.0);
      return;
    }
    if (pl.cmd.resid_rows) {
      if (schedule_exact_final(pl)) return;
      double worst = 0.0;
      for (int j = 0; j < m; ++j) worst = dmax_(worst, pl.w[j].residual);
      r.residual = worst;
      finish_final(pl);
      return;
    }
  }
  if (P.job == JOB_RESIDUAL_H) {            // projection.cpp:259-265
    for (int j = 0; j < m; ++j) r.h[j] = t[j] + P.y_in[j] / P.opt.c - P.ghat_in[j];
  } else if (pl.cmd.resid_rows) {           // |r(ym)| per walked row, projection.cpp:108
    double worst = 0.0;
    for (int j = 0; j < m; ++j) {
      Walk& w = pl.w[j];
      if (w.residual < 0.0) w.residual = fabs(t[j] - w.ghat);
      worst = dmax_(worst, w.residual);
    }
    r.residual = worst;
  }
  pl.stage = SG_DONE;
  pl.cmd.phase = PH_DONE;
  pl.cmd.nslots = 0;
  r.status = ST_OK;
}

TOPT_NOINLINE void consume_step(Plan& pl, const double* t) {
  const Problem& P = pl.P;
  const PgdSettings& s = P.set;
  Result& r = pl.res;
  const int fallback = (P.t == 0) || (P.t >= s.t_warmup && P.violation > s.tol_n);
  if (P.strict && !fallback && pl.cmd.phase == PH_STEP_REDUCE) {
    // BB / PR+ sums in oracle.c's order (no reference code)
    for (int k = 0; k < 6; ++k) pl.step_save[k] = t[k];
    ex_begin(pl, EXW_STEP, -1);
    for (int k = 0; k < 5; ++k) ex_add(pl, CH_STEP, 0, k, 0.0, 0.0);
    return;
  }
  for (int k = 0; k < 6; ++k) r.step_sums[k] = t[k];
  double alpha, beta = 0.0;
  if (fallback) {                           // SPEC.md:308 / PAPER.md Alg. 3 lines 4-8
    alpha = dmin_(s.alpha_max, s.alpha_fallback / t[5]);
  } else {
    const double ss = t[0], sy = t[1], yy = t[2];   // SPEC.md:290 (Eq. 13)
    if (yy == 0.0) {
      alpha = s.alpha_max;
    } else {
      const double ns = sqrt(ss), ny = sqrt(yy);
      if (sy <= s.eps_alpha) alpha = dmin_(ns / ny, s.alpha_max);
      else alpha = dmin_(dmin_(ss / sy, 2.0 * ns / ny), s.alpha_max);
    }
    beta = (t[4] == 0.0) ? 0.0 : dmax_(t[3] / t[4], 0.0);   // SPEC.md:299 (Eq. 14, PR+)
  }
  r.alpha = alpha;
  r.beta = beta;
  r.fallback = fallback;
  Cmd& c = pl.cmd;
  c.phase = PH_PREP;
  c.compute_dir = 1;
  c.use_dprev = !fallback;
  c.beta = beta;
  c.wa = s.omega * alpha;
  c.compute_dot = 1;
  c.validate_part = 0;
  c.nslots = P.m * PREP_SLOTS;
  pl.dot_mode = 1;
}

// First command of a job.
TOPT_HDN inline void plan_start(Plan& pl) {
  Problem& P = pl.P;
  Result z = {};
  pl.res = z;
  pl.res.min_margin = 1e300;
  pl.res.stage1_row = -1;
  pl.stage = SG_INIT;
  Cmd& c = pl.cmd;
  c.compute_dir = 0; c.use_dprev = 0; c.compute_dot = 0; c.validate_part = 0;
  c.write_delta = c.write_x = c.write_mask = 0;
  c.compact = 0;
  c.local = 0;
  c.sample = 0;
  pl.sketch_left = 0;
  c.pat_hint = (P.pat_hint && P.job == JOB_PGD_STEP && P.m == 7 && !P.strict && !P.has_part &&
                !P.structured && P.n_global == P.n) ? 1 : 0;
  if (P.job == JOB_PGD_STEP || P.job == JOB_DIRECTION) {
    c.phase = PH_STEP_REDUCE;
    c.nslots = 6;
    return;
  }
  if (P.job == JOB_DELTA || P.job == JOB_RESIDUAL_H) {
    for (int j = 0; j < P.m; ++j) pl.w[j].ghat = P.ghat_in[j];
    cmd_final(pl, P.y_in, P.job == JOB_RESIDUAL_H);
    return;
  }
  c.phase = PH_PREP;
  c.compute_dot = (P.job == JOB_BUILD) || (P.gd_step != nullptr && P.has_part);
  c.validate_part = P.has_part && (P.job == JOB_BUILD || P.which == W_INDEPENDENT ||
                                   (P.which == W_AUTO && P.m > 1));
  c.nslots = P.m * PREP_SLOTS;
  pl.dot_mode = (P.job == JOB_BUILD);
}

// Results of a chain pass (t[c] = chain c's reference-order sum).
TOPT_NOINLINE void consume_exact(Plan& pl, const double* t) {
  Problem& P = pl.P;
  const int m = P.m;
  Cmd& c = pl.cmd;
  pl.res.exact_passes++;
  switch (c.ex_what) {
    case EXW_STEP: {
      double tt[6];
      for (int k = 0; k < 5; ++k) tt[k] = t[k];
      tt[5] = pl.step_save[5];   // max |g| (exact in any order)
      consume_step(pl, tt);      // (cmd.phase is PH_EXACT: the sums are consumed)
      break;
    }
    case EXW_GHAT: {
      for (int j = 0; j < m; ++j) pl.ghat_dot_ex[j] = t[j];
      pl.ghat_ex_ok = 1;
      consume_prep(pl, pl.prep_save);
      break;
    }
    case EXW_WALK: {
      const Evals none = {nullptr, nullptr, 0};
      int touched[MAX_M];
      for (int j = 0; j < m; ++j) touched[j] = 0;
      for (int q = 0; q < c.ex_n; ++q) {
        const int j = c.ex[q].j;
        Walk& w = pl.w[j];
        touched[j] = 1;
        if (w.ex_state == 2) {   // exact r(0): redo the walk's set-up (projection.cpp:53-97)
          const int hok = w.hok;
          const double hy = w.hy, hs = w.hs;
          walk_init(w, w.eq, w.ghat, w.E, t[q], w.S0, w.bp_lo, w.bp_hi, w.any_, w.count,
                    true, true);
          w.hok = hok; w.hy = hy; w.hs = hs;
        } else {
          walk_exact_value(w, c.ex[q].y, t[q]);
        }
      }
      for (int j = 0; j < m; ++j) {
        if (!touched[j]) continue;
        Walk& w = pl.w[j];
        if (w.status == WK_EXACT) w.status = WK_NEED;
        w.ex_state = 0;
        walk_advance(w, P.opt, none, true);
      }
      if (!schedule_sweep(pl)) after_walks(pl);
      break;
    }
    case EXW_FEAS:
      consume_feas(pl, t);       // (cmd.phase is PH_EXACT: decided on these dots)
      break;
    case EXW_NEWTON:
      consume_newton(pl, t);
      break;
    case EXW_FINAL: {
      for (int q = 0; q < c.ex_n; ++q) pl.w[c.ex[q].j].residual = fabs(t[q]);
      if (schedule_exact_final(pl)) break;
      double worst = 0.0;
      for (int j = 0; j < m; ++j) worst = dmax_(worst, pl.w[j].residual);
      pl.res.residual = worst;
      finish_final(pl);
      break;
    }
    case EXW_RESH:
      for (int j = 0; j < m; ++j) pl.res.h[j] = t[j] + P.y_in[j] / P.opt.c - P.ghat_in[j];
      finish_final(pl);
      break;
    default:
      set_error(pl, ST_INTERNAL);
      break;
  }
}

TOPT_NOINLINE void plan_consume(Plan& pl, const double* t) {
  pl.res.passes++;
  switch (pl.cmd.phase) {
    case PH_EXACT: consume_exact(pl, t); break;
    case PH_STEP_REDUCE: consume_step(pl, t); break;
    case PH_PREP: consume_prep(pl, t); break;
    case PH_SWEEP: consume_sweep(pl, t); break;
    case PH_FEAS: consume_feas(pl, t); break;
    case PH_NEWTON: consume_newton(pl, t); break;
    case PH_FINAL: consume_final(pl, t); break;
    case PH_GATHER: consume_gather(pl); break;
    default: break;
  }
  if (pl.res.passes > 4096 && pl.cmd.phase != PH_DONE) set_error(pl, ST_INTERNAL);
}

#if defined(__CUDACC__)
// Warp-parallel full-pivot LU + solve, the same algorithm and arithmetic as
// fullpiv_solve (Eigen::FullPivLU as used at projection.cpp:401-407): lane l
// holds the column-major entries l and l + 32 of the m x m matrix (m <= 8);
// the pivot search is a warp arg-max with the scalar scan's tie rule (first
// in column-major order, NaN never chosen), row / column swaps and the
// elimination read their operands with shuffles, and every entry gets the
// scalar code's operations in the scalar code's order.  The triangular solves
// (O(m^2), sequential) run on lane 0 from the factors written back.  All 32
// lanes call it; returns false if the matrix is not invertible.
__device__ __noinline__ bool fullpiv_solve_warp(int m, double* a, const double* b, double* x) {
  const int lane = threadIdx.x & 31;
  const unsigned F = 0xffffffffu;
  if (m > 8) {
    int ok = 0;
    if (lane == 0) ok = fullpiv_solve(m, a, b, x) ? 1 : 0;
    return __shfl_sync(F, ok, 0) != 0;
  }
  const int mm = m * m;
  const int x0 = lane, x1 = lane + 32;
  double e0 = x0 < mm ? a[x0] : 0.0, e1 = x1 < mm ? a[x1] : 0.0;
  const int r0 = x0 % m, c0 = x0 / m, r1 = x1 % m, c1 = x1 / m;
  auto fetch = [&](int idx) -> double {   // entry idx (lane-dependent) from its owner
    const double v0 = __shfl_sync(F, e0, idx & 31), v1 = __shfl_sync(F, e1, idx & 31);
    return idx < 32 ? v0 : v1;
  };
  unsigned rowperm = 0, colperm = 0;   // 4 bits per index
  for (int i = 0; i < m; ++i) { rowperm |= (unsigned)i << (4 * i); colperm |= (unsigned)i << (4 * i); }
  auto pswap = [](unsigned p, int u, int v) {
    const unsigned pu = (p >> (4 * u)) & 15u, pv = (p >> (4 * v)) & 15u;
    p &= ~((15u << (4 * u)) | (15u << (4 * v)));
    return p | (pv << (4 * u)) | (pu << (4 * v));
  };
  int nz = m;
  double maxpivot = 0.0;
  for (int k = 0; k < m; ++k) {
    double bv = -1.0;
    int bi = k * m + k;
    // this lane's candidates in scan order (x0 < x1), first strict max kept
    if (x0 < mm && r0 >= k && c0 >= k) { const double v = fabs(e0); if (v > bv) { bv = v; bi = x0; } }
    if (x1 < mm && r1 >= k && c1 >= k) { const double v = fabs(e1); if (v > bv) { bv = v; bi = x1; } }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(F, bv, o);
      const int oi = __shfl_xor_sync(F, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if (bv == 0.0) { nz = k; break; }
    if (bv > maxpivot) maxpivot = bv;
    const int br = bi % m, bc = bi / m;
    if (br != k) {   // swap rows k, br (all columns)
      const int s0 = c0 * m + (r0 == k ? br : (r0 == br ? k : r0));
      const int s1 = c1 * m + (r1 == k ? br : (r1 == br ? k : r1));
      const double n0 = fetch(s0 < mm ? s0 : 0), n1 = fetch(s1 < mm ? s1 : 0);
      if (x0 < mm) e0 = n0;
      if (x1 < mm) e1 = n1;
      rowperm = pswap(rowperm, k, br);
    }
    if (bc != k) {   // swap columns k, bc (all rows)
      const int s0 = (c0 == k ? bc : (c0 == bc ? k : c0)) * m + r0;
      const int s1 = (c1 == k ? bc : (c1 == bc ? k : c1)) * m + r1;
      const double n0 = fetch(s0 < mm ? s0 : 0), n1 = fetch(s1 < mm ? s1 : 0);
      if (x0 < mm) e0 = n0;
      if (x1 < mm) e1 = n1;
      colperm = pswap(colperm, k, bc);
    }
    const double piv = fetch(k * m + k);
    if (x0 < mm && c0 == k && r0 > k) e0 = e0 / piv;
    if (x1 < mm && c1 == k && r1 > k) e1 = e1 / piv;
    {   // A(i,j) = A(i,j) - A(i,k) * A(k,j) for i, j > k
      const double l0 = fetch(x0 < mm ? k * m + r0 : 0), u0 = fetch(x0 < mm ? c0 * m + k : 0);
      const double l1 = fetch(x1 < mm ? k * m + r1 : 0), u1 = fetch(x1 < mm ? c1 * m + k : 0);
      if (x0 < mm && r0 > k && c0 > k) e0 = e0 - l0 * u0;
      if (x1 < mm && r1 > k && c1 > k) e1 = e1 - l1 * u1;
    }
  }
  const double thr = fabs(maxpivot) * 2.220446049250313e-16 * (double)m;
  const bool d0 = x0 < mm && r0 == c0 && r0 < nz && fabs(e0) > thr;
  const bool d1 = x1 < mm && r1 == c1 && r1 < nz && fabs(e1) > thr;
  const int rank = __popc(__ballot_sync(F, d0)) + __popc(__ballot_sync(F, d1));
  if (rank != m) return false;
  if (x0 < mm) a[x0] = e0;
  if (x1 < mm) a[x1] = e1;
  __syncwarp();
  if (lane == 0) {
#define A_(i, j) a[(j) * m + (i)]
    double cv[8];
    for (int i = 0; i < m; ++i) cv[i] = b[(rowperm >> (4 * i)) & 15u];
    for (int i = 0; i < m; ++i) {
      double s2 = cv[i];
      for (int k = 0; k < i; ++k) s2 = s2 - A_(i, k) * cv[k];
      cv[i] = s2;
    }
    for (int i = nz - 1; i >= 0; --i) {
      double s2 = cv[i];
      for (int k = i + 1; k < nz; ++k) s2 = s2 - A_(i, k) * cv[k];
      cv[i] = s2 / A_(i, i);
    }
    for (int i = 0; i < m; ++i) x[(colperm >> (4 * i)) & 15u] = (i < nz) ? cv[i] : 0.0;
#undef A_
  }
  __syncwarp();
  return true;
}

// Warp-parallel candidate choice (same set as walk_candidates).  Lane 0
// walks the predicted path -- a bisection toward the estimate, where a level
// certified by (yL, yH) is skipped, a near-certain level only updates the
// certifier of its direction, and every other level is recorded with its
// branch probability.  The lanes then price the recorded nodes in parallel
// (prefix product), pick the MAX_HEDGE most probable first-level alternatives
// by warp arg-max, and merge path and hedges by probability with ballots.
constexpr int WPATH = 32;
struct WarpPath {
  double y[WPATH], lo[WPATH], hi[WPATH];
  int rt[WPATH];   // direction taken at the node (1: lo = ym)
  double cert_lo, cert_hi, clo, chi;
  int np, n0, has_cl, has_ch;
  RootEst e;
};

__device__ __noinline__ int walk_candidates_warp(const Walk& w, const ProjOptions& o, int K, double* out,
                                    WarpPath& wp) {
  const int lane = threadIdx.x & 31;
  if (lane == 0) {
    int n0 = 0;
    if (!w.feas_done) out[n0++] = w.up ? w.bp_hi : w.bp_lo;
    ctl_mark(2);
    const RootEst e = walk_estimate(w);
    ctl_mark(3);
    double clo, chi;
    walk_window(w, &clo, &chi);
    int np = 0, lev = 0;
    double lo = w.lo, hi = w.hi, ym = w.ym;
    int it = w.iters;
    const bool hasL = w.hasL, hasH = w.hasH;
    const double yL = w.yL, yH = w.yH;
    const int Kp = (K - n0 < WPATH) ? K - n0 : WPATH;
    double cert_lo = 0.0, cert_hi = 0.0;
    int has_cl = 0, has_ch = 0;
    // Direction = one comparison with the estimate's median (p_above >= 0.5);
    // the loop body is written branch-free so a level costs the ym chain
    // (compare, select, add, multiply), not three resolved branches.
    const double L2 = e.L - 33.0;
    const double thr = e.thr;                      // est_certain: |ym - ye| >= thr
    const bool k0 = e.kind == 0, k1 = e.kind == 1;
    const double ye = e.ye;
    const double tol_b = o.tol_b;
    const int maxit = o.binary_maxiter;
    if (k0) {   // point estimate: certain levels feed the certifiers
#pragma unroll 1
      while (np < Kp && lev < kMaxPathLevels && (hi - lo) > tol_b && it < maxit) {
        const bool cH = hasH && yH <= ym, cL = hasL && yL >= ym;
        const bool unc = !cH && !cL;
        const bool right = !cH && (cL || ym <= ye);
        const int lev1 = lev + (unc ? 1 : 0);
        const bool cert = unc && lev1 > 1 && fabs(ym - ye) >= thr;
        cert_lo = (cert && right) ? ym : cert_lo;
        cert_hi = (cert && !right) ? ym : cert_hi;
        has_cl |= (cert && right) ? 1 : 0;
        has_ch |= (cert && !right) ? 1 : 0;
        wp.y[np] = ym; wp.lo[np] = lo; wp.hi[np] = hi; wp.rt[np] = right;   // kept iff recorded
        np += (unc && !cert) ? 1 : 0;
        lev = lev1;
        lo = right ? ym : lo;
        hi = right ? hi : ym;
        ym = 0.5 * (lo + hi);
        ++it;
      }
    } else {    // log-uniform prior: every uncertain level is a path node
#pragma unroll 1
      while (np < Kp && lev < kMaxPathLevels && (hi - lo) > tol_b && it < maxit) {
        const bool cH = hasH && yH <= ym, cL = hasL && yL >= ym;
        const bool unc = !cH && !cL;
        const double lg = approx_log2(fabs(ym));
        const bool right = !cH && (cL || (k1 ? (lg >= L2) : (lg <= L2)));
        wp.y[np] = ym; wp.lo[np] = lo; wp.hi[np] = hi; wp.rt[np] = right;
        np += unc ? 1 : 0;
        lev += unc ? 1 : 0;
        lo = right ? ym : lo;
        hi = right ? hi : ym;
        ym = 0.5 * (lo + hi);
        ++it;
      }
    }
    if (has_cl && n0 < K) out[n0++] = cert_lo;
    if (has_ch && n0 < K) out[n0++] = cert_hi;
    wp.e = e;
    wp.np = np;
    wp.n0 = n0;
    wp.clo = clo;
    wp.chi = chi;
    ctl_mark(4);
  }
  __syncwarp();
  const int np = wp.np, n0 = wp.n0;
  const double clo = wp.clo, chi = wp.chi;
  // level k = lane: branch probability, path probability, hedge
  double q = 1.0, ym = 0.0, alt = 0.0;
  if (lane < np) {
    ym = wp.y[lane];
    const double pa = est_p_above(wp.e, ym);
    const bool right = wp.rt[lane] != 0;
    q = right ? pa : 1.0 - pa;
    alt = right ? 0.5 * (wp.lo[lane] + ym) : 0.5 * (ym + wp.hi[lane]);
  }
  // P_k = prod_{i<k} q_i (exclusive prefix product; the scalar version
  // multiplies in the same left-to-right order for k <= 1 and by a fixed tree
  // after that -- only the ranking uses it)
  double P = q;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const double v = __shfl_up_sync(0xffffffffu, P, off);
    if (lane >= off) P = P * v;
  }
  double pp = __shfl_up_sync(0xffffffffu, P, 1);
  if (lane == 0) pp = 1.0;
  if (lane == 0) ctl_mark(8);
  const double hp = pp * (1.0 - q);
  bool elig = lane < np && hp > 1e-12 && alt > clo && alt < chi;
  // the MAX_HEDGE most probable hedges, descending (ties: lower level first):
  // one integer max-reduction per pick on a 32-bit key = the top 27 bits of
  // the (positive) float probability above the complemented lane index
  double hv[MAX_HEDGE], hy[MAX_HEDGE];
  int nh = 0;
  const unsigned key = elig ? (((__float_as_uint((float)hp) >> 5) << 5) | (31u - (unsigned)lane))
                            : 0u;   // hp > 1e-12, so an eligible key is >= 32
#pragma unroll
  for (int r = 0; r < MAX_HEDGE; ++r) {
    const unsigned active = __ballot_sync(0xffffffffu, elig);
    hv[r] = -1.0; hy[r] = 0.0;
    if (active) {
      const unsigned best = __reduce_max_sync(0xffffffffu, elig ? key : 0u);
      const int src = 31 - (int)(best & 31u);
      hv[r] = __shfl_sync(0xffffffffu, hp, src);
      hy[r] = __shfl_sync(0xffffffffu, alt, src);
      if (lane == src) elig = false;
      ++nh;
    }
  }
  if (lane == 0) ctl_mark(9);
  // merge: path node k goes to k + #{hedges > pp_k}; hedge r to
  // r + #{path nodes with pp >= h_r}; keep the first `room` positions
  const int room = K - n0;
  int taken = 0;
  if (lane < np) {
    int pos = lane;
#pragma unroll
    for (int r = 0; r < MAX_HEDGE; ++r) pos += (r < nh && hv[r] > pp) ? 1 : 0;
    if (pos < room) out[n0 + pos] = ym;
  }
#pragma unroll
  for (int r = 0; r < MAX_HEDGE; ++r) {
    if (r < nh) {
      const unsigned ge = __ballot_sync(0xffffffffu, lane < np && pp >= hv[r]);
      const int pos = r + __popc(ge);
      if (lane == 0 && pos < room) out[n0 + pos] = hy[r];
    }
  }
  taken = np + nh < room ? np + nh : room;
  __syncwarp();
  if (lane == 0) ctl_mark(10);
  return n0 + taken;
}

// Warp version of schedule_sweep (same command layout).
// Candidates of row j, ascending (rank sort, ties by index), into out[];
// returns their count.  One warp.
__device__ __noinline__ int schedule_row_warp(Plan& pl, int j, int per, double* out,
                                              WarpPath& wp) {
  const int lane = threadIdx.x & 31;
  const Walk& w = pl.w[j];   // shared memory (a copy would live in local memory)
  const int nc = walk_candidates_warp(w, pl.P.opt, per, out, wp);
  const double v = lane < nc ? out[lane] : 0.0;
  int rk = 0;
  for (int q = 0; q < nc; ++q) {
    const double u = __shfl_sync(0xffffffffu, v, q);
    rk += (u < v || (u == v && q < lane)) ? 1 : 0;
  }
  __syncwarp();
  if (lane < nc) out[rk] = v;
  __syncwarp();
  if (lane == 0) ctl_mark(11);
  return nc;
}


// The sweep command around the candidates already in cmd.cand_y (lane 0).
TOPT_HDN inline void schedule_finish(Plan& pl, int tot) {
  Cmd& c = pl.cmd;
  const int m = pl.P.m;
  c.phase = PH_SWEEP;
  for (int j = m; j <= MAX_M; ++j) c.row_start[j] = tot;
  // the first global sweep of a job classifies nothing away (its window is
  // the whole bracket): it runs the plain full sweep with the queued fast
  // path; the active lists start with the second
  c.compact = (pl.P.compact_cap > 0 && (m == 1 || pl.P.has_part) &&
               (c.local || pl.res.sweeps > 0)) ? 1 : 0;
  for (int j = 0; j < m; ++j) walk_window(pl.w[j], &c.wlo[j], &c.whi[j]);
  c.ncand = tot;
  c.nslots = 2 * tot + ((c.compact && !c.local) ? 2 : 0);
  if (c.local) pl.res.local_sweeps++; else pl.res.sweeps++;
  sketch_command(pl);
}

__device__ __noinline__ bool schedule_sweep_warp(Plan& pl, WarpPath& wp) {
  const int lane = threadIdx.x & 31;
  const int m = pl.P.m;
  {
    __shared__ int s_ex;
    if (lane == 0) s_ex = schedule_exact_walks(pl) ? 1 : 0;
    __syncwarp();
    if (s_ex) return true;
  }
  int need = 0;
  for (int j = 0; j < m; ++j) need += (pl.w[j].status == WK_NEED);
  if (!need) return false;
  const int per = schedule_per(pl, need);
  Cmd& c = pl.cmd;
  int tot = 0;
  for (int j = 0; j < m; ++j) {
    if (lane == 0) c.row_start[j] = tot;
    if (pl.w[j].status == WK_NEED) tot += schedule_row_warp(pl, j, per, c.cand_y + tot, wp);
  }
  __syncwarp();
  if (lane == 0) schedule_finish(pl, tot);
  __syncwarp();
  return true;
}

// Warp-parallel version of consume_sweep (all 32 lanes of one warp): lane k
// holds candidate k; bracket updates are warp arg-reductions and each
// replayed midpoint is matched with one ballot.  Same decisions as the
// scalar consume_sweep (candidates are distinct duals).
// Ingest + replay of row j's evaluations (one warp): lane k holds candidate
// k; bracket updates are warp arg-reductions and each replayed midpoint is
// matched with one ballot.
__device__ __noinline__ void consume_sweep_row_warp(Plan& pl, const double* t, int j) {
  const int lane = threadIdx.x & 31;
  Cmd& c = pl.cmd;
  {
    const int b = c.row_start[j], e = c.row_start[j + 1], nc = e - b;
    if (nc <= 0) return;
    Walk w = pl.w[j];
    // lane k holds candidate k; the row's candidates are ascending, so the
    // nearest qualifying point below (above) is the highest (lowest) lane
    const bool mine = lane < nc;
    const double cy = mine ? c.cand_y[b + lane] : 0.0;
    const double cR = mine ? t[2 * (b + lane)] - w.ghat : 0.0;
    const double cS = mine ? t[2 * (b + lane) + 1] : 0.0;
    const double E = w.E;
    const unsigned mA = __ballot_sync(0xffffffffu, mine && cR <= 0.0);
    const unsigned mB = __ballot_sync(0xffffffffu, mine && cR > 0.0);
    const unsigned mL = __ballot_sync(0xffffffffu, mine && cR < -E);
    const unsigned mH = __ballot_sync(0xffffffffu, mine && cR > E);
    const unsigned mNear = __ballot_sync(0xffffffffu, mine && fabs(cR) <= E);
    const int sA = mA ? 31 - __clz(mA) : 0, sB = mB ? __ffs(mB) - 1 : 0;
    const int sL = mL ? 31 - __clz(mL) : 0, sH = mH ? __ffs(mH) - 1 : 0;
    const double yA = __shfl_sync(0xffffffffu, cy, sA), RA = __shfl_sync(0xffffffffu, cR, sA);
    const double SA = __shfl_sync(0xffffffffu, cS, sA);
    const double yB = __shfl_sync(0xffffffffu, cy, sB), RB = __shfl_sync(0xffffffffu, cR, sB);
    const double SB = __shfl_sync(0xffffffffu, cS, sB);
    const double yLc = __shfl_sync(0xffffffffu, cy, sL), yHc = __shfl_sync(0xffffffffu, cy, sH);
    if (mA && (!w.hasA || yA > w.ya)) { w.hasA = 1; w.ya = yA; w.Ra = RA; w.Sa = SA; }
    if (mB && (!w.hasB || yB < w.yb)) { w.hasB = 1; w.yb = yB; w.Rb = RB; w.Sb = SB; }
    if (mL && (!w.hasL || yLc > w.yL)) { w.hasL = 1; w.yL = yLc; }
    if (mH && (!w.hasH || yHc < w.yH)) { w.hasH = 1; w.yH = yHc; }
    if (lane == 0) ctl_mark(0);
    // replay (every lane runs the same loop; a lookup is one ballot)
    if (w.status == WK_NEED) {
      const bool strict = pl.P.strict != 0;
      const bool hasL = w.hasL, hasH = w.hasH, hasL0 = w.hasL0;
      const double yL = w.yL, yH = w.yH, yL0 = w.yL0;
      unsigned used = 0u;   // lanes whose value decided a level directly
      bool stop = false;
      if (!w.feas_done) {
        const double yb = w.up ? w.bp_hi : w.bp_lo;
        const unsigned hit = __ballot_sync(0xffffffffu, mine && cy == yb);
        int infeasible = -1;
        // certificates first (proofs), then a direct evaluation
        if (hasH && yH <= yb) {
          infeasible = w.up ? 0 : 1;
        } else if (hasL && yL >= yb) {
          infeasible = w.up ? 1 : 0;
        } else if (hasL0 && (w.up ? yL0 == yb : yL0 >= yb)) {
          infeasible = 0;
        } else if (hit) {
          // projection.cpp:80-94: R < 0 (up) / R > 0 (down) => infeasible
          const double R = __shfl_sync(0xffffffffu, cR, __ffs(hit) - 1);
          if (strict && fabs(R) <= E) {
            w.status = WK_EXACT; w.ex_state = 1; w.ex_y = yb;
            stop = true;
          } else {
            infeasible = w.up ? (R < 0.0) : (R > 0.0);
            used |= hit;
          }
        }
        if (stop) {}
        else if (infeasible < 0) { stop = true; }
        else if (infeasible) { w.status = WK_INFEASIBLE; stop = true; }
        else w.feas_done = 1;
      }
      int direct = 0;
      if (!stop) {
        double lo = w.lo, hi = w.hi, ym = w.ym;
        int it = w.iters;
        const double tol_b = pl.P.opt.tol_b;
        const int maxit = pl.P.opt.binary_maxiter;
        int status = WK_DONE;
#pragma unroll 1
        while ((hi - lo) > tol_b && it < maxit) {
          const bool cH = hasH && yH <= ym;
          const bool cL = (hasL && yL >= ym) || (hasL0 && yL0 >= ym);
          const unsigned hit = __ballot_sync(0xffffffffu, mine && cy == ym);
          const bool unc = !cH && !cL;
          if (unc && !hit) { status = WK_NEED; break; }
          if (unc && strict && (hit & mNear) != 0u) {   // within the bound: reference order
            status = WK_EXACT; w.ex_state = 1; w.ex_y = ym;
            break;
          }
          used |= unc ? hit : 0u;
          direct += unc ? 1 : 0;
          const bool up = cH || (unc && (hit & mB) != 0u);   // evaluated: R > 0.0
          hi = up ? ym : hi;
          lo = up ? lo : ym;
          ym = 0.5 * (lo + hi);
          ++it;
        }
        w.lo = lo; w.hi = hi; w.ym = ym; w.iters = it;
        w.status = status;
        if (status == WK_DONE) w.y = ym;
      }
      // diagnostics over the directly used evaluations
      w.near_ties += __popc(used & mNear);
      w.n_direct += direct;
      if (used) {
        double mm = ((used >> lane) & 1u) ? fabs(cR) / E : 1e300;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) mm = dmin_(mm, __shfl_xor_sync(0xffffffffu, mm, off));
        w.min_margin = dmin_(w.min_margin, mm);
      }
    }
    __syncwarp();
    if (lane == 0) pl.w[j] = w;
    __syncwarp();
  }
}

__device__ __noinline__ void consume_sweep_warp(Plan& pl, const double* t) {
  const int lane = threadIdx.x & 31;
  const int m = pl.P.m;
  Cmd& c = pl.cmd;
  __shared__ WarpPath s_wpk;
  if (__shfl_sync(0xffffffffu, (int)c.sample, 0)) {   // a sketch (see consume_sketch)
    if (lane == 0) {
      pl.res.passes++;
      consume_sketch(pl, t);
    }
    __syncwarp();
    const bool more = schedule_sweep_warp(pl, s_wpk);
    if (lane == 0 && !more) after_walks(pl);
    __syncwarp();
    return;
  }
  const bool was_global_compact = c.compact && !c.local;
  for (int j = 0; j < m; ++j) consume_sweep_row_warp(pl, t, j);
  __shared__ WarpPath s_wp;
  __shared__ int s_act;
  if (lane == 0) {
    ctl_mark(1);
    if (was_global_compact) pl.res.active = t[2 * c.ncand];
    pl.res.passes++;
    int need = 0;
    for (int j = 0; j < m; ++j) need += (pl.w[j].status == WK_NEED);
    s_act = 0;
    if (need && was_global_compact && pl.res.active <= (double)GATHER_TRIGGER) {
      if (t[2 * c.ncand + 1] == 0.0) {   // every CTA published its items (fused gather)
        c.local = 1;
        c.load_fused = 1;
        pl.res.gathered = 1;
        s_act = 1;
      } else {
        c.phase = PH_GATHER;
        c.nslots = 0;
      }
    } else {
      s_act = 1;
    }
  }
  __syncwarp();
  if (s_act) {
    const bool more = schedule_sweep_warp(pl, s_wp);
    if (lane == 0) ctl_mark(6);
    if (lane == 0 && !more) after_walks(pl);
  }
  if (lane == 0) ctl_mark(7);
  if (lane == 0 && pl.res.passes > 4096 && pl.cmd.phase != PH_DONE) set_error(pl, ST_INTERNAL);
  __syncwarp();
}

// Called by all lanes of one warp.
__device__ void plan_consume_warp(Plan& pl, const double* t) {
  const int lane = threadIdx.x & 31;
  __shared__ WarpPath s_wp2;
  // One phase value for the whole warp, taken before any lane goes on: lane 0
  // rewrites cmd.phase below, and a lane that read it late took a different
  // branch to a different __syncwarp (hang seen with the very short m = 0
  // PREP step of JOB_DIRECTION).
  __syncwarp();
  const int ph = __shfl_sync(0xffffffffu, (int)pl.cmd.phase, 0);
  if (ph == PH_SWEEP) {
    consume_sweep_warp(pl, t);
    return;
  }
  if (ph == PH_PREP || ph == PH_GATHER) {
    if (lane == 0) {
      pl.res.passes++;
      ctl_mark(0);
      if (ph == PH_PREP && prep_needs_exact(pl)) {
        schedule_exact_ghat(pl, t);
      } else if (ph == PH_PREP) {
        consume_prep_core(pl, t);
        ctl_mark(1);
      } else {
        pl.cmd.local = 1;
        pl.res.gathered = 1;
        pl.cmd.phase = PH_SWEEP;
        pl.cmd.nslots = -1;
      }
    }
    __syncwarp();
    if (pl.cmd.phase == PH_SWEEP && pl.cmd.nslots == -1) {
      const bool more = schedule_sweep_warp(pl, s_wp2);
      if (lane == 0) ctl_mark(6);
      if (lane == 0 && !more) after_walks(pl);
    }
    if (lane == 0) ctl_mark(7);
    __syncwarp();
    return;
  }
  if (ph == PH_NEWTON || (ph == PH_EXACT && pl.cmd.ex_what == EXW_NEWTON)) {
    // the m x m solve on the whole warp
    __shared__ int s_pend;
    if (lane == 0) {
      pl.res.passes++;
      if (ph == PH_EXACT) pl.res.exact_passes++;
      s_pend = consume_newton_core(pl, t);
    }
    __syncwarp();
    if (s_pend) {
      const bool ok = fullpiv_solve_warp(pl.P.m, pl.sc.jp, pl.nt.phi, pl.nt.step);
      if (lane == 0) finish_newton_post(pl, ok);
    }
    if (lane == 0 && pl.res.passes > 4096 && pl.cmd.phase != PH_DONE) set_error(pl, ST_INTERNAL);
    __syncwarp();
    return;
  }
  if (lane == 0) plan_consume(pl, t);
  __syncwarp();
}

// CTA-level controller step (all threads of the CTA call it).  With several
// rows (stage-1 walks, independent partitions), the per-row work of a sweep
// step -- ingest + replay, then candidate choice -- runs on warp j for row j;
// warp 0 does the bookkeeping in between and concatenates the rows'
// candidates in row order, so the command is the same as the one-warp
// controller's.  Everything else is plan_consume_warp on warp 0.
__device__ __noinline__ void plan_consume_cta(Plan& pl, const double* t) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int m = pl.P.m;
  const int ph = pl.cmd.phase;
  const bool sketch = ph == PH_SWEEP && pl.cmd.sample != 0;
  __syncthreads();   // every thread has the phase before warp 0 may rewrite it
  const bool multi = m > 1 && m <= (int)(blockDim.x >> 5) && (ph == PH_SWEEP || ph == PH_PREP);
  if (!multi) {
    if (warp == 0) plan_consume_warp(pl, t);
    __syncthreads();
    return;
  }
  __shared__ int s_sched;
  __shared__ int s_nc[MAX_M];
  __shared__ double s_cand[MAX_M * MAX_K];
  __shared__ WarpPath s_wpr[MAX_M];
  Cmd& c = pl.cmd;
  if (sketch) {   // steer the candidates, decide nothing (consume_sketch)
    if (threadIdx.x == 0) {
      pl.res.passes++;
      consume_sketch(pl, t);
      s_sched = 1;
    }
  } else if (ph == PH_SWEEP) {
    const bool was_global_compact = c.compact && !c.local;
    if (warp < m) consume_sweep_row_warp(pl, t, warp);
    __syncthreads();
    if (threadIdx.x == 0) {
      ctl_mark(1);
      if (was_global_compact) pl.res.active = t[2 * c.ncand];
      pl.res.passes++;
      int need = 0;
      for (int j = 0; j < m; ++j) need += (pl.w[j].status == WK_NEED);
      s_sched = 1;
      if (need && was_global_compact && pl.res.active <= (double)GATHER_TRIGGER) {
        if (t[2 * c.ncand + 1] == 0.0) {   // fused gather
          c.local = 1;
          c.load_fused = 1;
          pl.res.gathered = 1;
        } else {
          c.phase = PH_GATHER;
          c.nslots = 0;
          s_sched = 0;
        }
      }
    }
  } else {   // PH_PREP
    if (threadIdx.x == 0) {
      pl.res.passes++;
      ctl_mark(0);
      if (prep_needs_exact(pl)) schedule_exact_ghat(pl, t);
      else consume_prep_core(pl, t);
      ctl_mark(1);
      s_sched = (pl.cmd.phase == PH_SWEEP && pl.cmd.nslots == -1) ? 1 : 0;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && s_sched && schedule_exact_walks(pl)) s_sched = 0;
  __syncthreads();
  if (s_sched) {
    int need = 0;
    for (int j = 0; j < m; ++j) need += (pl.w[j].status == WK_NEED);
    if (need) {
      const int per = schedule_per(pl, need);
      if (warp < m) {
        const int nc = pl.w[warp].status == WK_NEED
                           ? schedule_row_warp(pl, warp, per, s_cand + warp * MAX_K, s_wpr[warp])
                           : 0;
        if (lane == 0) s_nc[warp] = nc;
      }
      __syncthreads();
      if (warp == 0) {   // concatenate in row order (the one-warp layout)
        int tot = 0;
        for (int j = 0; j < m; ++j) {
          if (lane == 0) c.row_start[j] = tot;
          if (lane < s_nc[j]) c.cand_y[tot + lane] = s_cand[j * MAX_K + lane];
          tot += s_nc[j];
        }
        __syncwarp();
        if (lane == 0) schedule_finish(pl, tot);
      }
    } else if (threadIdx.x == 0) {
      after_walks(pl);
    }
  }
  if (threadIdx.x == 0) {
    ctl_mark(7);
    if (pl.res.passes > 4096 && pl.cmd.phase != PH_DONE) set_error(pl, ST_INTERNAL);
  }
  __syncthreads();
}
#endif

}  // namespace topt_b200
