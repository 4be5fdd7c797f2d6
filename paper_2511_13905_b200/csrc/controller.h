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

#include "topt_core.h"

namespace topt_b200 {

constexpr double kUnit = 1.1102230246251565e-16;  // 2^-53
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
  PREP_SLOTS = 9
};

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
TOPT_HDN inline bool fullpiv_solve(int m, double* a, const double* b, double* x) {
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

// Exact evaluation lookup among this sweep's candidates.
TOPT_HD bool walk_lookup(const Walk& w, double y, double* R) {
  int hit = -1;
#pragma unroll
  for (int k = 0; k < MAX_K; ++k)
    if (k < w.nc && w.cy[k] == y) hit = k;
  if (hit < 0) return false;
  *R = w.cR[hit];
  return true;
}

// +1: reference sees r(y) > 0 ; -1: reference sees r(y) <= 0 ; 0: unknown.
TOPT_HDN inline int walk_decide(Walk& w, double y, bool record) {
  double R;
  if (walk_lookup(w, y, &R)) {
    if (record) {
      const double mg = fabs(R) / w.E;
      if (mg < w.min_margin) w.min_margin = mg;
      if (fabs(R) <= w.E) w.near_ties++;
      w.n_direct++;
    }
    return R > 0.0 ? 1 : -1;
  }
  if (w.hasH && w.yH <= y) return 1;
  if (w.hasL && w.yL >= y) return -1;
  return 0;
}

// Replay the reference walk as far as evaluations/certificates allow.
TOPT_HDN inline void walk_advance(Walk& w, const ProjOptions& o) {
  if (w.status == WK_DONE || w.status == WK_INFEASIBLE || w.status == WK_IDLE) return;
  if (!w.feas_done) {
    // projection.cpp:80-94: r(y_lo) > 0 (down) / r(y_hi) < 0 (up) => infeasible
    const double yb = w.up ? w.bp_hi : w.bp_lo;
    double R;
    int infeasible;
    if (walk_lookup(w, yb, &R)) {
      infeasible = w.up ? (R < 0.0) : (R > 0.0);
      const double mg = fabs(R) / w.E;
      if (mg < w.min_margin) w.min_margin = mg;
      if (fabs(R) <= w.E) w.near_ties++;
    } else if (w.hasH && w.yH <= yb) {
      infeasible = w.up ? 0 : 1;
    } else if (w.hasL && w.yL >= yb) {
      infeasible = w.up ? 1 : 0;
    } else {
      w.status = WK_NEED;
      return;
    }
    if (infeasible) { w.status = WK_INFEASIBLE; return; }
    w.feas_done = 1;
  }
  while ((w.hi - w.lo) > o.tol_b && w.iters < o.binary_maxiter) {
    const int d = walk_decide(w, w.ym, true);
    if (d == 0) { w.status = WK_NEED; return; }
    if (d > 0) w.hi = w.ym; else w.lo = w.ym;
    w.ym = 0.5 * (w.lo + w.hi);
    ++w.iters;
  }
  w.status = WK_DONE;
  w.y = w.ym;
}

// Root estimate used to choose speculative midpoints (never a decision).
struct RootEst {
  int kind;        // 0: gaussian(ye, sig) ; 1: log-uniform prior below 0 ; 2: above 0
  double ye, sig, L;
};

TOPT_HDN inline RootEst walk_estimate(const Walk& w) {
  RootEst e;
  e.kind = 0; e.ye = 0.0; e.sig = 1.0; e.L = 0.0;
  if (w.hasA && w.hasB && w.ya < w.yb) {
    const double ya = w.ya, yb = w.yb;
    double sec = ya - w.Ra * (yb - ya) / (w.Rb - w.Ra);
    if (!(sec >= ya)) sec = ya;
    if (!(sec <= yb)) sec = yb;
    double spread = 0.0;
    if (w.Sa > 0.0) {
      const double t = dmin_(dmax_(ya - w.Ra / w.Sa, ya), yb);
      spread = dmax_(spread, fabs(t - sec));
    }
    if (w.Sb > 0.0) {
      const double t = dmin_(dmax_(yb - w.Rb / w.Sb, ya), yb);
      spread = dmax_(spread, fabs(t - sec));
    }
    double sig = dmax_(spread, (yb - ya) * 1e-6);
    sig = dmax_(sig, fabs(sec) * 1e-15);
    e.ye = sec;
    e.sig = dmax_(sig, 1e-300);
    return e;
  }
  if (!w.up) {  // root in [bp_lo, 0], r(0) > 0 known
    if (w.hasB && w.Sb > 0.0) {
      e.ye = dmax_(w.yb - w.Rb / w.Sb, w.lo);
      e.sig = dmax_(0.5 * fabs(e.ye), 1e-300);
      return e;
    }
    e.kind = 1;
    e.L = log(fabs(w.lo) + 1e-300);
    return e;
  }
  if (w.hasA && w.Sa > 0.0) {  // root in [0, bp_hi], r(0) < 0 known
    e.ye = dmin_(w.ya - w.Ra / w.Sa, w.hi);
    e.sig = dmax_(0.5 * fabs(e.ye), 1e-300);
    return e;
  }
  e.kind = 2;
  e.L = log(fabs(w.hi) + 1e-300);
  return e;
}

// Probability that the root lies above y.
TOPT_HDN inline double est_p_above(const RootEst& e, double y) {
  if (e.kind == 0) return 0.5 * erfc((y - e.ye) / (e.sig * 1.4142135623730951));
  const double ay = fabs(y);
  if (!(ay > 0.0)) return e.kind == 1 ? 0.0 : 1.0;
  double p = (log(ay) - (e.L - 46.0)) / 46.0;  // P(|root| < |y|), log-uniform prior
  p = dmin_(dmax_(p, 0.0), 1.0);
  return e.kind == 1 ? p : 1.0 - p;
}

// Choose up to K midpoints of the walk's remaining decision tree to evaluate
// next: the predicted path (most probable branch at every uncertain level),
// plus first-level alternatives ("hedges") of its least certain levels,
// ranked by the probability of being visited.  O(K + certain levels).
TOPT_HDN inline int walk_candidates(const Walk& w, const ProjOptions& o, int K, double* out,
                                    Scratch& scr) {
  int n = 0;
  if (w.status != WK_NEED || K <= 0) return 0;
  if (!w.feas_done) out[n++] = w.up ? w.bp_hi : w.bp_lo;
  const RootEst e = walk_estimate(w);
  double* pp = scr.np;    // path node probability
  double* py = scr.nlo;   // path node y
  double* hp = scr.nhi;   // hedge probability
  double* hy = scr.nym;   // hedge y
  int np = 0, nh = 0;
  double lo = w.lo, hi = w.hi, ym = w.ym, p = 1.0;
  int it = w.iters;
  while (np < K && (hi - lo) > o.tol_b && it < o.binary_maxiter) {
    int d = 0;
    if (w.hasH && w.yH <= ym) d = 1;
    else if (w.hasL && w.yL >= ym) d = -1;
    if (d == 0) {
      const double pa = est_p_above(e, ym);   // root above ym -> r(ym) <= 0 -> lo = ym
      const bool right = pa >= 0.5;
      py[np] = ym; pp[np] = p; ++np;
      const double palt = right ? 1.0 - pa : pa;
      if (palt > 1e-12 && nh < CAND_CAP) {
        hy[nh] = right ? 0.5 * (lo + ym) : 0.5 * (ym + hi);
        hp[nh] = p * palt;
        ++nh;
      }
      p = p * (right ? pa : 1.0 - pa);
      if (right) lo = ym; else hi = ym;
    } else {
      if (d > 0) hi = ym; else lo = ym;
    }
    ym = 0.5 * (lo + hi);
    ++it;
  }
  // merge: path nodes are a prefix ordered by decreasing probability; take
  // hedges greedily when more probable than the next path node.
  int ip = 0;
  while (n < K && (ip < np || nh > 0)) {
    int bh = -1;
    for (int k = 0; k < nh; ++k)
      if (bh < 0 || hp[k] > hp[bh]) bh = k;
    if (ip < np && (bh < 0 || pp[ip] >= hp[bh])) {
      out[n++] = py[ip++];
    } else {
      // a hedge is useless if its parent path node will not be evaluated; its
      // parent was evaluated iff it was taken (parents precede in pp order).
      out[n++] = hy[bh];
      hy[bh] = hy[nh - 1]; hp[bh] = hp[nh - 1]; --nh;
    }
  }
  return n;
}

// Record one evaluation R^(y) (already offset by -ghat) with slope S.
TOPT_HD void walk_add_point(Walk& w, double y, double R, double S) {
  if (w.nc < MAX_K) { w.cy[w.nc] = y; w.cR[w.nc] = R; w.cS[w.nc] = S; ++w.nc; }
  if (R <= 0.0 && (!w.hasA || y > w.ya)) { w.hasA = 1; w.ya = y; w.Ra = R; w.Sa = S; }
  if (R > 0.0 && (!w.hasB || y < w.yb)) { w.hasB = 1; w.yb = y; w.Rb = R; w.Sb = S; }
  if (R < -w.E && (!w.hasL || y > w.yL)) { w.hasL = 1; w.yL = y; }
  if (R > w.E && (!w.hasH || y < w.yH)) { w.hasH = 1; w.yH = y; }
}

// Initialise a walk from the PREP totals (projection.cpp:53-97).
TOPT_HDN inline void walk_init(Walk& w, int eq, double ghat, double E, double r0, double S0,
                               double bp_lo, double bp_hi, double any, double count) {
  Walk z = {};
  w = z;
  w.eq = eq; w.ghat = ghat; w.E = E; w.r0 = r0; w.S0 = S0;
  w.bp_lo = bp_lo; w.bp_hi = bp_hi; w.count = count;
  w.min_margin = 1e300;
  if (!eq && r0 <= 0.0) {             // inactive: y = 0, residual = max(r0, 0)
    w.status = WK_DONE; w.y = 0.0; w.residual = dmax_(r0, 0.0);
    if (fabs(r0) <= E) { w.near_ties++; }
    w.min_margin = fabs(r0) / E;
    return;
  }
  if (eq && r0 == 0.0) { w.status = WK_DONE; w.y = 0.0; w.residual = 0.0; return; }
  if (!(any > 0.0)) { w.status = WK_INFEASIBLE; return; }
  if (r0 > 0.0) {
    w.up = 0; w.lo = bp_lo; w.hi = 0.0;
    w.hasB = 1; w.yb = 0.0; w.Rb = r0; w.Sb = S0;
    if (r0 > E) { w.hasH = 1; w.yH = 0.0; }
  } else {
    w.up = 1; w.lo = 0.0; w.hi = bp_hi;
    w.hasA = 1; w.ya = 0.0; w.Ra = r0; w.Sa = S0;
    if (r0 < -E) { w.hasL = 1; w.yL = 0.0; }
  }
  w.ym = 0.5 * (w.lo + w.hi);
  w.iters = 0;
  w.status = WK_NEED;
  w.residual = -1.0;   // filled by the FINAL pass (|r(ym)|)
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

TOPT_HDN inline void cmd_final(Plan& pl, const double* y, int resid_rows) {
  Cmd& c = pl.cmd;
  c.phase = PH_FINAL;
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
  c.phase = PH_NEWTON;
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

// Build the next sweep over all walks that need evaluations; if none do,
// advance the stage.  Returns true if a sweep was scheduled.
TOPT_HDN inline bool schedule_sweep(Plan& pl) {
  const int m = pl.P.m;
  int need = 0;
  for (int j = 0; j < m; ++j) need += (pl.w[j].status == WK_NEED);
  if (!need) return false;
  int per = MAX_CAND / need;
  if (per > MAX_K) per = MAX_K;
  Cmd& c = pl.cmd;
  c.phase = PH_SWEEP;
  int tot = 0;
  for (int j = 0; j < m; ++j) {
    c.row_start[j] = tot;
    Walk& w = pl.w[j];
    w.nc = 0;
    if (w.status == WK_NEED) tot += walk_candidates(w, pl.P.opt, per, c.cand_y + tot, pl.sc);
  }
  for (int j = m; j <= MAX_M; ++j) c.row_start[j] = tot;
  c.ncand = tot;
  c.nslots = 2 * tot;
  pl.res.sweeps++;
  return true;
}

TOPT_HDN inline void after_walks(Plan& pl);

TOPT_HDN inline void finish_newton_or_loop(Plan& pl) {
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
    if (!fullpiv_solve(m, jp, nt.phi, nt.step)) { set_error(pl, ST_NUMERICAL); return; }
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
    return;
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
}

TOPT_HDN inline void consume_newton(Plan& pl, const double* t) {
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
    finish_newton_or_loop(pl);
    return;
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
    finish_newton_or_loop(pl);
    return;
  }
  nt.gamma = nt.gamma * 0.5;
  for (int j = 0; j < m; ++j) nt.ty[j] = nt.y[j] - nt.gamma * nt.step[j];
  cmd_newton(pl);
}

// Stage-1 feasibility (projection.cpp:320-342) over every row whose bisection
// succeeded, evaluated in one pass; first feasible row by index wins.
TOPT_HDN inline void schedule_feas(Plan& pl) {
  const int m = pl.P.m;
  Cmd& c = pl.cmd;
  c.phase = PH_FEAS;
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
  pl.stage = SG_FEAS;
  if (nf == 0) start_newton(pl);
}

TOPT_HDN inline void consume_feas(Plan& pl, const double* t) {
  const Problem& P = pl.P;
  const int m = P.m;
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
  start_newton(pl);
}

TOPT_HDN inline void after_walks(Plan& pl) {
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
TOPT_HDN inline void consume_prep(Plan& pl, const double* t) {
  Problem& P = pl.P;
  const int m = P.m;
  Result& r = pl.res;
  for (int j = 0; j < m; ++j) {
    const double* s = t + j * PREP_SLOTS;
    double ghat, gerr;
    const double cnt = P.row_count[j];
    const double ours = P.ours_len;
    if (pl.dot_mode) {  // projection.cpp:139-145: (G - g) + dot
      ghat = P.G_minus_g[j] + s[PS_DOT];
      gerr = (gamma_k((double)P.n_global + 2.0) + gamma_k(ours)) * s[PS_DABS] +
             2.0 * kUnit * fabs(ghat);
    } else {
      ghat = P.ghat_in[j];
      gerr = P.ghat_err_in[j];
      if (pl.cmd.validate_part && P.gd_step) {  // validate(): 1e-14 consistency
        const double expect = P.G_minus_g[j] + s[PS_DOT];
        const double scale = dmax_(dmax_(1.0, fabs(expect)), fabs(ghat));
        if (fabs(ghat - expect) > 1e-14 * scale) { set_error(pl, ST_DOMAIN); return; }
      }
    }
    r.ghat[j] = ghat;
    r.ghat_err[j] = (gamma_k((double)P.n_global + 2.0) + gamma_k(ours)) * s[PS_DABS];
    if (pl.cmd.validate_part && s[PS_NZOUT] > 0.0) { set_error(pl, ST_DOMAIN); return; }
    const double E = 1.0625 * (gamma_k(cnt + 2.0) * (fabs(ghat) + s[PS_T]) + gerr +
                               gamma_k(ours) * (fabs(ghat) + s[PS_T])) + 1e-300;
    const double r0 = s[PS_S0] - ghat;
    walk_init(pl.w[j], P.is_eq[j], ghat, E, r0, s[PS_SLOPE0], s[PS_BPLO], s[PS_BPHI],
              s[PS_ANY], cnt);
  }
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
  for (int j = 0; j < m; ++j) walk_advance(pl.w[j], P.opt);
  if (!schedule_sweep(pl)) after_walks(pl);
}

TOPT_HDN inline void consume_sweep(Plan& pl, const double* t) {
  const int m = pl.P.m;
  const Cmd& c = pl.cmd;
  for (int j = 0; j < m; ++j) {
    Walk& w = pl.w[j];
    const int b = c.row_start[j], e = c.row_start[j + 1];
    if (e <= b) continue;
    for (int k = b; k < e; ++k) walk_add_point(w, c.cand_y[k], t[2 * k] - w.ghat, t[2 * k + 1]);
    walk_advance(w, pl.P.opt);
  }
  if (!schedule_sweep(pl)) after_walks(pl);
}

TOPT_HDN inline void consume_final(Plan& pl, const double* t) {
  Problem& P = pl.P;
  Result& r = pl.res;
  const int m = P.m;
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

TOPT_HDN inline void consume_step(Plan& pl, const double* t) {
  const Problem& P = pl.P;
  const PgdSettings& s = P.set;
  Result& r = pl.res;
  for (int k = 0; k < 6; ++k) r.step_sums[k] = t[k];
  const int fallback = (P.t == 0) || (P.t >= s.t_warmup && P.violation > s.tol_n);
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

TOPT_HDN inline void plan_consume(Plan& pl, const double* t) {
  pl.res.passes++;
  switch (pl.cmd.phase) {
    case PH_STEP_REDUCE: consume_step(pl, t); break;
    case PH_PREP: consume_prep(pl, t); break;
    case PH_SWEEP: consume_sweep(pl, t); break;
    case PH_FEAS: consume_feas(pl, t); break;
    case PH_NEWTON: consume_newton(pl, t); break;
    case PH_FINAL: consume_final(pl, t); break;
    default: break;
  }
  if (pl.res.passes > 4096 && pl.cmd.phase != PH_DONE) set_error(pl, ST_INTERNAL);
}

}  // namespace topt_b200
