// ctl_sim.cpp — TEST HARNESS: drives the product controller (controller.h,
// compiled for the host) with pass totals computed on the CPU, so the control
// logic (walk replay, candidate choice, stage 1, Newton, path dispatch) and
// the rank-sharded reduction can be tested without a GPU.  The per-element
// arithmetic mirrors passes.cuh; sums are sequential per rank slab.
#include <cmath>
#include <cstdint>
#include <cstring>

#include "controller.h"

using namespace topt_b200;

namespace {
double clipd(double v, double lo, double hi) { return v < lo ? lo : (v > hi ? hi : v); }
double op(int o, double a, double b) { return o == 0 ? a + b : (o == 1 ? dmin_(a, b) : dmax_(a, b)); }
}  // namespace

extern "C" {

int64_t sim_plan_size() { return (int64_t)sizeof(Plan); }

// Fill the Problem of a zeroed Plan (host pointers) and start it.
void sim_setup(Plan* pl, int job, int which, int64_t n_local, int64_t n_global, int m,
               const double* x, const double* x_prev, const double* g, const double* g_prev,
               const double* d_prev, const double* grad, const double* gd_step, const int8_t* owner,
               double* rho, double* d_out, double* delta_out, double* x_out,
               const double* G_minus_g, const double* ghat_in, const int32_t* is_eq,
               const double* row_count, double lower, double upper, int t, double violation,
               double ours_len) {
  std::memset(pl, 0, sizeof(Plan));
  Problem& P = pl->P;
  P.n = n_local; P.n_global = n_global; P.m = m; P.job = job; P.which = which;
  P.has_part = owner != nullptr; P.t = t; P.lower = lower; P.upper = upper;
  P.violation = violation;
  P.opt.c = 1e12; P.opt.tol_b = 1e-8; P.opt.tol_n = 1e-6; P.opt.newton_maxiter = 50;
  P.opt.binary_maxiter = 200;
  P.set.alpha_max = 1e2; P.set.alpha_fallback = 0.2; P.set.omega = 1.0; P.set.eps_alpha = 1e-6;
  P.set.tol_n = 1e-6; P.set.t_warmup = 50;
  P.x = x; P.x_prev = x_prev; P.g = g; P.g_prev = g_prev; P.d_prev = d_prev; P.grad = grad;
  P.ld = n_local; P.gd_step = gd_step; P.owner = owner; P.rho = rho; P.d_out = d_out;
  P.delta_out = delta_out; P.x_out = x_out;
  for (int j = 0; j < m; ++j) {
    P.G_minus_g[j] = G_minus_g ? G_minus_g[j] : 0.0;
    P.ghat_in[j] = ghat_in ? ghat_in[j] : 0.0;
    P.is_eq[j] = is_eq ? is_eq[j] : 0;
    P.row_count[j] = row_count ? row_count[j] : (double)n_global;
  }
  P.ours_len = ours_len;
  plan_start(*pl);
}

int sim_phase(const Plan* pl) { return pl->cmd.phase; }
int sim_nslots(const Plan* pl) { return pl->cmd.nslots; }
int sim_slot_op(const Plan* pl, int s) { return slot_op(pl->cmd.phase, s); }
void sim_consume(Plan* pl, const double* totals) { plan_consume(*pl, totals); }
void sim_set_hint(Plan* pl, int j, double y, double sig) {
  pl->hint_y[j] = y; pl->hint_sig[j] = sig; pl->hint_ok[j] = 1;
}
// walk j state: lo hi ym yL yH (nan if absent) iters status; candidates of the next sweep
void sim_walk(const Plan* pl, int j, double* w, double* cand, int* ncand) {
  const Walk& k = pl->w[j];
  const double nan = 0.0 / 0.0;
  w[0] = k.lo; w[1] = k.hi; w[2] = k.ym; w[3] = k.hasL ? k.yL : nan; w[4] = k.hasH ? k.yH : nan;
  w[5] = k.iters; w[6] = k.status; w[7] = k.E; w[8] = k.n_direct;
  w[9] = pl->cmd.wlo[j]; w[10] = pl->cmd.whi[j];
  { const RootEst e = walk_estimate(k); w[11] = e.kind; w[12] = e.ye; w[13] = e.sig; }
  const int b = pl->cmd.row_start[j], e = pl->cmd.row_start[j + 1];
  *ncand = (pl->cmd.phase == PH_SWEEP) ? e - b : 0;
  for (int q = 0; q < *ncand; ++q) cand[q] = pl->cmd.cand_y[b + q];
}

void sim_result(const Plan* pl, int32_t* ints /* status path newton_iters converged curv passes sweeps stage1 near_ties fallback */,
                double* dbl /* residual alpha beta min_margin */, double* y, double* ghat) {
  const Result& r = pl->res;
  const int32_t iv[10] = {r.status, r.path, r.newton_iters, r.converged, r.curvature_violations,
                          r.passes, r.sweeps, r.stage1_row, r.near_ties, r.fallback};
  std::memcpy(ints, iv, sizeof(iv));
  dbl[0] = r.residual; dbl[1] = r.alpha; dbl[2] = r.beta; dbl[3] = r.min_margin;
  for (int j = 0; j < pl->P.m; ++j) { y[j] = r.y[j]; ghat[j] = r.ghat[j]; }
}

// This rank's partial slots for the current command (writes its outputs).
void sim_partials(const Plan* pl, double* out) {
  const Problem& P = pl->P;
  const Cmd& c = pl->cmd;
  const int m = P.m;
  const double L = P.lower, U = P.upper;
  for (int s = 0; s < c.nslots; ++s) out[s] = 0.0;
  switch (c.phase) {
    case PH_STEP_REDUCE:
      for (int64_t i = 0; i < P.n; ++i) {
        const double s = P.x[i] - P.x_prev[i], y = P.g[i] - P.g_prev[i];
        out[0] += s * s; out[1] += s * y; out[2] += y * y; out[3] += P.g[i] * y;
        out[4] += P.g_prev[i] * P.g_prev[i]; out[5] = dmax_(out[5], std::fabs(P.g[i]));
      }
      break;
    case PH_PREP: {
      if (c.compute_dir)
        for (int64_t i = 0; i < P.n; ++i) {
          const double d = c.use_dprev ? P.g[i] + c.beta * P.d_prev[i] : P.g[i];
          P.d_out[i] = d;
          P.rho[i] = P.x[i] - c.wa * d;
        }
      for (int j = 0; j < m; ++j) {
        double* v = out + j * PREP_SLOTS;
        const double* a = P.grad + (int64_t)j * P.ld;
        for (int64_t i = 0; i < P.n; ++i) {
          if (P.owner && P.owner[i] != j) { v[PS_NZOUT] += a[i] != 0.0; continue; }
          const double lo = L - P.rho[i], hi = U - P.rho[i];
          if (c.compute_dot) {
            const double gd = c.compute_dir ? c.wa * P.d_out[i] : P.gd_step[i];
            v[PS_DOT] += gd * a[i]; v[PS_DABS] += std::fabs(gd * a[i]);
          }
          v[PS_S0] += a[i] * clipd(0.0, lo, hi);
          if (!(0.0 < lo || 0.0 > hi)) v[PS_SLOPE0] += a[i] * a[i];
          v[PS_T] += std::fabs(a[i]) * dmax_(std::fabs(lo), std::fabs(hi));
          if (std::fabs(a[i]) >= kGradFloor) {
            v[PS_ANY] += 1.0;
            const double c1 = lo / a[i], c2 = hi / a[i];
            v[PS_BPLO] = dmin_(v[PS_BPLO], dmin_(c1, c2));
            v[PS_BPHI] = dmax_(v[PS_BPHI], dmax_(c1, c2));
          }
        }
      }
      break;
    }
    case PH_SWEEP:
      for (int j = 0; j < m; ++j) {
        const double* a = P.grad + (int64_t)j * P.ld;
        for (int k = c.row_start[j]; k < c.row_start[j + 1]; ++k) {
          const double y = c.cand_y[k];
          double R = 0.0, S = 0.0;
          for (int64_t i = 0; i < P.n; ++i) {
            if (P.owner && P.owner[i] != j) continue;
            const double lo = L - P.rho[i], hi = U - P.rho[i];
            const double v = y * a[i];
            const bool b = v < lo, ab = v > hi;
            R += a[i] * (b ? lo : (ab ? hi : v));
            if (!(b || ab)) S += a[i] * a[i];
          }
          out[2 * k] = R; out[2 * k + 1] = S;
        }
      }
      break;
    case PH_FEAS:
      for (int f = 0; f < c.nfeas; ++f)
        for (int64_t i = 0; i < P.n; ++i) {
          const double lo = L - P.rho[i], hi = U - P.rho[i];
          double z = 0.0;
          if (c.feas_row[f] >= 0 && c.feas_y[f] != 0.0)
            z = 0.0 + c.feas_y[f] * P.grad[(int64_t)c.feas_row[f] * P.ld + i];
          const double dl = clipd(z, lo, hi);
          for (int k = 0; k < m; ++k) out[f * m + k] += P.grad[(int64_t)k * P.ld + i] * dl;
        }
      break;
    case PH_NEWTON:
      for (int64_t i = 0; i < P.n; ++i) {
        const double lo = L - P.rho[i], hi = U - P.rho[i];
        double z = 0.0;
        for (int j = 0; j < m; ++j)
          if (c.y[j] != 0.0) z += c.y[j] * P.grad[(int64_t)j * P.ld + i];
        const bool clipped = z < lo || z > hi;
        const double dl = clipd(z, lo, hi);
        for (int k = 0; k < m; ++k) out[k] += P.grad[(int64_t)k * P.ld + i] * dl;
        if (c.want_gram && !clipped)
          for (int j = 0; j < m; ++j)
            for (int k = j; k < m; ++k)
              out[m + gram_idx(m, j, k)] += P.grad[(int64_t)j * P.ld + i] * P.grad[(int64_t)k * P.ld + i];
      }
      break;
    case PH_FINAL:
      for (int64_t i = 0; i < P.n; ++i) {
        const double lo = L - P.rho[i], hi = U - P.rho[i];
        double z = 0.0;
        int o = -1;
        if (P.owner) {
          o = P.owner[i];
          if (o >= 0 && c.y[o] != 0.0) z = 0.0 + c.y[o] * P.grad[(int64_t)o * P.ld + i];
        } else {
          for (int j = 0; j < m; ++j)
            if (c.y[j] != 0.0) z += c.y[j] * P.grad[(int64_t)j * P.ld + i];
        }
        const double dl = clipd(z, lo, hi);
        if (P.delta_out) P.delta_out[i] = dl;
        if (P.x_out) P.x_out[i] = P.rho[i] + dl;
        if (c.resid_rows)
          for (int k = 0; k < m; ++k)
            if (o < 0 ? P.owner == nullptr : k == o) out[k] += P.grad[(int64_t)k * P.ld + i] * dl;
      }
      break;
    default:
      break;
  }
}

}  // extern "C"
