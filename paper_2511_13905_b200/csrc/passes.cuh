// passes.cuh — the O(n) passes of the PGD-TO step (device code).
//
// Every pass is a grid-stride sweep over this rank's slab that produces a
// small vector of partial sums (<= PMAX slots) per CTA.  Reductions are
// deterministic: a fixed per-thread order, a fixed shuffle tree per warp, a
// fixed warp order per CTA, and a fixed CTA order in the final combine, so
// the same inputs on the same launch geometry give the same bits.
//
// Element arithmetic follows projection.cpp exactly (the library is built
// with -fmad=false, so every product and sum is separately rounded):
//   lo = lower - rho_i, hi = upper - rho_i             (:32, :207)
//   clip(v, lo, hi) = v < lo ? lo : (v > hi ? hi : v)   (:15-17)
//   term = a_i * clip(y * a_i, lo, hi)                  (:32, :35)
//   z_i = sum_{j: y_j != 0} y_j a_ji, ascending j, from 0.0  (:199-205)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "controller.h"
#include "topt_core.h"

namespace topt_b200 {

constexpr int BLOCK = 256;
constexpr int NWARP = BLOCK / 32;

__device__ __forceinline__ double clipd(double v, double lo, double hi) {
  return v < lo ? lo : (v > hi ? hi : v);
}

__device__ __forceinline__ double apply_op(int op, double a, double b) {
  return op == 0 ? a + b : (op == 1 ? dmin_(a, b) : dmax_(a, b));
}

// Deterministic shuffle tree; lane 0 ends with the warp's value.
__device__ __forceinline__ double warp_reduce(int op, double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v = apply_op(op, v, __shfl_down_sync(0xffffffffu, v, off));
  return v;
}

// Reduce NS per-thread values (compile-time count) across the CTA and write
// them to out[slot0 + s] for s < ns (ns <= NS, runtime).  One __syncthreads.
template <int NS>
__device__ __forceinline__ void block_reduce_store(const double (&v)[NS], int ns, int phase,
                                                   int slot0, double* out, double* smem) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    if (s < ns) {
      const double r = warp_reduce(slot_op(phase, slot0 + s), v[s]);
      if (lane == 0) smem[warp * NS + s] = r;
    }
  }
  __syncthreads();
  if (threadIdx.x < ns) {
    const int s = threadIdx.x;
    const int op = slot_op(phase, slot0 + s);
    double r = smem[s];
    for (int w = 1; w < NWARP; ++w) r = apply_op(op, r, smem[w * NS + s]);
    out[slot0 + s] = r;
  }
  __syncthreads();
}

struct PassCtx {
  const Plan* plan;
  const Cmd* cmd;      // shared-memory copy
  double* out;         // this CTA's partial slots
  double* smem;        // reduction scratch (NWARP * 64 doubles)
  int64_t i0, stride;  // grid-stride
};

// ---- PH_STEP_REDUCE: BB / PR+ sums --------------------
__device__ void pass_step_reduce(const PassCtx& c) {
  const Problem& P = c.plan->P;
  double v[6] = {0, 0, 0, 0, 0, 0};
  for (int64_t i = c.i0; i < P.n; i += c.stride) {
    const double x = P.x[i], xp = P.x_prev[i], g = P.g[i], gp = P.g_prev[i];
    const double s = x - xp, y = g - gp;
    v[0] += s * s;
    v[1] += s * y;
    v[2] += y * y;
    v[3] += g * y;
    v[4] += gp * gp;
    v[5] = dmax_(v[5], fabs(g));
  }
  block_reduce_store<6>(v, 6, PH_STEP_REDUCE, 0, c.out, c.smem);
}

// ---- PH_PREP: direction, rho_tilde, g_hat dots, r(0), slope(0), bounds,
//      breakpoints (projection.cpp:53-73, :139-145, :150-181) ---------------
__device__ void pass_prep(const PassCtx& c) {
  const Plan& pl = *c.plan;
  const Problem& P = pl.P;
  const Cmd& cmd = *c.cmd;
  if (cmd.compute_dir) {  // d = g + beta d_prev ; gd = (omega alpha) d ; rho = x - gd
    for (int64_t i = c.i0; i < P.n; i += c.stride) {
      const double g = P.g[i];
      const double d = cmd.use_dprev ? g + cmd.beta * P.d_prev[i] : g;
      const double gd = cmd.wa * d;
      P.d_out[i] = d;
      P.rho[i] = P.x[i] - gd;
    }
  }
  const double L = P.lower, U = P.upper;
  for (int j = 0; j < P.m; ++j) {
    double v[PREP_SLOTS];
#pragma unroll
    for (int s = 0; s < PREP_SLOTS; ++s) v[s] = 0.0;
    v[PS_BPLO] = 0.0;  // projection.cpp:58 bp_lo = bp_hi = 0
    v[PS_BPHI] = 0.0;
    const double* a_row = P.grad + (int64_t)j * P.ld;
    for (int64_t i = c.i0; i < P.n; i += c.stride) {
      const double a = a_row[i];
      if (P.owner && P.owner[i] != j) {
        v[PS_NZOUT] += (a != 0.0) ? 1.0 : 0.0;
        continue;
      }
      const double r = P.rho[i];
      const double lo = L - r, hi = U - r;
      if (cmd.compute_dot) {
        const double gd = cmd.compute_dir ? cmd.wa * P.d_out[i] : P.gd_step[i];
        const double p = gd * a;
        v[PS_DOT] += p;
        v[PS_DABS] += fabs(p);
      }
      v[PS_S0] += a * clipd(0.0, lo, hi);
      if (!(0.0 < lo || 0.0 > hi)) v[PS_SLOPE0] += a * a;
      v[PS_T] += fabs(a) * dmax_(fabs(lo), fabs(hi));
      if (fabs(a) >= kGradFloor) {
        v[PS_ANY] += 1.0;
        const double c1 = lo / a, c2 = hi / a;
        v[PS_BPLO] = dmin_(v[PS_BPLO], dmin_(c1, c2));
        v[PS_BPHI] = dmax_(v[PS_BPHI], dmax_(c1, c2));
      }
    }
    block_reduce_store<PREP_SLOTS>(v, PREP_SLOTS, PH_PREP, j * PREP_SLOTS, c.out, c.smem);
  }
}

// ---- PH_SWEEP: r_j(y_k) and slope at up to MAX_K candidates per row -------
__device__ void pass_sweep(const PassCtx& c) {
  const Plan& pl = *c.plan;
  const Problem& P = pl.P;
  const Cmd& cmd = *c.cmd;
  const double L = P.lower, U = P.upper;
  for (int j = 0; j < P.m; ++j) {
    const int b = cmd.row_start[j], cnt = cmd.row_start[j + 1] - b;
    if (cnt <= 0) continue;
    double y[MAX_K], R[MAX_K], S[MAX_K];
#pragma unroll
    for (int k = 0; k < MAX_K; ++k) {
      y[k] = (k < cnt) ? cmd.cand_y[b + k] : 0.0;
      R[k] = 0.0;
      S[k] = 0.0;
    }
    const double* a_row = P.grad + (int64_t)j * P.ld;
    for (int64_t i = c.i0; i < P.n; i += c.stride) {
      if (P.owner && P.owner[i] != j) continue;
      const double a = a_row[i];
      const double r = P.rho[i];
      const double lo = L - r, hi = U - r;
      const double aa = a * a;
#pragma unroll
      for (int k = 0; k < MAX_K; ++k) {
        if (k < cnt) {
          const double v = y[k] * a;
          const bool below = v < lo, above = v > hi;
          const double cv = below ? lo : (above ? hi : v);
          R[k] += a * cv;
          S[k] += (below || above) ? 0.0 : aa;
        }
      }
    }
    double v[2 * MAX_K];
#pragma unroll
    for (int k = 0; k < MAX_K; ++k) { v[2 * k] = R[k]; v[2 * k + 1] = S[k]; }
    block_reduce_store<2 * MAX_K>(v, 2 * cnt, PH_SWEEP, 2 * b, c.out, c.smem);
  }
}

// ---- PH_FEAS: stage-1 dots a_k . clip(y_j a_j) (projection.cpp:320-333) ---
__device__ void pass_feas(const PassCtx& c) {
  const Plan& pl = *c.plan;
  const Problem& P = pl.P;
  const Cmd& cmd = *c.cmd;
  const double L = P.lower, U = P.upper;
  const int m = P.m;
  for (int f = 0; f < cmd.nfeas; ++f) {
    const int rj = cmd.feas_row[f];
    const double yj = cmd.feas_y[f];
    double acc[MAX_M];
#pragma unroll
    for (int k = 0; k < MAX_M; ++k) acc[k] = 0.0;
    for (int64_t i = c.i0; i < P.n; i += c.stride) {
      const double r = P.rho[i];
      const double lo = L - r, hi = U - r;
      double z = 0.0;
      if (rj >= 0 && yj != 0.0) z = 0.0 + yj * P.grad[(int64_t)rj * P.ld + i];
      const double dl = clipd(z, lo, hi);
#pragma unroll
      for (int k = 0; k < MAX_M; ++k)
        if (k < m) acc[k] += P.grad[(int64_t)k * P.ld + i] * dl;
    }
    block_reduce_store<MAX_M>(acc, m, PH_FEAS, f * m, c.out, c.smem);
  }
}

// ---- PH_NEWTON: delta(y), h-dots and the free-set Gram A D A^T ------------
// (eval_phi projection.cpp:279-298 and J_h projection.cpp:359-376)
template <int M>
__device__ __noinline__ void pass_newton_m(const PassCtx& c) {
  const Plan& pl = *c.plan;
  const Problem& P = pl.P;
  const Cmd& cmd = *c.cmd;
  const double L = P.lower, U = P.upper;
  const int m = P.m;
  constexpr int NG = M * (M + 1) / 2;
  double h[M], G[NG], y[M];
#pragma unroll
  for (int k = 0; k < M; ++k) { h[k] = 0.0; y[k] = (k < m) ? cmd.y[k] : 0.0; }
#pragma unroll
  for (int k = 0; k < NG; ++k) G[k] = 0.0;
  for (int64_t i = c.i0; i < P.n; i += c.stride) {
    double a[M];
#pragma unroll
    for (int k = 0; k < M; ++k) a[k] = (k < m) ? P.grad[(int64_t)k * P.ld + i] : 0.0;
    const double r = P.rho[i];
    const double lo = L - r, hi = U - r;
    double z = 0.0;
#pragma unroll
    for (int k = 0; k < M; ++k)
      if (k < m && y[k] != 0.0) z += y[k] * a[k];
    const bool clipped = (z < lo) || (z > hi);
    const double dl = clipd(z, lo, hi);
#pragma unroll
    for (int k = 0; k < M; ++k) h[k] += a[k] * dl;
    if (cmd.want_gram && !clipped) {
      int q = 0;
#pragma unroll
      for (int j = 0; j < M; ++j)
#pragma unroll
        for (int k = j; k < M; ++k) G[q++] += a[j] * a[k];
    }
  }
  // pack: slots [0, m) h ; [m, m + m(m+1)/2) upper-triangle of the m x m Gram
  double v[M + NG];
#pragma unroll
  for (int k = 0; k < M; ++k) v[k] = h[k];
  // re-pack from the M-wide triangle to the m-wide triangle
  {
    int q = 0;
#pragma unroll
    for (int j = 0; j < M; ++j)
#pragma unroll
      for (int k = j; k < M; ++k) {
        if (j < m && k < m) v[m + gram_idx(m, j, k)] = G[q];
        ++q;
      }
  }
  block_reduce_store<M + NG>(v, m + m * (m + 1) / 2, PH_NEWTON, 0, c.out, c.smem);
}

// ---- PH_FINAL: delta / x_{t+1} / mask writes and residual dots ------------
__device__ void pass_final(const PassCtx& c) {
  const Plan& pl = *c.plan;
  const Problem& P = pl.P;
  const Cmd& cmd = *c.cmd;
  const double L = P.lower, U = P.upper;
  const int m = P.m;
  double acc[MAX_M];
#pragma unroll
  for (int k = 0; k < MAX_M; ++k) acc[k] = 0.0;
  for (int64_t i = c.i0; i < P.n; i += c.stride) {
    const double r = P.rho[i];
    const double lo = L - r, hi = U - r;
    double z = 0.0;
    int o = -1;
    if (P.owner) {
      o = P.owner[i];
      if (o >= 0 && cmd.y[o] != 0.0) z = 0.0 + cmd.y[o] * P.grad[(int64_t)o * P.ld + i];
    } else {
      for (int j = 0; j < m; ++j) {
        const double yj = cmd.y[j];
        if (yj != 0.0) z += yj * P.grad[(int64_t)j * P.ld + i];
      }
    }
    const bool below = z < lo, above = z > hi;
    const double dl = below ? lo : (above ? hi : z);
    if (cmd.write_delta) P.delta_out[i] = dl;
    if (cmd.write_x) P.x_out[i] = r + dl;
    if (cmd.write_mask) P.mask_out[i] = below ? 1 : (above ? 2 : 0);
    if (cmd.resid_rows) {
#pragma unroll
      for (int k = 0; k < MAX_M; ++k) {
        if (k < m && (o < 0 ? P.owner == nullptr : k == o))
          acc[k] += P.grad[(int64_t)k * P.ld + i] * dl;
      }
    }
  }
  if (cmd.resid_rows) block_reduce_store<MAX_M>(acc, m, PH_FINAL, 0, c.out, c.smem);
}

__device__ void pass_newton(const PassCtx& c) {
  const int m = c.plan->P.m;
  if (m <= 1) pass_newton_m<1>(c);
  else if (m <= 2) pass_newton_m<2>(c);
  else if (m <= 4) pass_newton_m<4>(c);
  else if (m <= 8) pass_newton_m<8>(c);
  else pass_newton_m<16>(c);
}

__device__ void run_pass(const PassCtx& c) {
  switch (c.cmd->phase) {
    case PH_STEP_REDUCE: pass_step_reduce(c); break;
    case PH_PREP: pass_prep(c); break;
    case PH_SWEEP: pass_sweep(c); break;
    case PH_FEAS: pass_feas(c); break;
    case PH_NEWTON: pass_newton(c); break;
    case PH_FINAL: pass_final(c); break;
    default: break;
  }
}

}  // namespace topt_b200
