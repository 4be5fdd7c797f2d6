// fea.cu — the FE solve upstream of the step:
// plane-stress Q4 linear elasticity on an nx x ny structured grid
// (assemble_and_solve, /root/reference/proj/src/fea.cpp:60-144), solved with
// the reference's algorithm -- conjugate gradients with the diagonal (Jacobi)
// preconditioner, relative tolerance on ||r|| / ||f||, at most 10 N_free
// iterations (Eigen's ConjugateGradient as configured at fea.cpp:122-131) --
// but matrix-free and in ONE persistent cooperative kernel:
//   * K p is gathered per degree of freedom from the <= 4 adjacent elements
//     (E_e k0 p_e, the element matrix in registers / constant parameters):
//     no assembled sparse matrix, no atomics, a fixed summation order;
//   * each iteration is two grid-synchronized phases (K p and p.Kp; then the
//     x / r / z updates and r.r, r.z), the direction update p = z + beta p
//     folded into the next phase's gather;
//   * dot products reduce per CTA in a fixed tree and combine in CTA order in
//     every CTA, so all CTAs take the same decisions and a solve is bitwise
//     reproducible.
// Fixed dofs are excluded exactly like the reference's free-dof system
// (their entries of x, r, z, p stay 0, so they never contribute).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "../../include/topt_b200.h"

namespace cg = cooperative_groups;

namespace {

constexpr int FBLOCK = 256;
constexpr int FWARPS = FBLOCK / 32;

struct KeMat {
  double k[64];
};

struct PcgArgs {
  int nx, ny;
  KeMat ke;
  const double* E;       // element moduli (nx ny)
  const uint8_t* fixed;  // 1 = fixed dof (ndof)
  const double* f;       // right-hand side on all dofs (0 on fixed)
  double* x;
  double* r;
  double* z;
  double* p[2];          // direction, double-buffered
  double* ap;
  double* invd;          // inverse diagonal (Eigen DiagonalPreconditioner)
  double* part;          // [nb][4] per-CTA partial sums
  double tol;
  int64_t maxit;
  int64_t* out_iters;
  double* out_res2;      // ||r||^2 at exit
  double* out_rhs2;      // ||f||^2
};

// Element e's dof j (grid.cpp:15-24: nodes (ex,ey), (ex+1,ey), (ex+1,ey+1), (ex,ey+1)).
__device__ __forceinline__ int64_t edof(int nx, int ex, int ey, int j) {
  const int a = j >> 1, c = j & 1;
  const int ix = ex + ((a == 1 || a == 2) ? 1 : 0);
  const int iy = ey + ((a >= 2) ? 1 : 0);
  return 2 * ((int64_t)iy * (nx + 1) + ix) + c;
}

// (K v)_d for a free dof d = 2 (iy (nx+1) + ix) + c, gathered over the <= 4
// adjacent elements in (ey, ex) order; v_j is produced by `val(j)`.
template <typename V>
__device__ __forceinline__ double kmul(const PcgArgs& a, int ix, int iy, int c, V&& val) {
  double y = 0.0;
  for (int ey = iy - 1; ey <= iy; ++ey) {
    if (ey < 0 || ey >= a.ny) continue;
    for (int ex = ix - 1; ex <= ix; ++ex) {
      if (ex < 0 || ex >= a.nx) continue;
      const int loc = (ix == ex) ? (iy == ey ? 0 : 3) : (iy == ey ? 1 : 2);
      const int li = 2 * loc + c;
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < 8; ++j) s += a.ke.k[li * 8 + j] * val(edof(a.nx, ex, ey, j));
      y += a.E[(int64_t)ey * a.nx + ex] * s;
    }
  }
  return y;
}

__device__ __forceinline__ double kdiag(const PcgArgs& a, int ix, int iy, int c) {
  double y = 0.0;
  for (int ey = iy - 1; ey <= iy; ++ey) {
    if (ey < 0 || ey >= a.ny) continue;
    for (int ex = ix - 1; ex <= ix; ++ex) {
      if (ex < 0 || ex >= a.nx) continue;
      const int loc = (ix == ex) ? (iy == ey ? 0 : 3) : (iy == ey ? 1 : 2);
      const int li = 2 * loc + c;
      y += a.E[(int64_t)ey * a.nx + ex] * a.ke.k[li * 8 + li];
    }
  }
  return y;
}

// Deterministic CTA reduction of NS values, written to part[blockIdx][0..NS).
template <int NS>
__device__ __forceinline__ void cta_reduce(double (&v)[NS], double* part, double* smem) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int s = 0; s < NS; ++s)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[s] += __shfl_down_sync(0xffffffffu, v[s], o);
  if (lane == 0)
#pragma unroll
    for (int s = 0; s < NS; ++s) smem[warp * 4 + s] = v[s];
  __syncthreads();
  if (threadIdx.x < NS) {
    double t = 0.0;
    for (int w = 0; w < FWARPS; ++w) t += smem[w * 4 + threadIdx.x];
    part[(size_t)blockIdx.x * 4 + threadIdx.x] = t;
  }
  __syncthreads();
}

// Every CTA sums the CTA partials in CTA order (same bits everywhere).
template <int NS>
__device__ __forceinline__ void combine(const double* part, int nb, double (&out)[NS], double* smem) {
  if (threadIdx.x < NS) {
    double t = 0.0;
    for (int b = 0; b < nb; ++b) t += __ldcg(part + (size_t)b * 4 + threadIdx.x);
    smem[32 + threadIdx.x] = t;
  }
  __syncthreads();
#pragma unroll
  for (int s = 0; s < NS; ++s) out[s] = smem[32 + s];
  __syncthreads();
}

__global__ void __launch_bounds__(FBLOCK) k_pcg(PcgArgs a) {
  __shared__ double smem[64];
  cg::grid_group grid = cg::this_grid();
  const int nb = gridDim.x;
  const int64_t nn = (int64_t)(a.nx + 1) * (a.ny + 1), nd = 2 * nn;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t st = (int64_t)nb * blockDim.x;
  // set-up: invd, x = 0, r = f, z = invd r, p = z; partials f.f, r.r, r.z
  {
    double v[3] = {0.0, 0.0, 0.0};
    for (int64_t d = t0; d < nd; d += st) {
      const int64_t node = d >> 1;
      const int c = (int)(d & 1), ix = (int)(node % (a.nx + 1)), iy = (int)(node / (a.nx + 1));
      const bool fr = !a.fixed[d];
      const double dg = fr ? kdiag(a, ix, iy, c) : 0.0;
      const double iv = (fr && dg != 0.0) ? 1.0 / dg : (fr ? 1.0 : 0.0);
      const double fd = fr ? a.f[d] : 0.0;
      a.invd[d] = iv;
      a.x[d] = 0.0;
      a.r[d] = fd;
      const double zd = iv * fd;
      a.z[d] = zd;
      a.p[0][d] = zd;
      v[0] += fd * fd;
      v[1] += fd * fd;
      v[2] += fd * zd;
    }
    cta_reduce<3>(v, a.part, smem);
  }
  grid.sync();
  double s3[3];
  combine<3>(a.part, nb, s3, smem);
  const double rhs2 = s3[0];
  double rr = s3[1], absNew = s3[2];
  int64_t it = 0;
  const double thr = fmax(a.tol * a.tol * rhs2, 2.2250738585072014e-308);
  bool done = rhs2 == 0.0 || rr < thr;
  int cur = 0;          // p[cur] holds the current direction
  double beta = 0.0;
  bool fresh = true;    // p[cur] already computed (first iteration)
  while (!done && it < a.maxit) {
    // phase A: p = z + beta p_old (on the fly for the gather), Ap = K p, p.Ap
    const double* po = a.p[cur];
    double* pn = a.p[cur ^ 1];
    {
      double v[1] = {0.0};
      for (int64_t d = t0; d < nd; d += st) {
        const int64_t node = d >> 1;
        const int c = (int)(d & 1), ix = (int)(node % (a.nx + 1)), iy = (int)(node / (a.nx + 1));
        double apd = 0.0, pd = 0.0;
        if (fresh) {
          pd = po[d];
          if (!a.fixed[d]) apd = kmul(a, ix, iy, c, [&](int64_t j) { return po[j]; });
        } else {
          pd = a.z[d] + beta * po[d];
          if (!a.fixed[d])
            apd = kmul(a, ix, iy, c, [&](int64_t j) { return a.z[j] + beta * po[j]; });
          pn[d] = pd;
        }
        a.ap[d] = apd;
        v[0] += pd * apd;
      }
      cta_reduce<1>(v, a.part, smem);
    }
    if (!fresh) cur ^= 1;
    fresh = false;
    grid.sync();
    double s1[1];
    combine<1>(a.part, nb, s1, smem);
    const double alpha = absNew / s1[0];
    // phase B: x += alpha p, r -= alpha Ap, r.r, z = invd r, r.z
    {
      const double* p = a.p[cur];
      double v[2] = {0.0, 0.0};
      for (int64_t d = t0; d < nd; d += st) {
        a.x[d] += alpha * p[d];
        const double rd = a.r[d] - alpha * a.ap[d];
        a.r[d] = rd;
        const double zd = a.invd[d] * rd;
        a.z[d] = zd;
        v[0] += rd * rd;
        v[1] += rd * zd;
      }
      cta_reduce<2>(v, a.part, smem);
    }
    grid.sync();
    double s2[2];
    combine<2>(a.part, nb, s2, smem);
    rr = s2[0];
    if (rr < thr) { done = true; break; }
    const double absOld = absNew;
    absNew = s2[1];
    beta = absNew / absOld;
    ++it;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *a.out_iters = it;
    *a.out_res2 = rr;
    *a.out_rhs2 = rhs2;
  }
}

// (K u - f) on free dofs, for the reported relative residual (fea.cpp:130).
__global__ void k_residual(PcgArgs a, const double* u, double* res) {
  const int64_t nn = (int64_t)(a.nx + 1) * (a.ny + 1), nd = 2 * nn;
  for (int64_t d = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; d < nd;
       d += (int64_t)gridDim.x * blockDim.x) {
    if (a.fixed[d]) { res[d] = 0.0; continue; }
    const int64_t node = d >> 1;
    const int c = (int)(d & 1), ix = (int)(node % (a.nx + 1)), iy = (int)(node / (a.nx + 1));
    res[d] = kmul(a, ix, iy, c, [&](int64_t j) { return a.fixed[j] ? 0.0 : u[j]; }) - a.f[d];
  }
}

struct Bufs {
  void* p = nullptr;
  size_t bytes = 0;
  void* get(size_t b) {
    if (bytes < b) {
      cudaFree(p);
      p = nullptr;
      bytes = 0;
      if (cudaMalloc(&p, b) != cudaSuccess) return nullptr;
      bytes = b;
    }
    return p;
  }
};
thread_local Bufs g_work, g_bc;

}  // namespace

extern "C" {

int topt_b200_fe_solve_dev(topt_b200_ctx* ctx, int32_t nx, int32_t ny, double element_size,
                           double poisson, const double* moduli_dev, const int32_t* fixed_dofs,
                           int64_t n_fixed, const int32_t* load_dofs, const double* load_values,
                           int64_t n_loads, double rel_tol, double* u_dev, int64_t* iterations,
                           double* residual) {
  if (nx < 1 || ny < 1) return TOPT_ERR_PARAMETER;
  const int64_t nn = (int64_t)(nx + 1) * (ny + 1), nd = 2 * nn, ne = (int64_t)nx * ny;
  // BoundaryConditions::validate (grid.cpp:26-38)
  if (n_fixed <= 0) return TOPT_ERR_PARAMETER;   // rigid-body modes present
  std::vector<uint8_t> fixed(nd, 0);
  for (int64_t k = 0; k < n_fixed; ++k) {
    if (fixed_dofs[k] < 0 || fixed_dofs[k] >= nd) return TOPT_ERR_PARAMETER;
    fixed[fixed_dofs[k]] = 1;
  }
  std::vector<double> f(nd, 0.0);
  for (int64_t k = 0; k < n_loads; ++k) {
    const int32_t d = load_dofs[k];
    if (d < 0 || d >= nd) return TOPT_ERR_PARAMETER;
    if (fixed[d]) return TOPT_ERR_PARAMETER;        // load applied on a fixed dof
    f[d] += load_values[k];                          // fea.cpp:98-101
  }
  int64_t nfree = 0;
  for (int64_t d = 0; d < nd; ++d) nfree += !fixed[d];
  PcgArgs a;
  a.nx = nx; a.ny = ny;
  if (int rc = topt_b200_element_stiffness_q4(poisson, element_size, a.ke.k)) return rc;
  cudaStream_t s = (cudaStream_t)topt_b200_get_stream(ctx);
  int dev = 0, nsm = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_pcg, FBLOCK, 0);
  const int nb = std::max(1, std::min(nsm * std::max(per, 1), (int)((nd + FBLOCK - 1) / FBLOCK)));
  const size_t vb = sizeof(double) * (size_t)nd;
  char* w = (char*)g_work.get(7 * vb + sizeof(double) * 4 * (size_t)nb + 64);
  char* bcb = (char*)g_bc.get(vb + (size_t)nd + 16);
  if (!w || !bcb) return TOPT_ERR_CUDA;
  a.r = (double*)w; a.z = a.r + nd; a.p[0] = a.z + nd; a.p[1] = a.p[0] + nd; a.ap = a.p[1] + nd;
  a.invd = a.ap + nd;
  double* res = a.invd + nd;
  a.part = res + nd;
  int64_t* d_iters = (int64_t*)(a.part + 4 * (size_t)nb);
  double* d_res2 = (double*)(d_iters + 1);
  double* d_rhs2 = d_res2 + 1;
  double* df = (double*)bcb;
  uint8_t* dfix = (uint8_t*)(df + nd);
  bool ok = cudaMemcpyAsync(df, f.data(), vb, cudaMemcpyHostToDevice, s) == cudaSuccess &&
            cudaMemcpyAsync(dfix, fixed.data(), (size_t)nd, cudaMemcpyHostToDevice, s) == cudaSuccess;
  if (!ok) return TOPT_ERR_CUDA;
  a.E = moduli_dev; a.fixed = dfix; a.f = df; a.x = u_dev;
  a.tol = rel_tol;
  a.maxit = 10 * nfree;                               // fea.cpp:127
  a.out_iters = d_iters; a.out_res2 = d_res2; a.out_rhs2 = d_rhs2;
  (void)ne;
  void* args[] = {&a};
  if (cudaLaunchCooperativeKernel((const void*)k_pcg, nb, FBLOCK, args, 0, s) != cudaSuccess)
    return TOPT_ERR_CUDA;
  // reported relative residual ||K u - f|| / ||f|| (fea.cpp:130), own pass
  k_residual<<<nb, FBLOCK, 0, s>>>(a, u_dev, res);
  int64_t its = 0;
  double rhs2 = 0.0;
  std::vector<double> hres(nd);
  ok = cudaMemcpyAsync(&its, d_iters, sizeof(int64_t), cudaMemcpyDeviceToHost, s) == cudaSuccess &&
       cudaMemcpyAsync(&rhs2, d_rhs2, sizeof(double), cudaMemcpyDeviceToHost, s) == cudaSuccess &&
       cudaMemcpyAsync(hres.data(), res, vb, cudaMemcpyDeviceToHost, s) == cudaSuccess &&
       cudaStreamSynchronize(s) == cudaSuccess;
  if (!ok) return TOPT_ERR_CUDA;
  double rn = 0.0;
  for (double v : hres) rn += v * v;
  const double rel = rhs2 > 0.0 ? std::sqrt(rn) / std::sqrt(rhs2) : 0.0;
  if (iterations) *iterations = its;
  if (residual) *residual = rel;
  if (its >= a.maxit && rel > rel_tol) return TOPT_ERR_SINGULAR;   // fea.cpp:132-137
  return TOPT_OK;
}

}  // extern "C"
