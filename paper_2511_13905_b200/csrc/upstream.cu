// upstream.cu — the producers of the step's inputs (SURVEY.md §8(f) ranks
// 2-3): the density filter W x and its chain rule W^T g, SIMP stiffness
// interpolation, and compliance sensitivities from a displacement field.
// Elementwise / stencil work, HBM-bound; every value is computed with the
// reference's own expressions in the reference's own order, so results are
// bit-identical to /root/reference/proj/src/{filter,material}.cpp (the one
// exception, std::pow, is noted at interpolate_stiffness).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/topt_b200.h"

namespace {

constexpr int UBLOCK = 256;
constexpr int MAX_REACH = 7;                       // radius <= 8 element units
constexpr int MAX_TAB = (2 * MAX_REACH + 1) * (2 * MAX_REACH + 1);

// Raw hat weights w(dx, dy) = radius - hypot(dx, dy) (filter.cpp:33), evaluated
// on the HOST with the C library's hypot -- the reference's own function, so
// the table is bit-identical -- and passed by value to the kernels.
struct HatTable {
  double w[MAX_TAB];
  int reach, width;
};

// Row total of element (ex, ey): the reference's sequential sum over the
// stencil in (dy, dx) order, skipping out-of-grid and non-positive weights
// (filter.cpp:24-36).
__device__ __forceinline__ double row_total(const HatTable& t, int nx, int ny, int ex, int ey) {
  double total = 0.0;
  for (int dy = -t.reach; dy <= t.reach; ++dy) {
    const int iy = ey + dy;
    if (iy < 0 || iy >= ny) continue;
    for (int dx = -t.reach; dx <= t.reach; ++dx) {
      const int ix = ex + dx;
      if (ix < 0 || ix >= nx) continue;
      const double w = t.w[(dy + t.reach) * t.width + (dx + t.reach)];
      if (w <= 0.0) continue;
      total = __dadd_rn(total, w);
    }
  }
  return total;
}

__global__ void k_filter_totals(HatTable t, int nx, int ny, double* totals) {
  const int64_t n = (int64_t)nx * ny;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    totals[e] = row_total(t, nx, ny, (int)(e % nx), (int)(e / nx));
}

// filtered_e = sum_i (w_i / total_e) raw_{col_i}, in CSR order (filter.cpp:45-56).
__global__ void k_filter_apply(HatTable t, int nx, int ny, const double* __restrict__ totals,
                               const double* __restrict__ raw, double* __restrict__ out) {
  const int64_t n = (int64_t)nx * ny;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int ex = (int)(e % nx), ey = (int)(e / nx);
    const double total = totals[e];
    double acc = 0.0;
    for (int dy = -t.reach; dy <= t.reach; ++dy) {
      const int iy = ey + dy;
      if (iy < 0 || iy >= ny) continue;
      for (int dx = -t.reach; dx <= t.reach; ++dx) {
        const int ix = ex + dx;
        if (ix < 0 || ix >= nx) continue;
        const double w = t.w[(dy + t.reach) * t.width + (dx + t.reach)];
        if (w <= 0.0) continue;
        acc = __dadd_rn(acc, __dmul_rn(__ddiv_rn(w, total), raw[(int64_t)iy * nx + ix]));
      }
    }
    out[e] = acc;
  }
}

// (W^T g)_c = sum over rows e containing c, in ascending e, of (w / total_e) g_e:
// the reference's scatter (filter.cpp:58-69) visits e in ascending order, so
// gathering the neighbours of c by ascending (oy, ox) reproduces its sums.
__global__ void k_filter_chain(HatTable t, int nx, int ny, const double* __restrict__ totals,
                               const double* __restrict__ g, double* __restrict__ out) {
  const int64_t n = (int64_t)nx * ny;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < n;
       c += (int64_t)gridDim.x * blockDim.x) {
    const int cx = (int)(c % nx), cy = (int)(c / nx);
    double acc = 0.0;
    for (int oy = -t.reach; oy <= t.reach; ++oy) {
      const int ey = cy + oy;
      if (ey < 0 || ey >= ny) continue;
      for (int ox = -t.reach; ox <= t.reach; ++ox) {
        const int ex = cx + ox;
        if (ex < 0 || ex >= nx) continue;
        // c seen from e is at offset (-ox, -oy)
        const double w = t.w[(-oy + t.reach) * t.width + (-ox + t.reach)];
        if (w <= 0.0) continue;
        const int64_t e = (int64_t)ey * nx + ex;
        acc = __dadd_rn(acc, __dmul_rn(__ddiv_rn(w, totals[e]), g[e]));
      }
    }
    out[c] = acc;
  }
}

// Generic CSR kernel (any FilterKernel, e.g. from the C++ drop-in): y = W x,
// one thread per row, the row's terms in CSR order.
__global__ void k_csr_apply(int64_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                            const double* __restrict__ w, const double* __restrict__ x,
                            double* __restrict__ y) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int i = rp[e]; i < rp[e + 1]; ++i) acc = __dadd_rn(acc, __dmul_rn(w[i], x[col[i]]));
    y[e] = acc;
  }
}
// Transposed CSR (CSC of W, entries of each column in ascending row order):
// (W^T g)_c = sum_k wt_k g_{rowt_k} -- the reference scatter's order.
__global__ void k_csc_apply(int64_t n, const int32_t* __restrict__ cp, const int32_t* __restrict__ row,
                            const double* __restrict__ w, const double* __restrict__ g,
                            double* __restrict__ y) {
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < n;
       c += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int k = cp[c]; k < cp[c + 1]; ++k) acc = __dadd_rn(acc, __dmul_rn(w[k], g[row[k]]));
    y[c] = acc;
  }
}

// SIMP (material.cpp:34-43): moduli_e = e_min + sum_j pow(r, p) (E_j - e_min)
// in channel order, der_{j,e} = p pow(r, p - 1) (E_j - e_min), r = clamp(rho).
// pow: CUDA's pow (<= 2 ulp) instead of the host C library's -- the one
// operation here that is not bit-identical (relative difference <= ~5e-16).
__global__ void k_simp(int64_t n, int k, const double* __restrict__ young, double e_min, double p,
                       const double* __restrict__ dens, double* __restrict__ moduli,
                       double* __restrict__ der) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    double mod = e_min;
    for (int j = 0; j < k; ++j) {
      const double scale = young[j] - e_min;
      const double r = fmin(1.0, fmax(0.0, dens[(int64_t)j * n + e]));
      mod = __dadd_rn(mod, __dmul_rn(pow(r, p), scale));
      if (der) der[(int64_t)j * n + e] = __dmul_rn(__dmul_rn(p, pow(r, p - 1.0)), scale);
    }
    moduli[e] = mod;
  }
}

// Element energy u_e^T k0 u_e (fea.cpp:162-174) and the compliance gradient
// -dE_{j,e} * energy_e (fea.cpp:176-181) from a displacement field, element e
// = ey nx + ex with dofs of nodes (ex,ey), (ex+1,ey), (ex+1,ey+1), (ex,ey+1)
// (grid.cpp:15-24).  ke in constant memory-like by-value struct.
struct Ke {
  double k[64];
};
__global__ void k_energy_grad(int nx, int ny, Ke ke, const double* __restrict__ u, int kmat,
                              const double* __restrict__ der, double* __restrict__ energy,
                              double* __restrict__ grad) {
  const int64_t n = (int64_t)nx * ny;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int ex = (int)(e % nx), ey = (int)(e / nx);
    const int64_t n1 = (int64_t)ey * (nx + 1) + ex, n2 = n1 + 1;
    const int64_t n3 = (int64_t)(ey + 1) * (nx + 1) + ex + 1, n4 = n3 - 1;
    double ue[8];
    ue[0] = u[2 * n1]; ue[1] = u[2 * n1 + 1];
    ue[2] = u[2 * n2]; ue[3] = u[2 * n2 + 1];
    ue[4] = u[2 * n3]; ue[5] = u[2 * n3 + 1];
    ue[6] = u[2 * n4]; ue[7] = u[2 * n4 + 1];
    double acc = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      double row = 0.0;
#pragma unroll
      for (int j = 0; j < 8; ++j) row = __dadd_rn(row, __dmul_rn(ke.k[i * 8 + j], ue[j]));
      acc = __dadd_rn(acc, __dmul_rn(ue[i], row));
    }
    if (energy) energy[e] = acc;
    if (grad)
      for (int j = 0; j < kmat; ++j)
        grad[(int64_t)j * n + e] = __dmul_rn(-der[(int64_t)j * n + e], acc);
  }
}

// interpolate_stiffness's range check (material.cpp:25-29): any density
// outside [-1e-12, 1 + 1e-12] (or NaN) sets *bad.
__global__ void k_range(int64_t cnt, const double* __restrict__ d, int* bad) {
  constexpr double slack = 1e-12;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double r = d[i];
    if (!(r >= -slack && r <= 1.0 + slack)) *bad = 1;
  }
}

int launch_grid(int64_t n) {
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (n + UBLOCK - 1) / UBLOCK;
  return (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)nsm * 8));
}

}  // namespace

struct topt_b200_filter {
  int nx = 0, ny = 0;
  double radius = 0.0;
  HatTable tab{};
  double* d_totals = nullptr;
  int64_t nnz = 0;
  int device = 0;
  std::string err;
};

namespace {
struct Scratch {
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
thread_local Scratch g_in, g_out, g_aux, g_aux2;

}  // namespace

extern "C" {

int topt_b200_filter_create(topt_b200_ctx* ctx, int32_t nx, int32_t ny, double radius,
                            topt_b200_filter** out) {
  (void)ctx;
  *out = nullptr;
  if (!(radius > 0.0)) return TOPT_ERR_PARAMETER;   // build_filter (filter.cpp:11)
  if (nx < 1 || ny < 1) return TOPT_ERR_PARAMETER;  // StructuredGrid (grid.cpp:11)
  const int reach = std::max(0, static_cast<int>(std::ceil(radius)) - 1);   // filter.cpp:20
  if (reach > MAX_REACH) return TOPT_ERR_UNSUPPORTED;
  auto* f = new topt_b200_filter();
  f->nx = nx; f->ny = ny; f->radius = radius;
  cudaGetDevice(&f->device);
  f->tab.reach = reach;
  f->tab.width = 2 * reach + 1;
  int per_row = 0;
  for (int dy = -reach; dy <= reach; ++dy)
    for (int dx = -reach; dx <= reach; ++dx) {
      const double w = radius - std::hypot(double(dx), double(dy));   // filter.cpp:33
      f->tab.w[(dy + reach) * f->tab.width + (dx + reach)] = w;
      per_row += w > 0.0;
    }
  (void)per_row;
  const int64_t n = (int64_t)nx * ny;
  if (cudaMalloc(&f->d_totals, sizeof(double) * (size_t)n) != cudaSuccess) {
    delete f;
    return TOPT_ERR_CUDA;
  }
  k_filter_totals<<<launch_grid(n), UBLOCK>>>(f->tab, nx, ny, f->d_totals);
  if (cudaDeviceSynchronize() != cudaSuccess) {
    cudaFree(f->d_totals);
    delete f;
    return TOPT_ERR_CUDA;
  }
  // nnz of build_filter's CSR (for topt_b200_filter_csr)
  int64_t nnz = 0;
  for (int ey = 0; ey < ny; ++ey)
    for (int ex = 0; ex < nx; ++ex)
      for (int dy = -reach; dy <= reach; ++dy) {
        const int iy = ey + dy;
        if (iy < 0 || iy >= ny) continue;
        for (int dx = -reach; dx <= reach; ++dx) {
          const int ix = ex + dx;
          if (ix < 0 || ix >= nx) continue;
          nnz += f->tab.w[(dy + reach) * f->tab.width + (dx + reach)] > 0.0;
        }
      }
  f->nnz = nnz;
  *out = f;
  return TOPT_OK;
}

void topt_b200_filter_destroy(topt_b200_filter* f) {
  if (!f) return;
  cudaFree(f->d_totals);
  delete f;
}

int64_t topt_b200_filter_nnz(const topt_b200_filter* f) { return f ? f->nnz : -1; }

// build_filter's CSR (filter.cpp:10-43), host arrays of n + 1 / nnz entries.
int topt_b200_filter_csr(const topt_b200_filter* f, int32_t* row_ptr, int32_t* col,
                         double* weight) {
  if (!f) return TOPT_ERR_INTERNAL;
  const int nx = f->nx, ny = f->ny, reach = f->tab.reach;
  int64_t k = 0;
  row_ptr[0] = 0;
  for (int ey = 0; ey < ny; ++ey)
    for (int ex = 0; ex < nx; ++ex) {
      const int64_t b = k;
      double total = 0.0;
      for (int dy = -reach; dy <= reach; ++dy) {
        const int iy = ey + dy;
        if (iy < 0 || iy >= ny) continue;
        for (int dx = -reach; dx <= reach; ++dx) {
          const int ix = ex + dx;
          if (ix < 0 || ix >= nx) continue;
          const double w = f->tab.w[(dy + reach) * f->tab.width + (dx + reach)];
          if (w <= 0.0) continue;
          col[k] = iy * nx + ix;
          weight[k] = w;
          total += w;
          ++k;
        }
      }
      for (int64_t i = b; i < k; ++i) weight[i] /= total;
      row_ptr[(int64_t)ey * nx + ex + 1] = (int32_t)k;
    }
  return TOPT_OK;
}

int topt_b200_filter_apply_dev(topt_b200_ctx* ctx, const topt_b200_filter* f, int transpose,
                               const double* in_dev, double* out_dev) {
  if (!f) return TOPT_ERR_INTERNAL;
  cudaStream_t s = (cudaStream_t)topt_b200_get_stream(ctx);
  const int64_t n = (int64_t)f->nx * f->ny;
  if (transpose)
    k_filter_chain<<<launch_grid(n), UBLOCK, 0, s>>>(f->tab, f->nx, f->ny, f->d_totals, in_dev, out_dev);
  else
    k_filter_apply<<<launch_grid(n), UBLOCK, 0, s>>>(f->tab, f->nx, f->ny, f->d_totals, in_dev, out_dev);
  return cudaGetLastError() == cudaSuccess ? TOPT_OK : TOPT_ERR_CUDA;
}

int topt_b200_filter_apply(topt_b200_ctx* ctx, const topt_b200_filter* f, int transpose,
                           const double* in, double* out) {
  if (!f) return TOPT_ERR_INTERNAL;
  const int64_t n = (int64_t)f->nx * f->ny;
  const size_t b = sizeof(double) * (size_t)n;
  double* din = (double*)g_in.get(b);
  double* dout = (double*)g_out.get(b);
  if (!din || !dout) return TOPT_ERR_CUDA;
  cudaStream_t s = (cudaStream_t)topt_b200_get_stream(ctx);
  if (cudaMemcpyAsync(din, in, b, cudaMemcpyHostToDevice, s) != cudaSuccess) return TOPT_ERR_CUDA;
  int rc = topt_b200_filter_apply_dev(ctx, f, transpose, din, dout);
  if (rc) return rc;
  if (cudaMemcpyAsync(out, dout, b, cudaMemcpyDeviceToHost, s) != cudaSuccess) return TOPT_ERR_CUDA;
  return cudaStreamSynchronize(s) == cudaSuccess ? TOPT_OK : TOPT_ERR_CUDA;
}

// Any CSR kernel (host arrays, e.g. a FilterKernel built elsewhere): W x or
// W^T x with the reference's summation orders (filter.cpp:45-69).
int topt_b200_csr_apply(topt_b200_ctx* ctx, int64_t n, const int32_t* row_ptr, const int32_t* col,
                        const double* weight, int transpose, const double* in, double* out) {
  if (n < 0) return TOPT_ERR_DOMAIN;
  if (n == 0) return TOPT_OK;
  const int64_t nnz = row_ptr[n];
  std::vector<int32_t> p2, c2;
  std::vector<double> w2;
  const int32_t *P = row_ptr, *Cc = col;
  const double* W = weight;
  if (transpose) {   // CSC: entries of each column in ascending row order
    p2.assign((size_t)n + 1, 0);
    for (int64_t k = 0; k < nnz; ++k) {
      if (col[k] < 0 || col[k] >= n) return TOPT_ERR_DOMAIN;
      p2[(size_t)col[k] + 1]++;
    }
    for (int64_t c = 0; c < n; ++c) p2[c + 1] += p2[c];
    c2.resize((size_t)nnz);
    w2.resize((size_t)nnz);
    std::vector<int32_t> fill(p2.begin(), p2.end() - 1);
    for (int64_t e = 0; e < n; ++e)
      for (int32_t k = row_ptr[e]; k < row_ptr[e + 1]; ++k) {
        const int32_t pos = fill[col[k]]++;
        c2[pos] = (int32_t)e;
        w2[pos] = weight[k];
      }
    P = p2.data(); Cc = c2.data(); W = w2.data();
  }
  cudaStream_t s = (cudaStream_t)topt_b200_get_stream(ctx);
  const size_t b = sizeof(double) * (size_t)n;
  const size_t ib = sizeof(int32_t) * (size_t)(n + 1), cb = sizeof(int32_t) * (size_t)nnz;
  char* buf = (char*)g_aux.get(ib + cb + sizeof(double) * (size_t)nnz + 64);
  double* din = (double*)g_in.get(b);
  double* dout = (double*)g_out.get(b);
  if (!buf || !din || !dout) return TOPT_ERR_CUDA;
  int32_t* dp = (int32_t*)buf;
  int32_t* dc = (int32_t*)(buf + ib);
  double* dw = (double*)(buf + ((ib + cb + 15) & ~size_t(15)));
  bool ok = cudaMemcpyAsync(dp, P, ib, cudaMemcpyHostToDevice, s) == cudaSuccess &&
            cudaMemcpyAsync(dc, Cc, cb, cudaMemcpyHostToDevice, s) == cudaSuccess &&
            cudaMemcpyAsync(dw, W, sizeof(double) * (size_t)nnz, cudaMemcpyHostToDevice, s) == cudaSuccess &&
            cudaMemcpyAsync(din, in, b, cudaMemcpyHostToDevice, s) == cudaSuccess;
  if (!ok) return TOPT_ERR_CUDA;
  if (transpose) k_csc_apply<<<launch_grid(n), UBLOCK, 0, s>>>(n, dp, dc, dw, din, dout);
  else k_csr_apply<<<launch_grid(n), UBLOCK, 0, s>>>(n, dp, dc, dw, din, dout);
  ok = cudaGetLastError() == cudaSuccess &&
       cudaMemcpyAsync(out, dout, b, cudaMemcpyDeviceToHost, s) == cudaSuccess &&
       cudaStreamSynchronize(s) == cudaSuccess;
  return ok ? TOPT_OK : TOPT_ERR_CUDA;
}

// interpolate_stiffness (material.cpp:19-46), device buffers; young (K) host.
int topt_b200_interpolate_stiffness_dev(topt_b200_ctx* ctx, int64_t n, int32_t k,
                                        const double* young, double e_min, double poisson,
                                        double penalty, const double* dens_dev,
                                        double* moduli_dev, double* der_dev) {
  // MaterialModel::validate (material.cpp:9-17)
  if (k < 1 || !(e_min > 0.0) || !(poisson > 0.0 && poisson < 0.5) || !(penalty >= 1.0))
    return TOPT_ERR_PARAMETER;
  for (int j = 0; j < k; ++j)
    if (!(young[j] > e_min)) return TOPT_ERR_PARAMETER;
  double* dy = (double*)g_aux2.get(sizeof(double) * (size_t)k + 16);
  cudaStream_t s = (cudaStream_t)topt_b200_get_stream(ctx);
  if (!dy || cudaMemcpyAsync(dy, young, sizeof(double) * (size_t)k, cudaMemcpyHostToDevice, s) != cudaSuccess)
    return TOPT_ERR_CUDA;
  int* dbad = reinterpret_cast<int*>(dy + k);
  int bad = 0;
  if (cudaMemsetAsync(dbad, 0, sizeof(int), s) != cudaSuccess) return TOPT_ERR_CUDA;
  k_range<<<launch_grid(n * k), UBLOCK, 0, s>>>(n * k, dens_dev, dbad);
  if (cudaMemcpyAsync(&bad, dbad, sizeof(int), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return TOPT_ERR_CUDA;
  if (bad) return TOPT_ERR_DOMAIN;   // "interpolate_stiffness: density outside [0,1]"
  k_simp<<<launch_grid(n), UBLOCK, 0, s>>>(n, k, dy, e_min, penalty, dens_dev, moduli_dev, der_dev);
  return cudaGetLastError() == cudaSuccess ? TOPT_OK : TOPT_ERR_CUDA;
}

// Element stiffness of the reference (fea.cpp:20-58), host.
int topt_b200_element_stiffness_q4(double poisson, double element_size, double* ke64) {
  if (!(poisson > 0.0 && poisson < 0.5) || !(element_size > 0.0)) return TOPT_ERR_PARAMETER;
  static const double xin[4] = {-1.0, 1.0, 1.0, -1.0}, etan[4] = {-1.0, -1.0, 1.0, 1.0};
  const double nu = poisson;
  const double d11 = 1.0 / (1.0 - nu * nu), d12 = nu * d11, d33 = 0.5 * (1.0 - nu) * d11;
  double ke[8][8] = {};
  const double gp = 1.0 / std::sqrt(3.0), h = element_size;
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b) {
      const double xi = a == 0 ? -gp : gp, eta = b == 0 ? -gp : gp;
      double dndx[4], dndy[4];
      for (int q = 0; q < 4; ++q) {
        dndx[q] = 0.25 * xin[q] * (1.0 + eta * etan[q]) * (2.0 / h);
        dndy[q] = 0.25 * etan[q] * (1.0 + xi * xin[q]) * (2.0 / h);
      }
      const double w = h * h / 4.0;
      for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) {
          ke[2 * i][2 * j] += w * (d11 * dndx[i] * dndx[j] + d33 * dndy[i] * dndy[j]);
          ke[2 * i][2 * j + 1] += w * (d12 * dndx[i] * dndy[j] + d33 * dndy[i] * dndx[j]);
          ke[2 * i + 1][2 * j] += w * (d12 * dndy[i] * dndx[j] + d33 * dndx[i] * dndy[j]);
          ke[2 * i + 1][2 * j + 1] += w * (d11 * dndy[i] * dndy[j] + d33 * dndx[i] * dndx[j]);
        }
    }
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) ke64[i * 8 + j] = ke[i][j];
  return TOPT_OK;
}

// Element energies and the compliance gradient from a displacement field
// (fea.cpp:162-181), device buffers: u (2 (nx+1)(ny+1)), der (N*K).
int topt_b200_compliance_gradient_dev(topt_b200_ctx* ctx, int32_t nx, int32_t ny,
                                      double element_size, double poisson, const double* u_dev,
                                      int32_t kmat, const double* der_dev, double* energy_dev,
                                      double* grad_dev) {
  Ke ke;
  int rc = topt_b200_element_stiffness_q4(poisson, element_size, ke.k);
  if (rc) return rc;
  if (nx < 1 || ny < 1 || kmat < 0) return TOPT_ERR_PARAMETER;
  cudaStream_t s = (cudaStream_t)topt_b200_get_stream(ctx);
  const int64_t n = (int64_t)nx * ny;
  k_energy_grad<<<launch_grid(n), UBLOCK, 0, s>>>(nx, ny, ke, u_dev, kmat, der_dev, energy_dev,
                                                   grad_dev);
  return cudaGetLastError() == cudaSuccess ? TOPT_OK : TOPT_ERR_CUDA;
}

}  // extern "C"
