// streambench.cu -- throughput of the TMA row-streaming engine (passes.cuh
// stream_tiles) against plain vectorised loads, on R rows of n doubles.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include "../paper_2511_13905_b200/csrc/passes.cuh"
using namespace topt_b200;

__global__ void __launch_bounds__(BLOCK, 1) k_stream(const double* base, int64_t n, int nr,
                                                      double* out, int heavy) {
  extern __shared__ __align__(128) char sm[];
  PassCtx c{};
  c.st_bar = reinterpret_cast<uint64_t*>(sm);
  c.st_buf = reinterpret_cast<double*>(sm + 128);
  StreamRows R;
  R.nr = nr;
  for (int r = 0; r < nr; ++r) R.row[r] = base + (int64_t)r * n;
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  stream_tiles(c, R, n, [&](int64_t, const double* v, bool ok) {
    if (!ok) return;
    double a[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) a[r] = r < nr ? v[r * ST_T] : 0.0;
    if (heavy) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[(j + k) & 7] += a[j] * a[k];
    } else {
#pragma unroll
      for (int r = 0; r < 8; ++r) acc[r] += a[r];
    }
  });
  double t = 0;
  for (int r = 0; r < 8; ++r) t += acc[r];
  if (t == 12345.678) out[0] = t;
}

__global__ void __launch_bounds__(BLOCK, 1) k_plain(const double* base, int64_t n, int nr,
                                                     double* out) {
  double acc = 0;
  const int64_t st = (int64_t)gridDim.x * BLOCK;
  const double2* b2 = reinterpret_cast<const double2*>(base);
  const int64_t n2 = n / 2;
  for (int64_t q = (int64_t)blockIdx.x * BLOCK + threadIdx.x; q < n2; q += st) {
    double2 v[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) v[r] = r < nr ? b2[(int64_t)r * n2 + q] : make_double2(0, 0);
#pragma unroll
    for (int r = 0; r < 8; ++r) acc += v[r].x + v[r].y;
  }
  if (acc == 12345.678) out[0] = acc;
}

int main() {
  const int64_t n = 8388608;
  const int nr = 8;
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double *base, *out, *flush;
  cudaMalloc(&base, sizeof(double) * n * nr);
  cudaMalloc(&out, 64);
  cudaMalloc(&flush, 256 << 20);
  cudaMemset(base, 0, sizeof(double) * n * nr);
  const size_t smem = STREAM_SMEM;
  cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const double bytes = 8.0 * n * nr;
  for (int rep = 0; rep < 2; ++rep)
  for (int mode = 0; mode < 3; ++mode) {
    float best = 1e9;
    for (int it = 0; it < 5; ++it) {
      cudaMemset(flush, it, 256 << 20);
      cudaEventRecord(e0);
      if (mode == 0) k_plain<<<nsm, BLOCK>>>(base, n, nr, out);
      else k_stream<<<nsm, BLOCK, smem>>>(base, n, nr, out, mode == 2);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    const char* nm[] = {"plain double2 x8 rows", "TMA stream (light)", "TMA stream (64 fma/elem)"};
    printf("%-28s %8.1f us  %7.0f GB/s\n", nm[mode], best * 1e3, bytes / (best * 1e-3) / 1e9);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
