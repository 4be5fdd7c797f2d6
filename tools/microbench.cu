// microbench.cu — grid-barrier and single-thread latency probes (diagnostics).
#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

struct Sync { unsigned count, gen; };

__device__ __forceinline__ unsigned ldv(const unsigned* p) {
  unsigned v; asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}

__global__ void k_bar(Sync* s, int iters, double* part, int work) {
  __shared__ unsigned gen;
  __shared__ int last;
  for (int it = 0; it < iters; ++it) {
    if (work) part[blockIdx.x * 64 + (threadIdx.x & 63)] = it;
    __syncthreads();
    if (threadIdx.x == 0) {
      gen = ldv(&s->gen);
      __threadfence();
      last = atomicAdd(&s->count, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last) {
      if (threadIdx.x == 0) { s->count = 0; __threadfence(); atomicExch(&s->gen, gen + 1); }
    } else {
      if (threadIdx.x == 0) { while (ldv(&s->gen) == gen) {} __threadfence(); }
    }
    __syncthreads();
  }
}

__global__ void k_cgbar(int iters) {
  cg::grid_group g = cg::this_grid();
  for (int it = 0; it < iters; ++it) g.sync();
}

__global__ void k_serial(double* out, int iters) {
  __shared__ double sm[64];
  if (threadIdx.x != 0) return;
  double a = out[0];
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) { sm[i & 63] = a; a = sm[(i * 7) & 63] * 1.0000001 + 0.5; }
  long long t1 = clock64();
  out[1] = a;
  out[2] = (double)(t1 - t0) / iters;
  double b = out[0];
  t0 = clock64();
  for (int i = 0; i < iters; ++i) b = b * 1.0000001 + 0.25;
  t1 = clock64();
  out[3] = b;
  out[4] = (double)(t1 - t0) / iters;
}

int main() {
  int dev = 0, nsm = 0; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  Sync* s; cudaMalloc(&s, sizeof(Sync)); cudaMemset(s, 0, sizeof(Sync));
  double* part; cudaMalloc(&part, 1 << 20);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int bps : {1, 2}) for (int work : {0, 1}) {
    int grid = nsm * bps, iters = 2000;
    void* args[] = {&s, &iters, &part, &work};
    cudaLaunchCooperativeKernel((void*)k_bar, grid, 256, args, 0, 0);
    cudaEventRecord(e0);
    cudaLaunchCooperativeKernel((void*)k_bar, grid, 256, args, 0, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("custom barrier grid=%d work=%d: %.3f us/barrier\n", grid, work, ms * 1e3 / iters);
  }
  for (int bps : {1, 2}) {
    int grid = nsm * bps, iters = 2000;
    void* args[] = {&iters};
    cudaLaunchCooperativeKernel((void*)k_cgbar, grid, 256, args, 0, 0);
    cudaEventRecord(e0);
    cudaLaunchCooperativeKernel((void*)k_cgbar, grid, 256, args, 0, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("cg grid.sync grid=%d: %.3f us/barrier\n", grid, ms * 1e3 / iters);
  }
  double* o; cudaMalloc(&o, 64); cudaMemset(o, 0, 64);
  k_serial<<<1, 32>>>(o, 10000);
  double h[5]; cudaMemcpy(h, o, sizeof(h), cudaMemcpyDeviceToHost);
  printf("single thread: smem st+ld+dfma chain %.1f cyc/iter, dfma chain %.1f cyc/iter\n", h[2], h[4]);
  cudaError_t e = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
