// Sequential-sum ("chain") throughput probe (diagnostics only).
//  (1) dependent DADD latency on one thread;
//  (2) one CTA: producer warps stage (a, rho) tiles in shared memory through a
//      named-barrier ring, consumer lanes each run one reference-order sum
//      s += a * clip(y_lane * a, lo, hi) over all n elements;
// reports cycles per element (the exact-parity evaluation's cost model).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_lat(double* out, int iters, double t) {
  double s = threadIdx.x;
  long long c0 = clock64();
  for (int i = 0; i < iters; ++i) s = __dadd_rn(s, t);
  long long c1 = clock64();
  out[0] = s;
  out[1] = (double)(c1 - c0) / iters;
}

constexpr int TE = 64;       // elements per tile
constexpr int NSLOT = 4;     // ring slots
template <int NCONS>
__global__ void __launch_bounds__(512, 1) k_chain(const double* a, const double* rho, long n,
                                                  double* out, double* cyc) {
  __shared__ double s_a[NSLOT][TE], s_lo[NSLOT][TE], s_hi[NSLOT][TE];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nprod = (blockDim.x >> 5) - NCONS;
  const long ntile = (n + TE - 1) / TE;
  long long c0 = clock64();
  if (warp >= NCONS) {   // producers
    const int pt = (warp - NCONS) * 32 + lane, np = nprod * 32;
    for (long t = 0; t < ntile; ++t) {
      const int s = t % NSLOT;
      if (t >= NSLOT) asm volatile("bar.sync %0, %1;" ::"r"(1 + NSLOT + s), "r"(blockDim.x));
      for (int e = pt; e < TE; e += np) {
        const long i = t * TE + e;
        const double av = i < n ? a[i] : 0.0, r = i < n ? rho[i] : 0.0;
        s_a[s][e] = av;
        s_lo[s][e] = __dsub_rn(0.0, r);
        s_hi[s][e] = __dsub_rn(1.0, r);
      }
      __threadfence_block();
      asm volatile("bar.arrive %0, %1;" ::"r"(1 + s), "r"(blockDim.x));
    }
  } else {
    const double y = -1e-3 * (1 + warp * 32 + lane);
    double acc = 0.0;
    for (long t = 0; t < ntile; ++t) {
      const int s = t % NSLOT;
      asm volatile("bar.sync %0, %1;" ::"r"(1 + s), "r"(blockDim.x));
      const int ne = (t + 1) * TE <= n ? TE : (int)(n - t * TE);
#pragma unroll 8
      for (int e = 0; e < ne; ++e) {
        const double av = s_a[s][e], lo = s_lo[s][e], hi = s_hi[s][e];
        const double v = __dmul_rn(y, av);
        const double c = v < lo ? lo : (v > hi ? hi : v);
        acc = __dadd_rn(acc, __dmul_rn(av, c));
      }
      if (t + NSLOT < ntile) asm volatile("bar.arrive %0, %1;" ::"r"(1 + NSLOT + s), "r"(blockDim.x));
    }
    out[warp * 32 + lane] = acc;
  }
  long long c1 = clock64();
  if (threadIdx.x == 0) cyc[0] = (double)(c1 - c0) / n;
}

int main() {
  const long n = 1 << 23;
  double *a, *rho, *out, *cyc;
  cudaMalloc(&a, n * 8); cudaMalloc(&rho, n * 8);
  cudaMalloc(&out, 4096 * 8); cudaMallocManaged(&cyc, 64);
  cudaMemset(a, 0, n * 8); cudaMemset(rho, 0, n * 8);
  k_lat<<<1, 1>>>(out, 1 << 20, 1.0000001);
  cudaDeviceSynchronize();
  double h[2];
  cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
  printf("DADD dependent latency: %.2f cycles\n", h[1]);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_chain<1><<<1, 512>>>(a, rho, n, out, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("chain 1 consumer warp (32 sums): %.3f ms for n=%ld, %.2f cycles/elem (%s)\n", ms, n,
           cyc[0], cudaGetErrorString(cudaGetLastError()));
    cudaEventRecord(e0);
    k_chain<2><<<1, 512>>>(a, rho, n, out, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("chain 2 consumer warps (64 sums): %.3f ms, %.2f cycles/elem\n", ms, cyc[0]);
    cudaEventRecord(e0);
    k_chain<4><<<1, 512>>>(a, rho, n, out, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("chain 4 consumer warps (128 sums): %.3f ms, %.2f cycles/elem\n", ms, cyc[0]);
  }
  return 0;
}
