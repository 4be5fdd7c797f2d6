// histbench.cu — cost of a breakpoint histogram in shared memory (diagnostics)
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
constexpr int BLOCK = 512, SUB = 8, NB = 128 * SUB;
__device__ __forceinline__ int bidx(float y) {
  const int bits = __float_as_int(fabsf(y));
  const int e = ((bits >> 23) & 0xff) - 127;
  const int m = (bits >> 20) & (SUB - 1);
  int k = (e + 32) * SUB + m;
  k = k < 0 ? 0 : (k > 64 * SUB - 1 ? 64 * SUB - 1 : k);
  return y < 0.f ? 64 * SUB - 1 - k : 64 * SUB + k;
}
__global__ void __launch_bounds__(BLOCK, 1) k_hist(const double* a, const double* rho, long n,
                                                   float* out, int mode, double* dummy) {
  __shared__ float h[4 * NB];
  for (int i = threadIdx.x; i < 4 * NB; i += BLOCK) h[i] = 0.f;
  __syncthreads();
  double acc = 0;
  for (long i = blockIdx.x * (long)BLOCK + threadIdx.x; i < n; i += (long)gridDim.x * BLOCK) {
    const double av = a[i], r = rho[i];
    if (av == 0.0) continue;
    const float fa = (float)av, ra = __frcp_rn(fa);
    const float lo = (float)(0.0 - r), hi = (float)(1.0 - r);
    const float b1 = lo * ra, b2 = hi * ra;
    const bool pos = fa > 0.f;
    const float bl = pos ? b1 : b2, bh = pos ? b2 : b1;
    const float cl = fa * (pos ? lo : hi), ch = fa * (pos ? hi : lo), aa = fa * fa;
    const int il = bidx(bl), ih = bidx(bh);
    if (mode == 0) { acc += il + ih + cl + ch + aa; continue; }
    if (mode == 1) {
      atomicAdd(&h[il], cl); atomicAdd(&h[NB + il], aa);
      atomicAdd(&h[2 * NB + ih], ch); atomicAdd(&h[3 * NB + ih], aa);
    } else if (mode == 2) {
      atomicAdd(&h[il], cl); atomicAdd(&h[2 * NB + ih], ch);
    } else if (mode == 3) {  // warp-aggregated by bucket (match_any)
      const unsigned g1 = __match_any_sync(__activemask(), il);
      const int l1 = __ffs(g1) - 1;
      // leader sums its group via shuffles over the group's lanes
      float s_cl = 0.f, s_aa = 0.f;
      for (unsigned m = g1; m; m &= m - 1) {
        const int src = __ffs(m) - 1;
        s_cl += __shfl_sync(g1, cl, src); s_aa += __shfl_sync(g1, aa, src);
      }
      if ((int)(threadIdx.x & 31) == l1) { atomicAdd(&h[il], s_cl); atomicAdd(&h[NB + il], s_aa); }
      const unsigned g2 = __match_any_sync(__activemask(), ih);
      const int l2 = __ffs(g2) - 1;
      float s_ch = 0.f, s_ah = 0.f;
      for (unsigned m = g2; m; m &= m - 1) {
        const int src = __ffs(m) - 1;
        s_ch += __shfl_sync(g2, ch, src); s_ah += __shfl_sync(g2, aa, src);
      }
      if ((int)(threadIdx.x & 31) == l2) { atomicAdd(&h[2 * NB + ih], s_ch); atomicAdd(&h[3 * NB + ih], s_ah); }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 4 * NB; i += BLOCK) out[(long)blockIdx.x * 4 * NB + i] = h[i];
  if (acc == 12345.0) dummy[0] = acc;
}
int main() {
  const long n = 1 << 20;
  std::vector<double> ha(n), hr(n);
  FILE* f = fopen("tools/c2_a.bin", "rb"); fread(ha.data(), 8, n, f); fclose(f);
  f = fopen("tools/c2_rho.bin", "rb"); fread(hr.data(), 8, n, f); fclose(f);
  double *a, *r, *dm; float* out;
  cudaMalloc(&a, n * 8); cudaMalloc(&r, n * 8); cudaMalloc(&dm, 8);
  cudaMalloc(&out, 4096L * 4 * NB * 4);
  cudaMemcpy(a, ha.data(), n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(r, hr.data(), n * 8, cudaMemcpyHostToDevice);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int mode = 0; mode < 4; ++mode) {
    for (int w = 0; w < 3; ++w) k_hist<<<nsm, BLOCK>>>(a, r, n, out, mode, dm);
    cudaEventRecord(e0);
    for (int w = 0; w < 20; ++w) k_hist<<<nsm, BLOCK>>>(a, r, n, out, mode, dm);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("mode %d: %.2f us\n", mode, ms * 1e3 / 20);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
