// fp64 pipe throughput probe (diagnostics): ops per SM per cycle for DFMA,
// DMUL, DADD, DSETP+select, with 8 independent chains per thread.
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(double* out, int iters, double s) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) a[i] = fma(a[i], s, 0.25);
      if (OP == 1) a[i] = a[i] * s;
      if (OP == 2) a[i] = a[i] + s;
      if (OP == 3) a[i] = (a[i] < s) ? a[i] + 1.0 : a[i] - 1.0;      // DSETP + DADD + select
      if (OP == 4) { double v = a[i] * s; a[i] = v < 0.5 ? 0.5 : (v > 2.0 ? 2.0 : v); }  // clip
    }
  }
  long long t1 = clock64();
  double r = 0; for (int i = 0; i < 8; ++i) r += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (double)(t1 - t0);
}

int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* o; cudaMalloc(&o, sizeof(double) * nsm * 1024);
  const char* names[] = {"DFMA", "DMUL", "DADD", "DSETP+DADD+sel", "DMUL+clip"};
  const int iters = 4096;
  for (int op = 0; op < 5; ++op) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto launch = [&]() {
      if (op == 0) k<0><<<nsm, 1024>>>(o, iters, 1.0000001);
      if (op == 1) k<1><<<nsm, 1024>>>(o, iters, 1.0000001);
      if (op == 2) k<2><<<nsm, 1024>>>(o, iters, 1.0000001);
      if (op == 3) k<3><<<nsm, 1024>>>(o, iters, 1.0000001);
      if (op == 4) k<4><<<nsm, 1024>>>(o, iters, 1.0000001);
    };
    launch();
    cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)nsm * 1024 * iters * 8;
    printf("%-16s %.1f Gop/s  = %.1f lane-ops/clk/SM (at 1.965 GHz)\n", names[op],
           ops / ms / 1e6, ops / (ms * 1e-3) / nsm / 1.965e9);
  }
  return 0;
}
