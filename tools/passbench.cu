// passbench.cu — time individual passes of passes.cuh in isolation
// (diagnostics): a fake Plan, L2-resident inputs, CUDA-event timing.
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#define TOPT_PB_VARIANT 1
#include "../paper_2511_13905_b200/csrc/passes.cuh"
__device__ int g_pb_variant;
using namespace topt_b200;

__global__ void __launch_bounds__(BLOCK, 1) k_sweep(const Plan* plan, double* part, int mode) {
  __shared__ double s_red[NWARP * 160];
  __shared__ Cmd s_cmd;
  {
    const int* src = reinterpret_cast<const int*>(&plan->cmd);
    int* dst = reinterpret_cast<int*>(&s_cmd);
    for (int k = threadIdx.x; k < (int)(sizeof(Cmd) / 4); k += BLOCK) dst[k] = src[k];
  }
  __syncthreads();
  PassCtx c;
  c.plan = plan; c.cmd = &s_cmd; c.out = part + blockIdx.x * PMAX; c.smem = s_red;
  c.i0 = (int64_t)blockIdx.x * BLOCK + threadIdx.x; c.stride = (int64_t)gridDim.x * BLOCK;
  c.list = nullptr; c.list_cnt = nullptr; c.fixC = c.fixS = nullptr; c.list_cap = 0;
  c.seg = nullptr; c.rtab = nullptr;

  if (mode == 0) pass_sweep_row<16>(c, 0, 0, 16);
  if (mode == 1) pass_sweep_row<8>(c, 0, 0, 8);
  if (mode == 2) pass_final(c);
  if (mode == 3) pass_prep(c);
  if (mode == 4) pass_step_reduce(c);
}

int main() {
  const int64_t n = 1 << 20;
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  std::vector<double> ha(n), hr(n);
  FILE* fa = fopen("tools/c2_a.bin", "rb");
  FILE* fr = fopen("tools/c2_rho.bin", "rb");
  if (fa && fr) { fread(ha.data(), 8, n, fa); fread(hr.data(), 8, n, fr); fclose(fa); fclose(fr); }
  else for (int64_t i = 0; i < n; ++i) { ha[i] = -3.0 * (0.1 + (i % 97) * 0.009); hr[i] = -99.5 + (i % 89) * 0.01; }
  double *a, *r, *x, *part, *d;
  cudaMalloc(&a, n * 8); cudaMalloc(&r, n * 8); cudaMalloc(&x, n * 8); cudaMalloc(&d, n * 8);
  cudaMalloc(&part, (size_t)PMAX * 8 * 4096);
  cudaMemcpy(a, ha.data(), n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(r, hr.data(), n * 8, cudaMemcpyHostToDevice);
  Plan* hp = new Plan; std::memset(hp, 0, sizeof(Plan));
  hp->P.n = n; hp->P.n_global = n; hp->P.m = 1; hp->P.ld = n; hp->P.lower = 0; hp->P.upper = 1;
  hp->P.grad = a; hp->P.rho = r; hp->P.x_out = x; hp->P.x = a; hp->P.x_prev = r; hp->P.g = a; hp->P.g_prev = r;
  hp->P.d_prev = r; hp->P.d_out = d;
  hp->cmd.ncand = 16; hp->cmd.row_start[0] = 0;
  for (int j = 1; j <= MAX_M; ++j) hp->cmd.row_start[j] = 16;
  // candidates of the first C2 sweep (octave-spaced path) or of a later one
  const double first[16] = {-1411062.76, -705531.381, -352765.691, -176382.845, -88191.4226,
                            -44095.7113, -22047.8557, -11023.9278, -5511.96392, -2755.98196,
                            -1377.99098, -688.995489, -344.497745, -172.248872, -86.1244362,
                            -43.0622181};
  const double second[16] = {-42.3893709, -41.7165238, -41.3801002, -41.0436766, -40.9595707,
                             -40.9175178, -40.8964913, -40.8859781, -40.8754648, -40.707253,
                             -40.3708295, -39.0251351, -37.6794408, -34.9880522, -32.2966636,
                             -21.531109};
  const bool use_second = getenv("SECOND") != nullptr;
  for (int k = 0; k < 16; ++k) hp->cmd.cand_y[k] = use_second ? second[k] : first[k];
  hp->cmd.y[0] = -38.0; hp->cmd.write_x = 1; hp->cmd.resid_rows = 1;
  hp->cmd.compute_dir = 1; hp->cmd.use_dprev = 1; hp->cmd.beta = 0.1; hp->cmd.wa = 1.0; hp->cmd.compute_dot = 1;
  Plan* dp; cudaMalloc(&dp, sizeof(Plan)); cudaMemcpy(dp, hp, sizeof(Plan), cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[] = {"sweep K=16", "sweep K=8", "final", "prep", "step_reduce"};
  if (getenv("PB_PREP")) {
    for (int var = 0; var < 4; ++var) {
      cudaMemcpyToSymbol(g_pb_variant, &var, sizeof(int));
      for (int w = 0; w < 3; ++w) k_sweep<<<nsm, BLOCK>>>(dp, part, 3);
      cudaEventRecord(e0);
      for (int w = 0; w < 20; ++w) k_sweep<<<nsm, BLOCK>>>(dp, part, 3);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("prep variant %d %8.2f us/launch\n", var, ms * 1e3 / 20);
    }
    for (int var = 0; var < 2; ++var) {   // empty kernel baseline
      cudaEventRecord(e0);
      for (int w = 0; w < 20; ++w) k_sweep<<<nsm, BLOCK>>>(dp, part, 99);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("empty launch %8.2f us/launch\n", ms * 1e3 / 20);
    }
    return 0;
  }
  for (int grid_mult : {1, 2, 4})
  for (int mode = 0; mode < 5; ++mode) {
    const int grid = nsm * grid_mult;
    for (int w = 0; w < 3; ++w) k_sweep<<<grid, BLOCK>>>(dp, part, mode);
    cudaEventRecord(e0);
    const int reps = 20;
    for (int w = 0; w < reps; ++w) k_sweep<<<grid, BLOCK>>>(dp, part, mode);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("grid %4d %-12s %8.2f us/launch\n", grid, names[mode], ms * 1e3 / reps);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
