// compactbench.cu — the compacted sweep (pass_sweep_row_compact) in isolation
// on C2 data: lists built by compact_init, then one compacted sweep with a
// given walk window (diagnostics).
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_2511_13905_b200/csrc/passes.cuh"
using namespace topt_b200;

__global__ void __launch_bounds__(BLOCK, 1) k_cs(const Plan* plan, double* part, int mode, int reps) {
  __shared__ double s_red[NWARP * 160];
  __shared__ Cmd s_cmd;
  __shared__ double s_fixC[MAX_M], s_fixS[MAX_M];
  __shared__ int s_lcnt[NWARP];
  extern __shared__ uint32_t s_list[];
  {
    const int* src = reinterpret_cast<const int*>(&plan->cmd);
    int* dst = reinterpret_cast<int*>(&s_cmd);
    for (int k = threadIdx.x; k < (int)(sizeof(Cmd) / 4); k += BLOCK) dst[k] = src[k];
  }
  __syncthreads();
  PassCtx c;
  c.plan = plan; c.cmd = &s_cmd; c.out = part + blockIdx.x * PMAX; c.smem = s_red;
  c.i0 = (int64_t)blockIdx.x * BLOCK + threadIdx.x; c.stride = (int64_t)gridDim.x * BLOCK;
  c.list = s_list; c.list_cnt = s_lcnt; c.fixC = s_fixC; c.fixS = s_fixS;
  c.list_cap = plan->P.compact_cap;
  c.timed_out = nullptr;
  for (int r = 0; r < reps; ++r) {
    compact_init(c);
    if (mode == 1) { pass_sweep_row_compact<16>(c, 0, 0, 16); }
  }
}

int main(int argc, char** argv) {
  const int64_t n = 1 << 20;
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  std::vector<double> ha(n), hr(n);
  FILE* f = fopen("tools/c2_a.bin", "rb"); fread(ha.data(), 8, n, f); fclose(f);
  f = fopen("tools/c2_rho.bin", "rb"); fread(hr.data(), 8, n, f); fclose(f);
  double *a, *r, *part;
  cudaMalloc(&a, n * 8); cudaMalloc(&r, n * 8); cudaMalloc(&part, (size_t)PMAX * 8 * 1024);
  cudaMemcpy(a, ha.data(), n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(r, hr.data(), n * 8, cudaMemcpyHostToDevice);
  const int grid = nsm;
  const int64_t per_thread = (n + (int64_t)grid * BLOCK - 1) / ((int64_t)grid * BLOCK);
  Plan* hp = new Plan; std::memset(hp, 0, sizeof(Plan));
  hp->P.n = n; hp->P.n_global = n; hp->P.m = 1; hp->P.ld = n; hp->P.lower = 0; hp->P.upper = 1;
  hp->P.grad = a; hp->P.rho = r; hp->P.compact_cap = (int)(32 * per_thread);
  hp->cmd.ncand = 16; hp->cmd.row_start[0] = 0;
  for (int j = 1; j <= MAX_M; ++j) hp->cmd.row_start[j] = 16;
  // candidates: around the C2 root (-38.49), window per argv
  const double wlo = argc > 1 ? atof(argv[1]) : -1411062.0, whi = argc > 2 ? atof(argv[2]) : 0.0;
  for (int k = 0; k < 16; ++k) hp->cmd.cand_y[k] = wlo + (whi - wlo) * (k + 0.5) / 16.0;
  hp->cmd.wlo[0] = wlo; hp->cmd.whi[0] = whi; hp->cmd.compact = 1;
  Plan* dp; cudaMalloc(&dp, sizeof(Plan)); cudaMemcpy(dp, hp, sizeof(Plan), cudaMemcpyHostToDevice);
  const int smem = NWARP * hp->P.compact_cap * 4;
  cudaFuncSetAttribute(k_cs, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int mode = 0; mode < 2; ++mode) {
    k_cs<<<grid, BLOCK, smem>>>(dp, part, mode, 2);
    cudaEventRecord(e0);
    const int reps = 20;
    k_cs<<<grid, BLOCK, smem>>>(dp, part, mode, reps);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("window [%g, %g] mode %d (%s): %.2f us per rep\n", wlo, whi, mode,
           mode ? "init + compact sweep" : "init only", ms * 1e3 / reps);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
