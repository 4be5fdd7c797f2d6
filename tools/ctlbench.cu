// ctlbench.cu — cycles of one controller step (plan_consume_warp) on a Plan
// snapshot taken from the host simulator (diagnostics).

#define TOPT_CTL_MARK_SMEM 1
#include <cstdio>
#include <vector>
#include <cstdlib>
#include <cooperative_groups.h>
#include "../paper_2511_13905_b200/csrc/passes.cuh"
using namespace topt_b200;

__global__ void __launch_bounds__(512, 1) k_ctl(const Plan* gplan, const double* gt, int nt,
                                                long long* cyc, int reps, unsigned long long* marks, int scalar) {
  extern __shared__ int4 s_dyn[];
  Plan& sp = *reinterpret_cast<Plan*>(s_dyn);
  __shared__ double s_t[PMAX];
  for (int r = 0; r < reps; ++r) {
    const int* src = reinterpret_cast<const int*>(gplan);
    int* dst = reinterpret_cast<int*>(&sp);
    for (int k = threadIdx.x; k < (int)(offsetof(Plan, sc) / 4); k += 512) dst[k] = src[k];
    for (int k = threadIdx.x; k < nt; k += 512) s_t[k] = gt[k];
    __syncthreads();
    (void)marks;
    if (threadIdx.x < 16) ctl_marks_smem()[threadIdx.x] = 0;
    __syncthreads();
    long long t0 = clock64();

    if (scalar) { if (threadIdx.x == 0) plan_consume(sp, s_t); }
    else if (threadIdx.x < 32) plan_consume_warp(sp, s_t);
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[r] = t1 - t0;
    if (r == reps - 1 && threadIdx.x < MAX_CAND) {
      reinterpret_cast<double*>(marks + 2048)[threadIdx.x] = sp.cmd.cand_y[threadIdx.x];
      if (threadIdx.x == 0) marks[2047] = sp.cmd.row_start[1];
    }
    if (threadIdx.x < 16) marks[16 * r + threadIdx.x] = ctl_marks_smem()[threadIdx.x] ? ctl_marks_smem()[threadIdx.x] - t0 : 0;
    __syncthreads();
  }
}

int main(int argc, char** argv) {
  for (int f = 1; f < argc; f += 2) {
    FILE* fp = fopen(argv[f], "rb");
    std::vector<char> pb(sizeof(Plan));
    size_t got = fread(pb.data(), 1, sizeof(Plan), fp); fclose(fp);
    fp = fopen(argv[f + 1], "rb");
    std::vector<double> t(PMAX);
    int nt = (int)fread(t.data(), 8, PMAX, fp); fclose(fp);
    Plan* dp; double* dt; long long* dc; unsigned long long* dm;
    cudaMalloc(&dp, sizeof(Plan)); cudaMalloc(&dt, PMAX * 8); cudaMalloc(&dc, 100000 * 8);
    cudaMalloc(&dm, 100000 * 8); cudaMemset(dm, 0, 100000 * 8);
    cudaMemcpy(dp, pb.data(), sizeof(Plan), cudaMemcpyHostToDevice);
    cudaMemcpy(dt, t.data(), PMAX * 8, cudaMemcpyHostToDevice);
    const int smem = (int)sizeof(Plan);
    cudaFuncSetAttribute(k_ctl, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int reps = getenv("REPS") ? atoi(getenv("REPS")) : 4;
    k_ctl<<<1, 512, smem>>>(dp, dt, nt, dc, reps, dm, getenv("CTL_SCALAR") != nullptr);
    long long c[64];
    cudaMemcpy(c, dc, 4 * 8, cudaMemcpyDeviceToHost);
    printf("%s (plan %zu B read %zu, %d totals): cycles %lld %lld %lld %lld  err=%s\n", argv[f],
           sizeof(Plan), got, nt, c[0], c[1], c[2], c[3], cudaGetErrorString(cudaGetLastError()));
    unsigned long long mk[64];
    {
      unsigned long long nc;
      double cy[MAX_CAND];
      cudaMemcpy(&nc, dm + 2047, 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(cy, dm + 2048, sizeof(cy), cudaMemcpyDeviceToHost);
      printf("   cand (%llu):", nc);
      for (unsigned long long k = 0; k < nc && k < MAX_CAND; ++k) printf(" %.9g", cy[k]);
      printf("\n");
    }
    cudaMemcpy(mk, dm, 64 * 8, cudaMemcpyDeviceToHost);
    printf("   marks (rep 3, cycles from start):");
    for (int k = 0; k < 16; ++k) if (mk[48 + k]) printf(" %d:%lld", k, (long long)mk[48 + k]);
    printf("\n");
  }
}
