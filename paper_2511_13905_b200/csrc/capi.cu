// capi.cu — kernels that drive the passes + the extern "C" boundary.
//
// Launch model (single GPU).  One kernel launch per pass: every CTA sweeps
// its grid-stride share of the slab and writes its partial slots; the CTA
// that finishes last (atomic ticket) combines all CTAs' partials in a fixed
// order and runs the controller (controller.h) on the device, which writes
// the next pass's command into the device-resident Plan.  The host only
// relaunches and polls one int (the next phase); no partial sum or decision
// ever crosses PCIe.
#include <cooperative_groups.h>
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstddef>
#include <cstdio>
#include <cstring>
#include <chrono>
#include <string>
#include <thread>
#include <vector>

#include "../../include/topt_b200.h"
#include "controller.h"
#include "passes.cuh"
#include "topt_core.h"

using namespace topt_b200;
namespace cg = cooperative_groups;

namespace {

constexpr int RED_SCRATCH = NWARP * 160;   // doubles (max NS = 16 + 136)
constexpr size_t PLAN_SMEM = (sizeof(Plan) + 255) & ~size_t(255);
constexpr size_t KPASS_SMEM = PLAN_SMEM;   // + the structured-row tables

// Combine all CTAs' partial slots in a fixed order into totals[].  Group g
// sums CTAs g, g+G, g+2G, ... sequentially (loads batched 8 deep, the
// addition order unchanged); groups combine in order.  The order depends only
// on (nb, ns): deterministic.
__device__ void finish_reduce(const double* partials, int nb, int ns, int phase,
                              double* totals, double* smem, int stride = PMAX);
// FEAS with Newton's first evaluation appended (cmd.feas_gram0): the appended
// slots are combined on their own, i.e. in the CTA grouping a NEWTON pass of
// the same slot count uses, so the evaluation has the bits that pass would give.
__device__ void finish_reduce_cmd(const double* partials, int nb, const topt_b200::Cmd& cmd,
                                  int m, double* totals, double* smem) {
  if (cmd.phase == topt_b200::PH_FEAS && cmd.feas_gram0) {
    const int n1 = cmd.nfeas * m;
    finish_reduce(partials, nb, n1, cmd.phase, totals, smem);
    finish_reduce(partials + n1, nb, cmd.nslots - n1, cmd.phase, totals + n1, smem);
    return;
  }
  finish_reduce(partials, nb, cmd.nslots, cmd.phase, totals, smem);
}
__device__ void finish_reduce(const double* partials, int nb, int ns, int phase,
                              double* totals, double* smem, int stride) {
  for (int s0 = 0; s0 < ns; s0 += BLOCK) {
    const int per = min(ns - s0, BLOCK);
    // G groups of CTAs per slot: ~sqrt(nb) balances the load chain (nb / G
    // loads, issued together) against the in-order combine of the G groups
    int G = BLOCK / per;
    if (G > nb) G = nb;
    if (G > 16) G = 16;
    if (G < 1) G = 1;
    const int t = threadIdx.x;
    const int s = t % per, g = t / per;
    if (g < G) {
      const int op = slot_op(phase, s0 + s);
      const double* src = partials + s0 + s;
      // issue every load of this thread's chain before combining (MLP)
      constexpr int CH = 16;
      double r = __ldcg(src + (size_t)g * stride);
      for (int b0 = g + G; b0 < nb; b0 += CH * G) {
        double v[CH];
#pragma unroll
        for (int k = 0; k < CH; ++k) {
          const int b = b0 + k * G;
          v[k] = (b < nb) ? __ldcg(src + (size_t)b * stride) : 0.0;
        }
#pragma unroll
        for (int k = 0; k < CH; ++k)
          if (b0 + k * G < nb) r = apply_op(op, r, v[k]);
      }
      smem[g * per + s] = r;
    }
    __syncthreads();
    if (t < per) {
      const int op = slot_op(phase, s0 + t);
      double r = smem[t];
      for (int gg = 1; gg < G; ++gg) r = apply_op(op, r, smem[gg * per + t]);
      totals[s0 + t] = r;
    }
    __syncthreads();
  }
}

// Copy the device-resident Plan into this CTA's shared memory, run the
// controller on it (thread 0), and write it back.  The controller's many
// small dependent accesses then see shared-memory latency, not L2.
__device__ __forceinline__ void copy_words(int* dst, const int* src, int nwords, bool cg_store) {
  for (int k = threadIdx.x; k < nwords; k += BLOCK) {
    const int v = __ldcg(src + k);
    if (cg_store) __stcg(dst + k, v); else dst[k] = v;
  }
}

__device__ void control_step(Plan* plan, Plan* s_plan, const double* totals) {
  // live controller state: [0, walks of the m rows) and [nt, sc); the
  // Problem is read-only and Scratch is scratch.
  const int m = plan->P.m;
  const int endA = (int)(offsetof(Plan, w) + sizeof(Walk) * (size_t)m) / 4;
  const int begB = (int)offsetof(Plan, nt) / 4, endB = (int)offsetof(Plan, sc) / 4;
  const int begCmd = (int)offsetof(Plan, cmd) / 4;
  int* gp = reinterpret_cast<int*>(plan);
  int* sp = reinterpret_cast<int*>(s_plan);
  copy_words(sp, gp, endA, false);
  copy_words(sp + begB, gp + begB, endB - begB, false);
  __syncthreads();
  if (threadIdx.x == 0) plan_consume(*s_plan, totals);
  __syncthreads();
  for (int k = begCmd + threadIdx.x; k < endA; k += BLOCK) __stcg(gp + k, sp[k]);
  for (int k = begB + threadIdx.x; k < endB; k += BLOCK) __stcg(gp + k, sp[k]);
  __threadfence();
  __syncthreads();
}

__device__ __forceinline__ void load_cmd(const Plan* plan, Cmd* s_cmd) {
  const int* src = reinterpret_cast<const int*>(&plan->cmd);
  int* dst = reinterpret_cast<int*>(s_cmd);
  for (int k = threadIdx.x; k < (int)(sizeof(Cmd) / sizeof(int)); k += BLOCK)
    dst[k] = __ldcg(src + k);
  __syncthreads();
}

// Multi-launch mode: one launch per pass; the last CTA runs the controller
// (single rank), or -- rank mode, totals != nullptr -- writes this rank's
// combined partial vector to totals[] for the cross-rank all-gather.
__global__ void __launch_bounds__(BLOCK, 1) k_pass(Plan* plan, double* partials,
                                                unsigned* counter, double* totals) {
  __shared__ Cmd s_cmd;
  __shared__ double s_red[RED_SCRATCH];
  __shared__ double s_tot[PMAX];
  __shared__ int s_last;
  extern __shared__ int4 s_dyn[];
  load_cmd(plan, &s_cmd);
  if (s_cmd.phase == PH_DONE) return;
  PassCtx c;
  c.plan = plan;
  c.cmd = &s_cmd;
  c.out = partials + (size_t)blockIdx.x * PMAX;
  c.smem = s_red;
  c.i0 = (int64_t)blockIdx.x * BLOCK + threadIdx.x;
  c.stride = (int64_t)gridDim.x * BLOCK;
  c.list = nullptr;
  c.list_cnt = nullptr;
  c.seg = nullptr;
  c.fixC = c.fixS = nullptr;
  c.list_cap = 0;
  c.timed_out = nullptr;   // never streamed
  c.ex_smem = nullptr;     // (strict parity runs in the persistent kernel only)
  c.ms_smem = nullptr;
  double* s_rtab = reinterpret_cast<double*>(reinterpret_cast<char*>(s_dyn) + PLAN_SMEM);
  c.rtab = s_rtab;
  build_row_tables(plan->P, s_rtab);
  __syncthreads();
  run_pass(c);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  finish_reduce_cmd(partials, gridDim.x, s_cmd, plan->P.m, s_tot, s_red);
  if (totals) {   // rank mode: publish this rank's totals, no control here
    for (int s = threadIdx.x; s < s_cmd.nslots; s += BLOCK) totals[s] = s_tot[s];
  } else {
    control_step(plan, reinterpret_cast<Plan*>(s_dyn), s_tot);
  }
  if (threadIdx.x == 0) {
    *counter = 0u;
    __threadfence();
  }
}

// Rank mode: combine the all-gathered per-rank totals in rank order (every
// rank computes the same bits) and run the controller on the device.
__global__ void __launch_bounds__(BLOCK, 1) k_control(Plan* plan, const double* gathered,
                                                   int world) {
  __shared__ double s_tot[PMAX];
  extern __shared__ int4 s_dyn[];
  const int ns = plan->cmd.nslots, phase = plan->cmd.phase;
  if (phase == PH_DONE) return;
  for (int s = threadIdx.x; s < ns; s += BLOCK) {
    const int op = slot_op(phase, s);
    double r = gathered[s];
    for (int q = 1; q < world; ++q) r = apply_op(op, r, gathered[(size_t)q * PMAX + s]);
    s_tot[s] = r;
  }
  __syncthreads();
  control_step(plan, reinterpret_cast<Plan*>(s_dyn), s_tot);
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Persistent mode: ONE cooperative launch runs every pass of the job.
// Every CTA holds a private shared-memory copy of the controller state; after
// each pass the CTAs meet at a grid barrier, then EVERY CTA combines all
// partials in the same fixed order and runs the same controller step, so all
// CTAs hold bit-identical commands without a second barrier or any global
// command broadcast.  Partials are double-buffered across passes.

struct GatherBufs {
  int* blk_cnt;
  double* g_a;
  double* g_r;
  int* g_row;
  double* g_fix;
  int* timed_out;   // streamed input never arrived (host checks after the launch)
};

// d is final once PREP's grid barrier has passed: release it to the copy
// stream waiting on out_flag (system scope: a copy engine reads it).
__device__ __forceinline__ void signal_out(const Problem& P) {
  if (P.chunk > 0 && P.out_flag) {
    __threadfence_system();
    asm volatile("st.release.sys.global.u32 [%0], %1;" :: "l"(P.out_flag), "r"(P.epoch) : "memory");
  }
}

// The controller state travels as a kernel parameter (no separate upload).
constexpr size_t PLAN_WORDS = offsetof(Plan, sc) / 4;
struct PlanBlob {
  int w[PLAN_WORDS];
};

#ifdef TOPT_ICACHE_EXPERIMENT
__device__ Plan g_plan_scratch[160];
#endif
// MULTI: the CTA-level controller (rows spread over warps, m > 1); the
// single-row instantiation keeps the one-warp controller and its smaller
// shared-memory and register footprint.
template <bool MULTI>
__global__ void __launch_bounds__(BLOCK, 1) k_step(Plan* plan, double* partials,
                                                   unsigned long long* trace, GatherBufs gb,
                                                   const __grid_constant__ PlanBlob blob) {
  __shared__ double s_red[RED_SCRATCH];
  __shared__ double s_tot[PMAX];
  __shared__ double s_fixC[MAX_M], s_fixS[MAX_M];
  __shared__ int s_lcnt[NWARP];
  __shared__ int s_seg[NWARP * MAX_M * 2];
  __shared__ int s_nitems;
  extern __shared__ int4 s_dyn[];
  Plan& sp = *reinterpret_cast<Plan*>(s_dyn);
  char* s_work = reinterpret_cast<char*>(s_dyn) + PLAN_SMEM;   // lists, later gathered items
  uint32_t* s_list = reinterpret_cast<uint32_t*>(s_work);
  cg::grid_group grid = cg::this_grid();
  const int nb = gridDim.x;
  {  // load the controller state (everything but scratch) from the parameter
    int* spi = reinterpret_cast<int*>(&sp);
    for (int k = threadIdx.x; k < (int)PLAN_WORDS; k += BLOCK) spi[k] = blob.w[k];
  }
  // structured rows: centroid tables after the staging area of the work region
  double* s_rtab = reinterpret_cast<double*>(s_work);   // no active lists when rows are structured
  __syncthreads();
  build_row_tables(sp.P, s_rtab);
  __syncthreads();
  if (threadIdx.x == 0) g_ctl_marks = nullptr;
  for (int pass = 0; pass < 8192; ++pass) {
    if (sp.cmd.phase == PH_DONE) break;
    progress_mark(0, ((unsigned long long)pass << 8) | (unsigned)sp.cmd.phase);
    unsigned long long* tr = (trace && pass < 64) ? trace + pass * 8 : nullptr;
    if (tr && blockIdx.x == 0 && threadIdx.x == 0) { tr[0] = gtimer(); tr[5] = sp.cmd.phase; }
    // partials alternate between grid-synchronized passes only (a CTA-local
    // sweep writes none, so it must not flip the buffer a lagging CTA may
    // still read in the previous combine)
    double* part = partials + (size_t)(sp.nglobal & 1) * PMAX * nb;
    PassCtx c;
    c.plan = &sp;
    c.cmd = &sp.cmd;
    c.out = part + (size_t)blockIdx.x * PMAX;
    c.smem = s_red;
    c.i0 = (int64_t)blockIdx.x * BLOCK + threadIdx.x;
    c.stride = (int64_t)nb * BLOCK;
    c.list = sp.P.compact_cap > 0 ? s_list : nullptr;
    c.list_cnt = s_lcnt;
    c.seg = s_seg;
    c.fixC = s_fixC;
    c.fixS = s_fixS;
    c.list_cap = sp.P.compact_cap;
    c.blk_cnt = gb.blk_cnt;
    c.g_a = gb.g_a;
    c.g_r = gb.g_r;
    c.g_row = gb.g_row;
    c.g_fix = gb.g_fix;
    c.it_a = reinterpret_cast<double*>(s_work);
    c.it_r = c.it_a + GATHER_CAP;
    c.it_row = reinterpret_cast<int8_t*>(c.it_r + GATHER_CAP);
    c.n_items = &s_nitems;
    c.timed_out = gb.timed_out;
    c.rtab = s_rtab;
    c.ex_smem = reinterpret_cast<char*>(s_dyn) + sp.P.ex_smem;
    c.ms_smem = sp.P.ms_smem ? reinterpret_cast<char*>(s_dyn) + sp.P.ms_smem : nullptr;
    if (sp.cmd.phase == PH_SWEEP && sp.cmd.local) {   // CTA-local sweep: no barrier
      local_sweep(c, s_tot);
      if (tr && blockIdx.x == 0 && threadIdx.x == 0) {
        tr[1] = tr[6] = tr[2] = tr[3] = gtimer();
        g_ctl_marks = trace + 512 + pass * 8;
      }
      if constexpr (MULTI) {
        plan_consume_cta(sp, s_tot);
      } else {
        if (threadIdx.x < 32) plan_consume_warp(sp, s_tot);
        __syncthreads();
      }
      if (tr && blockIdx.x == 0 && threadIdx.x == 0) { tr[4] = gtimer(); g_ctl_marks = nullptr; }
      continue;
    }
    run_pass(c);
    progress_mark(1, pass);
    if (tr && threadIdx.x == 0) {
      if (blockIdx.x == 0) tr[1] = gtimer();
      atomicMax(tr + 6, gtimer());
    }
    __threadfence();
    grid.sync();
    progress_mark(2, pass);
    if (tr && blockIdx.x == 0 && threadIdx.x == 0) tr[2] = gtimer();
    if (sp.cmd.phase == PH_PREP && blockIdx.x == 0 && threadIdx.x == 0) signal_out(sp.P);
    if (sp.cmd.phase == PH_GATHER) gather_load(c, nb);
    if (sp.cmd.phase == PH_EXACT) {   // the chains ran in CTA 0 alone: its values are the sums
      for (int k = threadIdx.x; k < sp.cmd.nslots; k += BLOCK) s_tot[k] = __ldcg(part + k);
      __syncthreads();
      if (sp.P.ex_debug && blockIdx.x == 0 && threadIdx.x == 0)
        printf("[exact] what=%d n=%d seq=%d len=%lld seg=%lld nst=%d wa=%.17g t0=%.17g t1=%.17g\n",
               sp.cmd.ex_what, sp.cmd.ex_n, sp.cmd.ex_seq, (long long)sp.P.n,
               (long long)sp.P.ex_seg, sp.P.ex_nst, sp.cmd.wa, s_tot[0],
               sp.cmd.ex_n > 1 ? s_tot[1] : 0.0);
    } else {
      finish_reduce_cmd(part, nb, sp.cmd, sp.P.m, s_tot, s_red);
    }
    progress_mark(3, pass);
    if (threadIdx.x == 0) sp.nglobal++;   // (read again only after the controller's barrier)
    if (tr && blockIdx.x == 0 && threadIdx.x == 0) {
      tr[3] = gtimer();
      g_ctl_marks = trace + 512 + pass * 8;
    }
#ifdef TOPT_ICACHE_EXPERIMENT
    {  // controller twice on the same state: cold (first) vs warm (second) code
      int* gp = reinterpret_cast<int*>(g_plan_scratch + blockIdx.x);
      int* spi = reinterpret_cast<int*>(&sp);
      for (int k = threadIdx.x; k < (int)(sizeof(Plan) / 4); k += BLOCK) gp[k] = spi[k];
      __syncthreads();
      plan_consume_cta(sp, s_tot);
      if (tr && blockIdx.x == 0 && threadIdx.x == 0) tr[7] = gtimer();
      for (int k = threadIdx.x; k < (int)(sizeof(Plan) / 4); k += BLOCK) spi[k] = gp[k];
      __syncthreads();
      if (tr && blockIdx.x == 0 && threadIdx.x == 0) tr[3] = gtimer();
    }
#endif
    if constexpr (MULTI) {
      plan_consume_cta(sp, s_tot);
    } else {
      if (threadIdx.x < 32) plan_consume_warp(sp, s_tot);
      __syncthreads();
    }
    progress_mark(4, pass);
    if (sp.cmd.load_fused) {   // fused gather: the items were published by the sweep
      gather_load_fused(c, nb);
      if (threadIdx.x == 0) sp.cmd.load_fused = 0;
      __syncthreads();
    }
    if (tr && blockIdx.x == 0 && threadIdx.x == 0) { tr[4] = gtimer(); g_ctl_marks = nullptr; }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) signal_out(sp.P);   // also on early exits
  if (blockIdx.x == 0 && threadIdx.x == 0) sp.res.final_phase = sp.cmd.phase;
  __syncthreads();
  if (blockIdx.x == 0) {  // publish the final state (results) once
    int* gp = reinterpret_cast<int*>(plan);
    const int* spi = reinterpret_cast<const int*>(&sp);
    const int b0 = (int)(offsetof(Plan, cmd) / 4), nw = (int)(offsetof(Plan, sc) / 4);
    for (int k = b0 + threadIdx.x; k < nw; k += BLOCK) gp[k] = spi[k];
  }
}

__global__ void k_owner_init(int32_t* o32, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    o32[i] = -1;
}

// validate(): range and overlap (projection.cpp:163-171)
__global__ void k_owner_scatter(int32_t* o32, int64_t n, const int32_t* idx, const int64_t* off,
                                int m, int* err) {
  const int64_t total = off[m];
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total;
       k += (int64_t)gridDim.x * blockDim.x) {
    int j = 0;
    while (j + 1 < m && off[j + 1] <= k) ++j;   // m <= 16
    const int32_t i = idx[k];
    if (i < 0 || (int64_t)i >= n) { atomicOr(err, 1); continue; }
    if (atomicCAS(o32 + i, -1, j) != -1) atomicOr(err, 2);
  }
}

__global__ void k_owner_pack(const int32_t* o32, int8_t* o8, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    o8[i] = (int8_t)o32[i];
}

// Streaming probe: spin (bounded, ~50 ms) on a flag that the copy stream
// writes after this launch.  It sees the write only when kernels and copy-
// stream operations really run concurrently -- not under CUDA_LAUNCH_BLOCKING,
// a serializing profiler or a sanitizer; the host then uploads first.
__global__ void k_stream_probe(const unsigned* flag, unsigned epoch, int* seen) {
  if (threadIdx.x != 0) return;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  int ok = 0;
  for (;;) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if ((int)(v - epoch) >= 0) { ok = 1; break; }
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 50000000ull) break;
    __nanosleep(1000);
  }
  *seen = ok;
}

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

constexpr int MAX_STREAM_CHUNKS = 32;

// Driver stream memory operations (flag write / wait on a copy stream),
// resolved through the runtime so no -lcuda link is needed.
struct MemOps {
  bool ok = false;
  CUresult (*write32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int) = nullptr;
  CUresult (*wait32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int) = nullptr;
};
MemOps& memops() {
  static MemOps m;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* w = nullptr;
    void* v = nullptr;
    cudaDriverEntryPointQueryResult q1, q2;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &w, cudaEnableDefault, &q1) == cudaSuccess &&
        cudaGetDriverEntryPoint("cuStreamWaitValue32", &v, cudaEnableDefault, &q2) == cudaSuccess &&
        q1 == cudaDriverEntryPointSuccess && q2 == cudaDriverEntryPointSuccess && w && v) {
      m.write32 = (decltype(m.write32))w;
      m.wait32 = (decltype(m.wait32))v;
      m.ok = true;
    }
    cudaGetLastError();
  }
  return m;
}

}  // namespace

struct topt_b200_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int nsm = 0;
  int grid = 0;
  Plan* d_plan = nullptr;
  double* d_part = nullptr;
  unsigned* d_counter = nullptr;
  double* d_totals = nullptr;
  int* h_phase = nullptr;   // pinned
  int* d_err = nullptr;
  Plan h_plan;
  std::string err;
  int64_t launches = 0;
  DevBuf bufs[20];
  int profile = 0;
  int persistent = 1;       // one cooperative launch per job when possible
  int coop_grid = 0;        // co-resident CTAs for k_step
  int compact = 1;          // active-set compaction of bisection sweeps
  // fused multi-row sweep (pass_sweep_multi; TOPT_B200_FUSED_SWEEP=1).  Off by
  // default: measured r02n, the per-row sweeps are faster on every sweep (C4
  // 409 / 187 / 175 us against 3878 / 357 / 230 us; C5 7.9 / 3.5 / 3.2 ms
  // against 48.6 / 6.6 / 6.4 ms) -- a wide first window sends nearly every
  // element through the queued per-candidate loop and its shuffle folds.
  int fused_sweep = 0;
  // root sketch (controller.h: consume_sketch): sampled sweeps before the first
  // full sweep for problems of at least this many elements (0: never;
  // TOPT_B200_SKETCH_MIN_N)
  int64_t sketch_min_n = (int64_t)1 << 22;
  // the last PGD step's PREP found the pat7 row layout on these buffers
  // (Problem::pat_hint; TOPT_B200_PAT_HINT=0 disables)
  int pat_hint_on = 1;
  // candidates per row in a walk's first full sweep after the sketch
  // (Problem::first_k, TOPT_B200_FIRST_K; r02y: 8 instead of 16 takes C5's
  // first sweep from 8.5 to 6.2 ms and C4's from 449 to 330 us; the third
  // sweep then uses its spare candidates)
  int first_k = 8;
  const double* pat_grad = nullptr;
  int64_t pat_n = 0, pat_ld = 0;
  int* d_blk_cnt = nullptr;
  double* d_ga = nullptr;
  double* d_gr = nullptr;
  int* d_grow = nullptr;
  double* d_gfix = nullptr;
  int max_dyn_smem = 0;
  int trace_on = 0;
  unsigned long long* d_trace = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  double prof_ms = 0.0, prof_max = 0.0;
  int64_t prof_n = 0;
  // whole-job device time (plan upload -> results downloaded), when profiling
  cudaEvent_t evs0 = nullptr, evs1 = nullptr;
  double step_ms = 0.0, step_max = 0.0;
  int64_t step_n = 0;
  // multi-rank (one process per GPU, NCCL over NVLink)
  int rank = 0, world = 1;
  void* comm = nullptr;          // ncclComm_t
  double* d_rank_tot = nullptr;  // [PMAX]
  double* d_gathered = nullptr;  // [world][PMAX]
  int64_t n_global_override = 0;
  const int64_t* row_counts_override = nullptr;
  // host-buffer streaming (copies overlap the step's first passes)
  cudaStream_t cstream = nullptr;  // copy stream
  cudaEvent_t ev_copy = nullptr;
  unsigned* d_flags = nullptr;     // [2 * MAX_STREAM_CHUNKS] in, [2 * MAX_STREAM_CHUNKS] out
  int* d_timed_out = nullptr;
  int* h_timed_out = nullptr;      // pinned
  uint32_t epoch = 0;
  int stream_inputs = 1;           // TOPT_B200_STREAM=0 disables
  int parity = 0;                  // 0 certified, 1 strict (TOPT_B200_PARITY=strict)
  int lockstep = 0;                // rank of a single-process lockstep job (no NCCL)
  int defer = 0;                   // run_plan_ranks: prepare only (the lockstep driver)
  cudaEvent_t ev_pass = nullptr, ev_copied = nullptr;
  int ex_debug = 0;
  const int32_t* last_pidx = nullptr;   // device partition indices of the last owner map
  int64_t last_poff[MAX_M + 1] = {};
  int stream_probe = -1;
  int stream_timeout = 0;          // the last streamed launch timed out waiting for a chunk           // can a running kernel see copy-stream writes? (-1: unknown)
  int* d_probe = nullptr;
  Plan* hp_pin = nullptr;          // pinned staging of the plan (upload / results)
  // structured rows for the following *_dev / *_ranks steps (topt_b200_set_structured_rows)
  int srows_m = 0;
  topt_row_desc srows[MAX_M] = {};
  int64_t sgrid[3] = {0, 0, 0};
  int64_t sidx_off = 0;
  // contiguous-range partitions detected by the owner maps built here (a
  // few, keyed by the owner map's device pointer: the host-buffer and the
  // device-buffer steps of one problem keep different maps)
  struct RangeEntry {
    const int8_t* owner = nullptr;
    int m = 0;
    int64_t lo[MAX_M] = {}, hi[MAX_M] = {};
  };
  static constexpr int N_RANGE = 4;
  RangeEntry rng[N_RANGE];
  int rng_next = 0;
};

// ---- NCCL, resolved at run time (the process may already hold torch's copy)
#include <dlfcn.h>
#include <nccl.h>
namespace {
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    // Prefer a copy already in the process (e.g. torch's, whose libtorch_cuda
    // needs its own newer NCCL symbols); never inject one into the global
    // symbol namespace.
    void* h = nullptr;
    if (const char* p = getenv("TOPT_B200_NCCL_LIB")) h = dlopen(p, RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
    if (h) {
      api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
      api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
      api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
      api.AllGather = (decltype(api.AllGather))dlsym(h, "ncclAllGather");
      api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
      api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllGather;
    }
  }
  return api;
}
}  // namespace

namespace {

int fail(topt_b200_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->err = msg;
  return code;
}

#define CUDA_TRY(ctx, expr)                                                         \
  do {                                                                              \
    cudaError_t e_ = (expr);                                                        \
    if (e_ != cudaSuccess)                                                          \
      return fail(ctx, TOPT_ERR_CUDA, std::string(#expr ": ") + cudaGetErrorString(e_)); \
  } while (0)

void* buf(topt_b200_ctx* ctx, int slot, size_t bytes) {
  DevBuf& b = ctx->bufs[slot];
  if (b.bytes < bytes) {
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.bytes = 0;
    if (cudaMalloc(&b.p, bytes) != cudaSuccess) return nullptr;
    b.bytes = bytes;
  }
  return b.p;
}

enum BufSlot {
  B_RHO = 0, B_GRAD, B_GD, B_DELTA, B_OWNER, B_OWNER32, B_X, B_XP, B_G, B_GP, B_DP, B_D,
  B_XNEW, B_PIDX, B_POFF, B_MASK, B_EXACT
};

const char* status_msg(int st) {
  switch (st) {
    case ST_OK: return "ok";
    case ST_PARAMETER: return "ParameterError";
    case ST_DOMAIN: return "DomainError";
    case ST_SINGULAR: return "SingularSystemError";
    case ST_INFEASIBLE: return "InfeasibleLinearization: linearized feasible set is empty";
    case ST_NUMERICAL: return "NumericalError: singular or non-finite Newton system";
    case ST_UNSUPPORTED: return "UnsupportedProblem";
    default: return "internal error";
  }
}

// Run a plan to completion on the device.  hp.P must be filled.
int run_plan_ranks(topt_b200_ctx* ctx, Plan& hp);

// Host-side half of the input streaming: the host arrays of one PGD step and
// where they go.  Issued on the copy stream right after the kernel launch.
struct StreamIn {
  const double *x, *xp, *g, *gp, *dp, *grad;   // host
  double *dx, *dxp, *dg, *dgp, *ddp, *dgrad;   // device
  int m;
  double* d_host;                              // optional: d out (device->host after PREP)
  const double* d_dev;
};

int issue_stream(topt_b200_ctx* ctx, const Plan& hp, const StreamIn& si) {
  const Problem& P = hp.P;
  MemOps& mo = memops();
  const int64_t n = P.n, ch = P.chunk;
  const int nch = P.nchunk;
  const CUstream cs = (CUstream)ctx->cstream;
  auto put = [&](double* dst, const double* src, int64_t lo, int64_t cnt) -> int {
    CUDA_TRY(ctx, cudaMemcpyAsync(dst + lo, src + lo, sizeof(double) * (size_t)cnt,
                                  cudaMemcpyHostToDevice, ctx->cstream));
    return TOPT_OK;
  };
  int rc;
  for (int k = 0; k < nch; ++k) {   // group A: what the BB / PR+ pass reads
    const int64_t lo = (int64_t)k * ch, cnt = std::min<int64_t>(ch, n - lo);
    if ((rc = put(si.dx, si.x, lo, cnt)) || (rc = put(si.dxp, si.xp, lo, cnt)) ||
        (rc = put(si.dg, si.g, lo, cnt)) || (rc = put(si.dgp, si.gp, lo, cnt)))
      return rc;
    if (mo.write32(cs, (CUdeviceptr)(ctx->d_flags + k), P.epoch, 0) != CUDA_SUCCESS)
      return fail(ctx, TOPT_ERR_CUDA, "cuStreamWriteValue32 failed");
  }
  for (int k = 0; k < nch; ++k) {   // group B: d_prev and the constraint rows
    const int64_t lo = (int64_t)k * ch, cnt = std::min<int64_t>(ch, n - lo);
    if ((rc = put(si.ddp, si.dp, lo, cnt))) return rc;
    for (int j = 0; j < si.m; ++j)
      if ((rc = put(si.dgrad + (int64_t)j * n, si.grad + (int64_t)j * n, lo, cnt))) return rc;
    if (mo.write32(cs, (CUdeviceptr)(ctx->d_flags + nch + k), P.epoch, 0) != CUDA_SUCCESS)
      return fail(ctx, TOPT_ERR_CUDA, "cuStreamWriteValue32 failed");
  }
  if (si.d_host && n > 0) {   // d is final after PREP: copy it while the bisection runs
    if (mo.wait32(cs, (CUdeviceptr)(ctx->d_flags + 2 * MAX_STREAM_CHUNKS), P.epoch,
                  CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
      return fail(ctx, TOPT_ERR_CUDA, "cuStreamWaitValue32 failed");
    CUDA_TRY(ctx, cudaMemcpyAsync(si.d_host, si.d_dev, sizeof(double) * (size_t)n,
                                  cudaMemcpyDeviceToHost, ctx->cstream));
  }
  CUDA_TRY(ctx, cudaEventRecord(ctx->ev_copy, ctx->cstream));
  CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->stream, ctx->ev_copy, 0));
  return TOPT_OK;
}

// The device needs the plan up to the scratch area; the host reads back only
// the next phase and the results.  Both go through pinned staging.
constexpr size_t PLAN_UP = offsetof(Plan, sc);
int plan_upload(topt_b200_ctx* ctx, const Plan& hp) {
  if (ctx->profile) cudaEventRecord(ctx->evs0, ctx->stream);
  std::memcpy(ctx->hp_pin, &hp, PLAN_UP);
  CUDA_TRY(ctx, cudaMemcpyAsync(ctx->d_plan, ctx->hp_pin, PLAN_UP, cudaMemcpyHostToDevice, ctx->stream));
  return TOPT_OK;
}
int plan_results_async(topt_b200_ctx* ctx) {
  CUDA_TRY(ctx, cudaMemcpyAsync(&ctx->hp_pin->cmd.phase, &ctx->d_plan->cmd.phase, sizeof(int32_t),
                                cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(ctx, cudaMemcpyAsync(&ctx->hp_pin->res, &ctx->d_plan->res, sizeof(Result),
                                cudaMemcpyDeviceToHost, ctx->stream));
  if (ctx->profile) cudaEventRecord(ctx->evs1, ctx->stream);
  return TOPT_OK;
}
// (after the stream synchronize)
void plan_results_take(topt_b200_ctx* ctx, Plan& hp) {
  hp.cmd.phase = ctx->hp_pin->cmd.phase;
  hp.res = ctx->hp_pin->res;
  if (ctx->profile) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, ctx->evs0, ctx->evs1) == cudaSuccess) {
      ctx->step_ms += ms;
      ctx->step_max = std::max(ctx->step_max, (double)ms);
      ctx->step_n++;
    }
  }
}

static int run_plan_(topt_b200_ctx* ctx, Plan& hp, const StreamIn* si);
int run_plan(topt_b200_ctx* ctx, Plan& hp, const StreamIn* si = nullptr) {
  if (ctx->comm || ctx->lockstep) return run_plan_ranks(ctx, hp);
  const bool step = hp.P.job == JOB_PGD_STEP && hp.P.m == 7;
  hp.P.pat_hint = (step && ctx->pat_hint_on && ctx->pat_grad == hp.P.grad &&
                   ctx->pat_n == hp.P.n && ctx->pat_ld == hp.P.ld) ? 1 : 0;
  const int rc = run_plan_(ctx, hp, si);
  if (step) {   // remember (or forget) the row layout PREP found on these buffers
    const bool found = rc == TOPT_OK && hp.res.pat7;
    ctx->pat_grad = found ? hp.P.grad : nullptr;
    ctx->pat_n = hp.P.n;
    ctx->pat_ld = hp.P.ld;
  }
  return rc;
}
static int run_plan_(topt_b200_ctx* ctx, Plan& hp, const StreamIn* si) {
  const bool persistent = ctx->persistent && ctx->coop_grid > 0;
  const int grid = persistent ? ctx->coop_grid : ctx->grid;
  const int64_t per_thread = (hp.P.n + (int64_t)grid * BLOCK - 1) / ((int64_t)grid * BLOCK);
  // per-thread summation depth: own elements + queued elements taken over
  // from other lanes (SweepAcc) + the CTA tree and the CTA combine
  hp.P.ours_len = 2.0 * (double)per_thread + (double)grid + 64.0;
  size_t dyn_smem = sizeof(Plan);
  hp.P.compact_cap = 0;
  // active lists only where compacted sweeps run (one row, or a partition);
  // otherwise the work area is free (structured rows keep their tables there)
  if (persistent && ctx->compact && (hp.P.m == 1 || hp.P.has_part)) {
    const int64_t cap = 32 * per_thread;
    size_t bytes = (size_t)NWARP * (size_t)cap * sizeof(uint32_t);
    const size_t item_bytes = (size_t)GATHER_CAP * (2 * sizeof(double) + 1);
    if (bytes < item_bytes) bytes = item_bytes;
    if (cap > 0 && PLAN_SMEM + bytes <= (size_t)ctx->max_dyn_smem && hp.P.n < (int64_t)4000000000LL) {
      hp.P.compact_cap = (int32_t)cap;
      dyn_smem = PLAN_SMEM + bytes;
    }
  }
  // the work area holds the structured rows' tables instead (no active
  // lists in that case)
  dyn_smem = std::max(dyn_smem, PLAN_SMEM + sizeof(double) * (size_t)hp.P.n_tab);
  // dense multi-row problems without a partition: the fused multi-row sweep's
  // queues and accumulators (pass_sweep_multi)
  hp.P.ms_smem = 0;
  if (persistent && ctx->fused_sweep && hp.P.m > 1 && !hp.P.has_part && !hp.P.structured) {
    const size_t off = (dyn_smem + 127) & ~size_t(127);
    // (leaves room for the strict-parity chain ring: >= 2 stages of 16 KB)
    if (off + multi_sweep_bytes() + 2 * EX_CHUNK_BYTES + 256 <= (size_t)ctx->max_dyn_smem) {
      hp.P.ms_smem = (int32_t)off;
      dyn_smem = off + multi_sweep_bytes();
    }
  }
  if (hp.P.strict) {
    // strict parity: chain passes (PH_EXACT) run inside the persistent kernel
    Problem& P = hp.P;
    if (!persistent || grid < 2)
      return fail(ctx, TOPT_ERR_UNSUPPORTED, "strict parity needs the persistent (cooperative) kernel");
    if (P.m > 9)
      return fail(ctx, TOPT_ERR_UNSUPPORTED, "strict parity supports m <= 9 constraint rows");
    if (P.structured)
      return fail(ctx, TOPT_ERR_UNSUPPORTED, "strict parity needs dense constraint rows");
    if (P.has_part && !P.part_ranges && !P.part_idx)
      return fail(ctx, TOPT_ERR_UNSUPPORTED,
                  "strict parity needs the partition's index lists (host-buffer call)");
    const size_t off = (dyn_smem + 127) & ~size_t(127);
    const size_t avail = (size_t)ctx->max_dyn_smem > off + 256 ? ctx->max_dyn_smem - off - 256 : 0;
    const int nst = (int)std::min<size_t>(8, avail / EX_CHUNK_BYTES);
    if (nst < 2) return fail(ctx, TOPT_ERR_UNSUPPORTED, "strict parity: no shared memory left for the chain ring");
    P.ex_nst = nst;
    P.ex_smem = (int32_t)off;
    dyn_smem = off + (size_t)nst * EX_CHUNK_BYTES + 2 * sizeof(uint64_t) * (size_t)nst;
    P.ex_seg = std::max<int64_t>(1, std::min<int64_t>(P.n, (int64_t)1 << 21));
    P.ex_buf = (double*)buf(ctx, B_EXACT, sizeof(double) * 2 * (size_t)P.ex_seg * MAX_EX);
    if (!P.ex_buf) return fail(ctx, TOPT_ERR_CUDA, "cudaMalloc failed (strict parity staging)");
  }
  plan_start(hp);
  int phase = hp.cmd.phase;
  if (persistent && phase != PH_DONE) {
    if (ctx->profile) cudaEventRecord(ctx->evs0, ctx->stream);
    PlanBlob* blob = reinterpret_cast<PlanBlob*>(ctx->hp_pin);
    std::memcpy(blob, &hp, sizeof(PlanBlob));
    unsigned long long* tr = ctx->trace_on ? ctx->d_trace : nullptr;
    if (tr) cudaMemsetAsync(tr, 0, 128 * 8 * sizeof(unsigned long long), ctx->stream);
    GatherBufs gb{ctx->d_blk_cnt, ctx->d_ga, ctx->d_gr, ctx->d_grow, ctx->d_gfix,
                  ctx->d_timed_out};
    void* args[] = {&ctx->d_plan, &ctx->d_part, &tr, &gb, blob};
    if (si) CUDA_TRY(ctx, cudaMemsetAsync(ctx->d_timed_out, 0, sizeof(int), ctx->stream));
    if (ctx->profile) cudaEventRecord(ctx->ev0, ctx->stream);
    const void* kfn = hp.P.m > 1 ? (const void*)k_step<true> : (const void*)k_step<false>;
    CUDA_TRY(ctx, cudaLaunchCooperativeKernel(kfn, grid, BLOCK, args, dyn_smem,
                                              ctx->stream));
    ctx->launches++;
    if (ctx->profile) cudaEventRecord(ctx->ev1, ctx->stream);
    if (si) {
      const int rc = issue_stream(ctx, hp, *si);
      if (rc) { cudaStreamSynchronize(ctx->stream); return rc; }
      CUDA_TRY(ctx, cudaMemcpyAsync(ctx->h_timed_out, ctx->d_timed_out, sizeof(int),
                                    cudaMemcpyDeviceToHost, ctx->stream));
    }
    CUDA_TRY(ctx, cudaMemcpyAsync(&ctx->hp_pin->res, &ctx->d_plan->res, sizeof(Result),
                                  cudaMemcpyDeviceToHost, ctx->stream));
    if (ctx->profile) cudaEventRecord(ctx->evs1, ctx->stream);
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    ctx->hp_pin->cmd.phase = ctx->hp_pin->res.final_phase;
    plan_results_take(ctx, hp);
    if (si && *ctx->h_timed_out) {
      ctx->stream_timeout = 1;
      return fail(ctx, TOPT_ERR_CUDA, "topt_b200: a streamed input chunk never arrived");
    }
    if (ctx->profile) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
      ctx->prof_ms += ms;
      ctx->prof_max = std::max(ctx->prof_max, (double)ms);
      ctx->prof_n++;
    }
    if (hp.cmd.phase != PH_DONE) return fail(ctx, TOPT_ERR_INTERNAL, "plan did not terminate");
    if (hp.res.status != ST_OK) return fail(ctx, hp.res.status, status_msg(hp.res.status));
    return TOPT_OK;
  }
  if (int rc = plan_upload(ctx, hp)) return rc;
  for (int it = 0; phase != PH_DONE && it < 4096; ++it) {
    if (ctx->profile) cudaEventRecord(ctx->ev0, ctx->stream);
    k_pass<<<ctx->grid, BLOCK, KPASS_SMEM + sizeof(double) * (size_t)hp.P.n_tab, ctx->stream>>>(ctx->d_plan, ctx->d_part,
                                                            ctx->d_counter, nullptr);
    ctx->launches++;
    CUDA_TRY(ctx, cudaGetLastError());
    if (ctx->profile) cudaEventRecord(ctx->ev1, ctx->stream);
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->h_phase, &ctx->d_plan->cmd.phase, sizeof(int),
                                  cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    if (ctx->profile) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
      ctx->prof_ms += ms;
      ctx->prof_max = std::max(ctx->prof_max, (double)ms);
      ctx->prof_n++;
    }
    phase = *ctx->h_phase;
    if (const char* dbg = getenv("TOPT_B200_DEBUG_PHASES")) {
      if (it < 64) fprintf(stderr, "[topt1] pass %d -> phase %d\n", it, phase);
      if (atoi(dbg) >= 2 && it < 64) {   // the next command's candidates and the walks' state
        static Plan dp;
        cudaMemcpy(&dp, ctx->d_plan, offsetof(Plan, sc), cudaMemcpyDeviceToHost);
        if (dp.cmd.phase == PH_SWEEP) {
          fprintf(stderr, "  sweep: sample %d compact %d ncand %d sketch_left %d\n", dp.cmd.sample,
                  dp.cmd.compact, dp.cmd.ncand, dp.sketch_left);
          for (int j = 0; j < dp.P.m; ++j) {
            const Walk& w = dp.w[j];
            fprintf(stderr, "  row %d status %d up %d feas %d lo %.6g hi %.6g hok %d hy %.9g hs %.3g E %.3g cand:", j,
                    w.status, w.up, w.feas_done, w.lo, w.hi, w.hok, w.hy, w.hs, w.E);
            for (int k = dp.cmd.row_start[j]; k < dp.cmd.row_start[j + 1]; ++k)
              fprintf(stderr, " %.9g", dp.cmd.cand_y[k]);
            fprintf(stderr, "\n");
          }
        }
      }
    }
  }
  if (int rc = plan_results_async(ctx)) return rc;
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  plan_results_take(ctx, hp);
  if (phase != PH_DONE) return fail(ctx, TOPT_ERR_INTERNAL, "plan did not terminate");
  if (hp.res.status != ST_OK) return fail(ctx, hp.res.status, status_msg(hp.res.status));
  return TOPT_OK;
}

// Multi-rank: per pass, every rank reduces its slab's partials on its GPU,
// the rank totals are all-gathered over NCCL (NVLink), and every rank
// combines them in rank order and runs the controller -- identical decisions
// everywhere, no host arithmetic.  The host only sequences the launches and
// polls the next phase.
constexpr int TOPT_DEFERRED = 100;   // internal: plan prepared, passes driven by the caller
constexpr int RANK_BATCH = 4;        // passes enqueued per host synchronization (rank mode)

int ranks_setup(topt_b200_ctx* ctx, Plan& hp) {
  if (hp.P.strict)   // a reference-order sum is sequential across the ranks' slabs
    return fail(ctx, TOPT_ERR_UNSUPPORTED, "strict parity is single-GPU only");
  const int grid = ctx->grid;
  const int64_t per_thread = (hp.P.n + (int64_t)grid * BLOCK - 1) / ((int64_t)grid * BLOCK);
  hp.P.ours_len = 2.0 * (double)per_thread + (double)grid + 64.0 + (double)ctx->world;
  hp.P.compact_cap = 0;
  plan_start(hp);
  return plan_upload(ctx, hp);
}

int ranks_pass_kernel(topt_b200_ctx* ctx, const Plan& hp) {
  k_pass<<<ctx->grid, BLOCK, KPASS_SMEM + sizeof(double) * (size_t)hp.P.n_tab, ctx->stream>>>(
      ctx->d_plan, ctx->d_part, ctx->d_counter, ctx->d_rank_tot);
  ctx->launches++;
  CUDA_TRY(ctx, cudaGetLastError());
  return TOPT_OK;
}

int ranks_control_kernel(topt_b200_ctx* ctx) {
  k_control<<<1, BLOCK, sizeof(Plan), ctx->stream>>>(ctx->d_plan, ctx->d_gathered, ctx->world);
  ctx->launches++;
  CUDA_TRY(ctx, cudaGetLastError());
  return TOPT_OK;
}

int ranks_finish(topt_b200_ctx* ctx, Plan& hp, int phase) {
  if (int rc = plan_results_async(ctx)) return rc;
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  plan_results_take(ctx, hp);
  if (phase != PH_DONE) return fail(ctx, TOPT_ERR_INTERNAL, "plan did not terminate");
  if (hp.res.status != ST_OK) return fail(ctx, hp.res.status, status_msg(hp.res.status));
  return TOPT_OK;
}

// Multi-rank over NCCL: per pass every rank reduces its slab's partials on
// its GPU (k_pass), the rank totals are all-gathered (NVLink), and every rank
// combines them in rank order and runs the controller (k_control) --
// identical decisions everywhere, no host arithmetic.  Passes are enqueued
// RANK_BATCH at a time between host reads of the phase: a pass after the
// last one is a no-op (k_pass / k_control return at PH_DONE, the all-gather
// moves stale bytes), and every rank enqueues the same count.
int run_plan_ranks(topt_b200_ctx* ctx, Plan& hp) {
  if (int rc = ranks_setup(ctx, hp)) return rc;
  if (ctx->defer) return TOPT_DEFERRED;
  int phase = hp.cmd.phase;
  NcclApi& api = nccl();
  for (int it = 0; phase != PH_DONE && it < 4096; it += RANK_BATCH) {
    if (ctx->profile) cudaEventRecord(ctx->ev0, ctx->stream);
    for (int b = 0; b < RANK_BATCH; ++b) {
      if (int rc = ranks_pass_kernel(ctx, hp)) return rc;
      const ncclResult_t nr = api.AllGather(ctx->d_rank_tot, ctx->d_gathered, PMAX, ncclDouble,
                                            (ncclComm_t)ctx->comm, ctx->stream);
      if (nr != ncclSuccess)
        return fail(ctx, TOPT_ERR_CUDA, std::string("ncclAllGather: ") +
                                            (api.GetErrorString ? api.GetErrorString(nr) : "?"));
      if (int rc = ranks_control_kernel(ctx)) return rc;
    }
    if (ctx->profile) cudaEventRecord(ctx->ev1, ctx->stream);
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->h_phase, &ctx->d_plan->cmd.phase, sizeof(int),
                                  cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    if (ctx->profile) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
      ctx->prof_ms += ms;
      ctx->prof_max = std::max(ctx->prof_max, (double)ms);
      ctx->prof_n += RANK_BATCH;
    }
    phase = *ctx->h_phase;
  }
  return ranks_finish(ctx, hp, phase);
}

void fill_meta(const Plan& hp, topt_proj_meta* meta) {
  if (!meta) return;
  const Result& r = hp.res;
  std::memset(meta, 0, sizeof(*meta));
  meta->path = r.path;
  meta->newton_iters = r.newton_iters;
  meta->converged = r.converged;
  meta->curvature_violations = r.curvature_violations;
  meta->residual = r.residual;
  meta->passes = r.passes;
  meta->sweeps = r.sweeps;
  meta->stage1_row = r.stage1_row;
  meta->near_ties = r.near_ties;
  meta->min_margin = r.min_margin;
  for (int j = 0; j < MAX_M; ++j) meta->bisect_iters[j] = r.bisect_iters[j];
  meta->alpha = r.alpha;
  meta->beta = r.beta;
  meta->fallback = r.fallback;
  meta->local_sweeps = r.local_sweeps;
  meta->gathered = r.gathered;
  meta->active = r.active;
  meta->exact_passes = r.exact_passes;
}

void default_opts(ProjOptions& o) {
  o.c = 1e12; o.tol_b = 1e-8; o.tol_n = 1e-6; o.newton_maxiter = 50; o.binary_maxiter = 200;
}

int init_problem(topt_b200_ctx* ctx, Plan& hp, int64_t n, int m, const topt_proj_options* opts) {
  std::memset(&hp, 0, sizeof(Plan));
  if (m > MAX_M)
    return fail(ctx, TOPT_ERR_UNSUPPORTED, "topt_b200: at most 16 constraint rows supported");
  if (m < 0 || n < 0) return fail(ctx, TOPT_ERR_DOMAIN, "topt_b200: negative sizes");
  Problem& P = hp.P;
  P.n = n;
  P.n_global = n;
  P.m = m;
  P.ld = n;
  if (opts) {
    P.opt.c = opts->c; P.opt.tol_b = opts->tol_b; P.opt.tol_n = opts->tol_n;
    P.opt.newton_maxiter = opts->newton_maxiter; P.opt.binary_maxiter = opts->binary_maxiter;
  } else {
    default_opts(P.opt);
  }
  for (int j = 0; j < m; ++j) P.row_count[j] = (double)n;
  P.strict = ctx->parity;
  P.ex_debug = ctx->ex_debug;
  P.sketch_min_n = ctx->sketch_min_n;
  P.first_k = ctx->first_k;
  return TOPT_OK;
}

void set_lin_scalars(Plan& hp, const topt_linearization* lin) {
  Problem& P = hp.P;
  const int m = P.m;
  for (int j = 0; j < m; ++j) {
    if (lin->bounds_g && lin->g_values) P.G_minus_g[j] = lin->bounds_g[j] - lin->g_values[j];
    if (lin->g_hat) P.ghat_in[j] = lin->g_hat[j];
    P.ghat_err_in[j] = lin->g_hat_err ? lin->g_hat_err[j] : 0.0;
    P.is_eq[j] = lin->is_equality ? (lin->is_equality[j] ? 1 : 0) : 0;
  }
  if (lin->part_offsets) {
    for (int j = 0; j < m; ++j)
      P.row_count[j] = (double)(lin->part_offsets[j + 1] - lin->part_offsets[j]);
  }
}

int upload(topt_b200_ctx* ctx, int slot, const void* src, size_t bytes, void** dst) {
  *dst = nullptr;
  if (!src || bytes == 0) return TOPT_OK;
  void* d = buf(ctx, slot, bytes);
  if (!d) return fail(ctx, TOPT_ERR_CUDA, "cudaMalloc failed");
  CUDA_TRY(ctx, cudaMemcpyAsync(d, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
  *dst = d;
  return TOPT_OK;
}

// Is every set of the partition one contiguous ascending index range?  (Host
// scan of the index arrays; remembered with the owner map it belongs to.)
void detect_ranges(topt_b200_ctx* ctx, int32_t m, const int64_t* off, const int32_t* idx,
                   const int8_t* owner_dev) {
  int slot = -1;   // a rebuilt map replaces what was known about its buffer
  for (int k = 0; k < topt_b200_ctx::N_RANGE; ++k)
    if (ctx->rng[k].owner == owner_dev) { ctx->rng[k].owner = nullptr; slot = k; }
  if (m < 1 || m > MAX_M) return;
  topt_b200_ctx::RangeEntry r;
  for (int j = 0; j < m; ++j) {
    const int64_t b = off[j], e = off[j + 1];
    if (e <= b) return;
    for (int64_t k = b + 1; k < e; ++k)
      if (idx[k] != idx[k - 1] + 1) return;
    r.lo[j] = idx[b];
    r.hi[j] = (int64_t)idx[e - 1] + 1;
  }
  r.m = m;
  r.owner = owner_dev;
  if (slot < 0) {
    slot = ctx->rng_next;
    ctx->rng_next = (ctx->rng_next + 1) % topt_b200_ctx::N_RANGE;
  }
  ctx->rng[slot] = r;
}

// Structured rows set on the context -> the Problem (device entries only).
int apply_structured(topt_b200_ctx* ctx, Problem& P) {
  P.structured = 0;
  P.n_tab = 0;
  if (ctx->srows_m == 0) return TOPT_OK;
  if (ctx->srows_m != P.m)
    return fail(ctx, TOPT_ERR_DOMAIN, "structured rows: row count differs from the problem's m");
  if (P.m < 2 || P.m > 8 || P.owner || (P.n & 1))
    return fail(ctx, TOPT_ERR_UNSUPPORTED,
                "structured rows: need 2 <= m <= 8, no partition and an even element count");
  int ntab = 0;
  for (int k = 0; k < P.m; ++k) {
    const topt_row_desc& d = ctx->srows[k];
    P.row_kind[k] = d.kind;
    P.row_axis[k] = d.axis;
    P.row_c[k] = d.kind == RK_CONST ? d.value : d.center;
    P.row_scale[k] = d.scale;
    P.row_sign[k] = d.sign < 0.0 ? -1.0 : 1.0;
    P.row_tab[k] = -1;
    if (d.kind == RK_DENSE) {
      if (!P.grad) return fail(ctx, TOPT_ERR_DOMAIN, "structured rows: a dense row needs grad");
      continue;
    }
    if (d.kind == RK_CONST) {   // one table entry holding the value
      P.row_tab[k] = ntab++;
      continue;
    }
    if (d.kind != RK_CENTROID || d.axis < 0 || d.axis > 2)
      return fail(ctx, TOPT_ERR_DOMAIN, "structured rows: unknown row kind / axis");
    for (int j = 0; j < k && P.row_tab[k] < 0; ++j)   // share an identical centroid row's table
      if (P.row_kind[j] == RK_CENTROID && P.row_axis[j] == d.axis &&
          P.row_c[j] == d.center && P.row_scale[j] == d.scale)
        P.row_tab[k] = P.row_tab[j];
    if (P.row_tab[k] < 0) {
      P.row_tab[k] = ntab;
      ntab += (int)ctx->sgrid[d.axis];
    }
  }
  if (ctx->sgrid[0] <= 0 || ctx->sgrid[1] <= 0 || ctx->sgrid[2] <= 0 || ntab > MAX_TAB)
    return fail(ctx, TOPT_ERR_UNSUPPORTED, "structured rows: grid missing or tables too large");
  for (int a = 0; a < 3; ++a) P.grid_n[a] = ctx->sgrid[a];
  P.idx_off = ctx->sidx_off;
  // one table per axis (the centre-of-mass pattern): the passes then fetch
  // three values per element and take every row as +-value / constant
  P.axis_fast = 1;
  for (int a = 0; a < 3; ++a) P.axis_tab[a] = -1;
  P.const_tab = -1;
  int kc = -1;   // first constant row
  for (int k = 0; k < P.m; ++k) {
    if (P.row_kind[k] == RK_CONST) {
      if (kc < 0) { kc = k; P.const_tab = P.row_tab[k]; }
      else if (!(P.row_c[k] == P.row_c[kc])) P.axis_fast = 0;
      continue;
    }
    if (P.row_kind[k] != RK_CENTROID) continue;
    const int a = P.row_axis[k];
    if (P.axis_tab[a] < 0) P.axis_tab[a] = P.row_tab[k];
    else if (P.axis_tab[a] != P.row_tab[k]) P.axis_fast = 0;
  }
  P.n_tab = ntab;
  P.structured = 1;
  return TOPT_OK;
}

void apply_ranges(const topt_b200_ctx* ctx, Problem& P) {
  P.part_ranges = 0;
  if (!P.owner) return;
  for (const auto& e : ctx->rng) {
    if (e.owner != P.owner || e.m != P.m) continue;
    for (int j = 0; j < P.m; ++j) {
      if (e.lo[j] < 0 || e.hi[j] > P.n) return;
      P.row_lo[j] = e.lo[j];
      P.row_hi[j] = e.hi[j];
    }
    P.part_ranges = 1;
    return;
  }
}

// The partition's device index lists (strict parity sums a subset walk over
// them in the partition's own order, projection.cpp:31-32).
void set_part_lists(const topt_b200_ctx* ctx, Problem& P) {
  P.part_idx = ctx->last_pidx;
  for (int j = 0; j <= P.m && j <= MAX_M; ++j) P.part_off[j] = ctx->last_poff[j];
}

int owner_map_impl(topt_b200_ctx* ctx, int64_t n, int32_t m, const int64_t* off,
                   const int32_t* idx, int8_t* owner_dev) {
  detect_ranges(ctx, m, off, idx, owner_dev);
  int32_t* o32 = (int32_t*)buf(ctx, B_OWNER32, sizeof(int32_t) * (size_t)std::max<int64_t>(n, 1));
  if (!o32) return fail(ctx, TOPT_ERR_CUDA, "cudaMalloc failed");
  const int64_t total = off[m];
  void* didx = nullptr;
  void* doff = nullptr;
  int rc = upload(ctx, B_PIDX, idx, sizeof(int32_t) * (size_t)total, &didx);
  if (rc) return rc;
  ctx->last_pidx = (const int32_t*)didx;
  for (int j = 0; j <= m && j <= MAX_M; ++j) ctx->last_poff[j] = off[j];
  rc = upload(ctx, B_POFF, off, sizeof(int64_t) * (size_t)(m + 1), &doff);
  if (rc) return rc;
  CUDA_TRY(ctx, cudaMemsetAsync(ctx->d_err, 0, sizeof(int), ctx->stream));
  const int g = ctx->nsm * 4;
  if (n > 0) k_owner_init<<<g, 256, 0, ctx->stream>>>(o32, n);
  if (total > 0)
    k_owner_scatter<<<g, 256, 0, ctx->stream>>>(o32, n, (const int32_t*)didx,
                                                (const int64_t*)doff, m, ctx->d_err);
  if (n > 0) k_owner_pack<<<g, 256, 0, ctx->stream>>>(o32, owner_dev, n);
  ctx->launches += 3;
  CUDA_TRY(ctx, cudaGetLastError());
  int herr = 0;
  CUDA_TRY(ctx, cudaMemcpyAsync(&herr, ctx->d_err, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  if (herr & 1) return fail(ctx, TOPT_ERR_DOMAIN, "ConstraintLinearization: partition index out of range");
  if (herr & 2) return fail(ctx, TOPT_ERR_DOMAIN, "ConstraintLinearization: partition sets overlap");
  return TOPT_OK;
}

}  // namespace

extern "C" {

const char* topt_b200_version(void) { return "topt_b200 0.1 (sm_100a)"; }

void topt_b200_default_options(topt_proj_options* o) {
  o->c = 1e12; o->tol_b = 1e-8; o->tol_n = 1e-6; o->newton_maxiter = 50; o->binary_maxiter = 200;
}

void topt_b200_default_settings(topt_pgd_settings* s) {
  s->alpha_max = 1e2; s->alpha_fallback = 0.2; s->omega = 1.0; s->eps_alpha = 1e-6;
  s->tol_n = 1e-6; s->t_warmup = 50;
}

int topt_b200_ctx_create(int device, topt_b200_ctx** out) {
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= device) return TOPT_ERR_CUDA;
  topt_b200_ctx* ctx = new topt_b200_ctx();
  ctx->device = device;
  if (cudaSetDevice(device) != cudaSuccess) { delete ctx; return TOPT_ERR_CUDA; }
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, device);
  ctx->nsm = prop.multiProcessorCount;
  ctx->grid = ctx->nsm * 2;
  bool ok = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) == cudaSuccess;
  ctx->own_stream = ok;
  ok = ok && cudaMalloc(&ctx->d_plan, sizeof(Plan)) == cudaSuccess;
  ok = ok && cudaMalloc(&ctx->d_part, 2 * sizeof(double) * PMAX * ctx->grid) == cudaSuccess;
  ok = ok && cudaMalloc(&ctx->d_counter, sizeof(unsigned)) == cudaSuccess;
  ok = ok && cudaMalloc(&ctx->d_totals, sizeof(double) * PMAX) == cudaSuccess;
  ok = ok && cudaMalloc(&ctx->d_err, sizeof(int)) == cudaSuccess;
  ok = ok && cudaMallocHost(&ctx->h_phase, sizeof(int)) == cudaSuccess;
  ok = ok && cudaMemset(ctx->d_counter, 0, sizeof(unsigned)) == cudaSuccess;
  ok = ok && cudaMalloc(&ctx->d_trace, 128 * 8 * sizeof(unsigned long long)) == cudaSuccess;
  ok = ok && cudaMalloc(&ctx->d_blk_cnt, sizeof(int) * ctx->grid) == cudaSuccess;
  // gather buffers: contiguous (gather pass) or one GATHER_BLK region per CTA (fused)
  const size_t gcap = std::max<size_t>(GATHER_CAP, (size_t)ctx->grid * GATHER_BLK);
  ok = ok && cudaMalloc(&ctx->d_ga, sizeof(double) * gcap) == cudaSuccess;
  ok = ok && cudaMalloc(&ctx->d_gr, sizeof(double) * gcap) == cudaSuccess;
  ok = ok && cudaMalloc(&ctx->d_grow, sizeof(int) * gcap) == cudaSuccess;
  ok = ok && cudaMalloc(&ctx->d_gfix, sizeof(double) * 2 * MAX_M * ctx->grid) == cudaSuccess;
  {   // everything the SM offers a CTA beyond the kernels' static shared memory
    cudaFuncAttributes fa0, fa1;
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    size_t st = 0;
    if (cudaFuncGetAttributes(&fa0, k_step<false>) == cudaSuccess) st = fa0.sharedSizeBytes;
    if (cudaFuncGetAttributes(&fa1, k_step<true>) == cudaSuccess)
      st = std::max(st, (size_t)fa1.sharedSizeBytes);
    ctx->max_dyn_smem = (int)std::min<size_t>((size_t)optin - st - 1024, 200 * 1024);
    cudaGetLastError();
  }
  ok = ok && cudaFuncSetAttribute(k_step<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  ctx->max_dyn_smem) == cudaSuccess;
  ok = ok && cudaFuncSetAttribute(k_step<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  ctx->max_dyn_smem) == cudaSuccess;
  ok = ok && cudaFuncSetAttribute(k_pass, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(KPASS_SMEM + sizeof(double) * MAX_TAB)) == cudaSuccess;
  ok = ok && cudaFuncSetAttribute(k_control, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)sizeof(Plan)) == cudaSuccess;
  if (ok) {
    int per_sm = 0, coop = 0;
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device);
    int per_sm2 = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_step<false>, BLOCK, (int)sizeof(Plan));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm2, k_step<true>, BLOCK, (int)sizeof(Plan));
    per_sm = std::min(per_sm, per_sm2);
    ctx->coop_grid = coop ? per_sm * ctx->nsm : 0;
    if (ctx->coop_grid > ctx->grid) ctx->coop_grid = ctx->grid;
    if (const char* e = getenv("TOPT_B200_PERSISTENT")) ctx->persistent = atoi(e);
    if (const char* e = getenv("TOPT_B200_COMPACT")) ctx->compact = atoi(e);
  }
  ok = ok && cudaEventCreate(&ctx->ev0) == cudaSuccess;
  ok = ok && cudaEventCreate(&ctx->ev1) == cudaSuccess;
  ok = ok && cudaEventCreate(&ctx->evs0) == cudaSuccess;
  ok = ok && cudaEventCreate(&ctx->evs1) == cudaSuccess;
  ok = ok && cudaStreamCreateWithFlags(&ctx->cstream, cudaStreamNonBlocking) == cudaSuccess;
  ok = ok && cudaEventCreateWithFlags(&ctx->ev_copy, cudaEventDisableTiming) == cudaSuccess;
  ok = ok && cudaMalloc(&ctx->d_flags, sizeof(unsigned) * 4 * MAX_STREAM_CHUNKS) == cudaSuccess;
  ok = ok && cudaMemset(ctx->d_flags, 0, sizeof(unsigned) * 4 * MAX_STREAM_CHUNKS) == cudaSuccess;
  ok = ok && cudaMalloc(&ctx->d_timed_out, sizeof(int)) == cudaSuccess;
  ok = ok && cudaMalloc(&ctx->d_probe, sizeof(int)) == cudaSuccess;
  ok = ok && cudaMallocHost(&ctx->h_timed_out, sizeof(int)) == cudaSuccess;
  ok = ok && cudaMallocHost(&ctx->hp_pin, sizeof(Plan)) == cudaSuccess;
  if (getenv("TOPT_B200_PROGRESS")) {
    static unsigned long long* hprog = nullptr;
    if (!hprog && cudaHostAlloc(&hprog, 32 * sizeof(unsigned long long), cudaHostAllocMapped) == cudaSuccess) {
      std::memset(hprog, 0, 32 * sizeof(unsigned long long));
      unsigned long long* dprog = nullptr;
      cudaHostGetDevicePointer(&dprog, hprog, 0);
      cudaMemcpyToSymbol(g_progress, &dprog, sizeof(dprog));
      std::thread([] {
        for (;;) {
          std::this_thread::sleep_for(std::chrono::seconds(2));
          volatile unsigned long long* h = hprog;
          fprintf(stderr, "[progress] pass %llu phase %llu | run %llu sync %llu red %llu ctl %llu | ctas: start %llu run %llu sync %llu red %llu ctl %llu | c5 %llu c6 %llu c7 %llu c8 %llu c9 %llu\n",
                  h[0] >> 8, h[0] & 255, h[1], h[2], h[3], h[4], h[16], h[17], h[18], h[19], h[20],
                  h[21], h[22], h[23], h[24], h[25]);
        }
      }).detach();
    }
  }
  if (const char* e = getenv("TOPT_B200_STREAM")) ctx->stream_inputs = atoi(e);
  if (const char* e = getenv("TOPT_B200_PARITY")) ctx->parity = (std::strcmp(e, "strict") == 0);
  if (const char* e = getenv("TOPT_B200_EXDEBUG")) ctx->ex_debug = atoi(e);
  if (const char* e = getenv("TOPT_B200_FUSED_SWEEP")) ctx->fused_sweep = atoi(e);
  if (const char* e = getenv("TOPT_B200_SKETCH_MIN_N")) ctx->sketch_min_n = atoll(e);
  if (const char* e = getenv("TOPT_B200_PAT_HINT")) ctx->pat_hint_on = atoi(e);
  if (const char* e = getenv("TOPT_B200_FIRST_K")) ctx->first_k = atoi(e);
  if (!ok) { topt_b200_ctx_destroy(ctx); return TOPT_ERR_CUDA; }
  *out = ctx;
  return TOPT_OK;
}

void topt_b200_ctx_destroy(topt_b200_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  for (auto& b : ctx->bufs)
    if (b.p) cudaFree(b.p);
  cudaFree(ctx->d_plan);
  cudaFree(ctx->d_part);
  cudaFree(ctx->d_counter);
  cudaFree(ctx->d_totals);
  cudaFree(ctx->d_err);
  cudaFree(ctx->d_trace);
  if (ctx->comm && nccl().ok) nccl().CommDestroy((ncclComm_t)ctx->comm);
  cudaFree(ctx->d_rank_tot);
  cudaFree(ctx->d_gathered);
  cudaFree(ctx->d_blk_cnt);
  cudaFree(ctx->d_ga);
  cudaFree(ctx->d_gr);
  cudaFree(ctx->d_grow);
  cudaFree(ctx->d_gfix);
  if (ctx->h_phase) cudaFreeHost(ctx->h_phase);
  if (ctx->cstream) cudaStreamSynchronize(ctx->cstream);
  cudaFree(ctx->d_flags);
  cudaFree(ctx->d_timed_out);
  cudaFree(ctx->d_probe);
  if (ctx->h_timed_out) cudaFreeHost(ctx->h_timed_out);
  if (ctx->hp_pin) cudaFreeHost(ctx->hp_pin);
  if (ctx->ev_copy) cudaEventDestroy(ctx->ev_copy);
  if (ctx->ev_pass) cudaEventDestroy(ctx->ev_pass);
  if (ctx->ev_copied) cudaEventDestroy(ctx->ev_copied);
  if (ctx->cstream) cudaStreamDestroy(ctx->cstream);
  if (ctx->ev0) cudaEventDestroy(ctx->ev0);
  if (ctx->ev1) cudaEventDestroy(ctx->ev1);
  if (ctx->evs0) cudaEventDestroy(ctx->evs0);
  if (ctx->evs1) cudaEventDestroy(ctx->evs1);
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

const char* topt_b200_last_error(const topt_b200_ctx* ctx) { return ctx ? ctx->err.c_str() : ""; }
int64_t topt_b200_kernel_launches(const topt_b200_ctx* ctx) { return ctx ? ctx->launches : 0; }
void* topt_b200_get_stream(const topt_b200_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }
int topt_b200_set_structured_rows(topt_b200_ctx* ctx, int32_t m, const topt_row_desc* rows,
                                  const int64_t* grid, int64_t index_offset) {
  if (!ctx) return TOPT_ERR_INTERNAL;
  if (!rows || m <= 0) { ctx->srows_m = 0; return TOPT_OK; }
  if (m > MAX_M || !grid) return fail(ctx, TOPT_ERR_DOMAIN, "structured rows: bad arguments");
  for (int k = 0; k < m; ++k) ctx->srows[k] = rows[k];
  for (int a = 0; a < 3; ++a) ctx->sgrid[a] = grid[a];
  ctx->sidx_off = index_offset;
  ctx->srows_m = m;
  return TOPT_OK;
}

int topt_b200_set_parity(topt_b200_ctx* ctx, int mode) {
  if (!ctx) return TOPT_ERR_INTERNAL;
  if (mode != TOPT_PARITY_CERTIFIED && mode != TOPT_PARITY_STRICT)
    return fail(ctx, TOPT_ERR_PARAMETER, "topt_b200_set_parity: unknown mode");
  ctx->parity = mode;
  return TOPT_OK;
}

int topt_b200_get_parity(const topt_b200_ctx* ctx) { return ctx ? ctx->parity : -1; }

int topt_b200_set_stream(topt_b200_ctx* ctx, void* stream) {
  if (!ctx) return TOPT_ERR_INTERNAL;
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  ctx->stream = (cudaStream_t)stream;
  ctx->own_stream = false;
  return TOPT_OK;
}

// Debug: per-pass device timestamps of the last persistent launch
// (64 passes x 8 u64: start, block0 pass end, finisher start, reduce end,
// control end, phase, last CTA pass end).  enable=1 arms, enable=0 reads.
int topt_b200_debug_trace(topt_b200_ctx* ctx, int enable, unsigned long long* out) {
  if (!ctx) return TOPT_ERR_INTERNAL;
  ctx->trace_on = enable;
  if (out) {
    cudaStreamSynchronize(ctx->stream);
    cudaMemcpy(out, ctx->d_trace, 128 * 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  }
  return TOPT_OK;
}

int topt_b200_nccl_unique_id(unsigned char* out, size_t len) {
  NcclApi& api = nccl();
  if (!api.ok) return TOPT_ERR_UNSUPPORTED;
  if (len < sizeof(ncclUniqueId)) return TOPT_ERR_PARAMETER;
  ncclUniqueId id;
  if (api.GetUniqueId(&id) != ncclSuccess) return TOPT_ERR_CUDA;
  std::memcpy(out, &id, sizeof(id));
  return TOPT_OK;
}

int topt_b200_ctx_create_ranks(int device, int rank, int world, const unsigned char* nccl_id,
                               topt_b200_ctx** out) {
  *out = nullptr;
  NcclApi& api = nccl();
  if (!api.ok) return TOPT_ERR_UNSUPPORTED;
  if (world < 1 || rank < 0 || rank >= world) return TOPT_ERR_PARAMETER;
  topt_b200_ctx* ctx = nullptr;
  int rc = topt_b200_ctx_create(device, &ctx);
  if (rc) return rc;
  ncclUniqueId id;
  std::memcpy(&id, nccl_id, sizeof(id));
  ncclComm_t comm = nullptr;
  if (api.CommInitRank(&comm, world, id, rank) != ncclSuccess) {
    topt_b200_ctx_destroy(ctx);
    return TOPT_ERR_CUDA;
  }
  ctx->comm = comm;
  ctx->rank = rank;
  ctx->world = world;
  bool ok = cudaMalloc(&ctx->d_rank_tot, sizeof(double) * PMAX) == cudaSuccess;
  ok = ok && cudaMalloc(&ctx->d_gathered, sizeof(double) * PMAX * world) == cudaSuccess;
  ok = ok && cudaMemset(ctx->d_rank_tot, 0, sizeof(double) * PMAX) == cudaSuccess;
  if (!ok) { topt_b200_ctx_destroy(ctx); return TOPT_ERR_CUDA; }
  *out = ctx;
  return TOPT_OK;
}

int topt_b200_set_profiling(topt_b200_ctx* ctx, int enabled) {
  if (!ctx) return TOPT_ERR_INTERNAL;
  ctx->profile = enabled ? 1 : 0;
  return TOPT_OK;
}

int topt_b200_kernel_time(topt_b200_ctx* ctx, double* total_ms, int64_t* launches,
                          double* max_ms) {
  if (!ctx) return TOPT_ERR_INTERNAL;
  if (total_ms) *total_ms = ctx->prof_ms;
  if (launches) *launches = ctx->prof_n;
  if (max_ms) *max_ms = ctx->prof_max;
  ctx->prof_ms = 0.0;
  ctx->prof_max = 0.0;
  ctx->prof_n = 0;
  return TOPT_OK;
}

int topt_b200_step_time(topt_b200_ctx* ctx, double* total_ms, int64_t* jobs, double* max_ms) {
  if (!ctx) return TOPT_ERR_INTERNAL;
  if (total_ms) *total_ms = ctx->step_ms;
  if (jobs) *jobs = ctx->step_n;
  if (max_ms) *max_ms = ctx->step_max;
  ctx->step_ms = 0.0;
  ctx->step_max = 0.0;
  ctx->step_n = 0;
  return TOPT_OK;
}

int topt_b200_owner_map(topt_b200_ctx* ctx, int64_t n, int32_t m, const int64_t* part_offsets,
                        const int32_t* part_indices, int8_t* owner_dev) {
  cudaSetDevice(ctx->device);
  return owner_map_impl(ctx, n, m, part_offsets, part_indices, owner_dev);
}

// ----- host-buffer linearization helpers ----------------------------------
static int stage_lin(topt_b200_ctx* ctx, Plan& hp, const topt_linearization* lin, bool need_gd,
                     bool with_part) {
  const int64_t n = (int64_t)lin->num_vars;
  const int m = (int)lin->num_constraints;
  void* dgrad = nullptr;
  void* dgd = nullptr;
  int rc = upload(ctx, B_GRAD, lin->grad, sizeof(double) * (size_t)m * (size_t)n, &dgrad);
  if (rc) return rc;
  if (need_gd && lin->gd_step) {
    rc = upload(ctx, B_GD, lin->gd_step, sizeof(double) * (size_t)n, &dgd);
    if (rc) return rc;
  }
  hp.P.grad = (const double*)dgrad;
  hp.P.gd_step = (const double*)dgd;
  if (with_part && lin->part_offsets) {
    int8_t* own = (int8_t*)buf(ctx, B_OWNER, (size_t)std::max<int64_t>(n, 1));
    if (!own) return fail(ctx, TOPT_ERR_CUDA, "cudaMalloc failed");
    rc = owner_map_impl(ctx, n, m, lin->part_offsets, lin->part_indices, own);
    if (rc) return rc;
    hp.P.owner = own;
    hp.P.has_part = 1;
    apply_ranges(ctx, hp.P);
    set_part_lists(ctx, hp.P);
  }
  return TOPT_OK;
}

int topt_b200_build(topt_b200_ctx* ctx, const topt_linearization* lin, double* g_hat_out,
                    double* g_hat_err_out) {
  cudaSetDevice(ctx->device);
  Plan& hp = ctx->h_plan;
  const int64_t n = (int64_t)lin->num_vars;
  const int m = (int)lin->num_constraints;
  int rc = init_problem(ctx, hp, n, m, nullptr);
  if (rc) return rc;
  if (m == 0) return TOPT_OK;
  if (!lin->gd_step || !lin->grad || !lin->g_values || !lin->bounds_g)
    return fail(ctx, TOPT_ERR_DOMAIN, "ConstraintLinearization: inconsistent dimensions");
  hp.P.job = JOB_BUILD;
  set_lin_scalars(hp, lin);
  rc = stage_lin(ctx, hp, lin, true, true);
  if (rc) return rc;
  void* drho = buf(ctx, B_RHO, sizeof(double) * (size_t)std::max<int64_t>(n, 1));
  if (!drho) return fail(ctx, TOPT_ERR_CUDA, "cudaMalloc failed");
  CUDA_TRY(ctx, cudaMemsetAsync(drho, 0, sizeof(double) * (size_t)n, ctx->stream));
  hp.P.rho = (double*)drho;
  rc = run_plan(ctx, hp);
  if (rc == TOPT_ERR_DOMAIN)
    ctx->err = "ConstraintLinearization: gradient nonzero outside partition set";
  if (rc) return rc;
  for (int j = 0; j < m; ++j) {
    if (g_hat_out) g_hat_out[j] = hp.res.ghat[j];
    if (g_hat_err_out) g_hat_err_out[j] = hp.res.ghat_err[j];
  }
  return TOPT_OK;
}

static int small_job(topt_b200_ctx* ctx, int job, const double* y, const topt_linearization* lin,
                     const double* rho, double lower, double upper, double c, double* out) {
  cudaSetDevice(ctx->device);
  Plan& hp = ctx->h_plan;
  const int64_t n = (int64_t)lin->num_vars;
  const int m = (int)lin->num_constraints;
  int rc = init_problem(ctx, hp, n, m, nullptr);
  if (rc) return rc;
  if (job == JOB_RESIDUAL_H && !(c > 0.0))
    return fail(ctx, TOPT_ERR_PARAMETER, "constraint_residual_h: c must be > 0");
  hp.P.job = job;
  hp.P.lower = lower;
  hp.P.upper = upper;
  hp.P.opt.c = c;
  set_lin_scalars(hp, lin);
  for (int j = 0; j < m; ++j) hp.P.y_in[j] = y[j];
  rc = stage_lin(ctx, hp, lin, false, false);
  if (rc) return rc;
  void* drho = nullptr;
  rc = upload(ctx, B_RHO, rho, sizeof(double) * (size_t)n, &drho);
  if (rc) return rc;
  hp.P.rho = (double*)drho;
  double* ddelta = nullptr;
  if (job == JOB_DELTA && n > 0) {
    ddelta = (double*)buf(ctx, B_DELTA, sizeof(double) * (size_t)n);
    if (!ddelta) return fail(ctx, TOPT_ERR_CUDA, "cudaMalloc failed");
    hp.P.delta_out = ddelta;
  }
  rc = run_plan(ctx, hp);
  if (rc) return rc;
  if (job == JOB_DELTA) {
    if (n > 0)
      CUDA_TRY(ctx, cudaMemcpyAsync(out, ddelta, sizeof(double) * (size_t)n, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  } else {
    for (int j = 0; j < m; ++j) out[j] = hp.res.h[j];
  }
  return TOPT_OK;
}

int topt_b200_delta_of_y(topt_b200_ctx* ctx, const double* y, const topt_linearization* lin,
                         const double* rho_tilde, double lower, double upper,
                         double* delta_out) {
  return small_job(ctx, JOB_DELTA, y, lin, rho_tilde, lower, upper, 1e12, delta_out);
}

int topt_b200_constraint_residual_h(topt_b200_ctx* ctx, const double* y,
                                    const topt_linearization* lin, const double* rho_tilde,
                                    double lower, double upper, double c, double* h_out) {
  return small_job(ctx, JOB_RESIDUAL_H, y, lin, rho_tilde, lower, upper, c, h_out);
}

static int project_common(topt_b200_ctx* ctx, Plan& hp, int which, double lower, double upper,
                          double* y_out, double* slacks_out, topt_proj_meta* meta) {
  hp.P.job = JOB_PROJECT;
  hp.P.which = which;
  hp.P.lower = lower;
  hp.P.upper = upper;
  const int m = hp.P.m;
  if (which == W_SINGLE && m != 1)
    return fail(ctx, TOPT_ERR_DOMAIN, "project_single_binary_search: exactly one constraint required");
  if (which == W_INDEPENDENT && !hp.P.has_part)
    return fail(ctx, TOPT_ERR_DOMAIN, "project_independent: linearization has no partition");
  if ((which == W_NEWTON || (which == W_AUTO && m != 1 && !hp.P.has_part)) && m < 1)
    return fail(ctx, TOPT_ERR_DOMAIN, "project_general_newton: no constraints");
  int rc = run_plan(ctx, hp);
  if (rc == TOPT_ERR_DOMAIN && hp.res.status == ST_DOMAIN)
    ctx->err = "ConstraintLinearization: partition/g_hat validation failed";
  if (rc) return rc;
  for (int j = 0; j < m; ++j) {
    if (y_out) y_out[j] = hp.res.y[j];
    if (slacks_out) slacks_out[j] = hp.res.slacks[j];
  }
  fill_meta(hp, meta);
  return TOPT_OK;
}

int topt_b200_project(topt_b200_ctx* ctx, int which, const double* rho_tilde,
                      const topt_linearization* lin, double lower, double upper,
                      const topt_proj_options* opts, double* delta_out, double* y_out,
                      double* slacks_out, topt_proj_meta* meta) {
  cudaSetDevice(ctx->device);
  Plan& hp = ctx->h_plan;
  const int64_t n = (int64_t)lin->num_vars;
  const int m = (int)lin->num_constraints;
  int rc = init_problem(ctx, hp, n, m, opts);
  if (rc) return rc;
  set_lin_scalars(hp, lin);
  const bool use_part = lin->part_offsets && which != W_SINGLE && which != W_NEWTON && m > 1;
  rc = stage_lin(ctx, hp, lin, use_part, use_part || (which == W_INDEPENDENT && lin->part_offsets));
  if (rc) return rc;
  void* drho = nullptr;
  rc = upload(ctx, B_RHO, rho_tilde, sizeof(double) * (size_t)n, &drho);
  if (rc) return rc;
  hp.P.rho = (double*)drho;
  double* dd = nullptr;
  if (delta_out && n > 0) {
    dd = (double*)buf(ctx, B_DELTA, sizeof(double) * (size_t)n);
    if (!dd) return fail(ctx, TOPT_ERR_CUDA, "cudaMalloc failed");
  }
  hp.P.delta_out = dd;
  if (which == W_INDEPENDENT && !lin->part_offsets) hp.P.has_part = 0;
  rc = project_common(ctx, hp, which, lower, upper, y_out, slacks_out, meta);
  if (rc) return rc;
  if (dd)
    CUDA_TRY(ctx, cudaMemcpyAsync(delta_out, dd, sizeof(double) * (size_t)n, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return TOPT_OK;
}

int topt_b200_project_dev(topt_b200_ctx* ctx, int which, const double* rho_tilde,
                          const topt_linearization* lin, double lower, double upper,
                          const topt_proj_options* opts, double* delta_out, uint8_t* mask_out,
                          double* y_out, double* slacks_out, topt_proj_meta* meta) {
  cudaSetDevice(ctx->device);
  Plan& hp = ctx->h_plan;
  const int64_t n = (int64_t)lin->num_vars;
  const int m = (int)lin->num_constraints;
  int rc = init_problem(ctx, hp, n, m, opts);
  if (rc) return rc;
  set_lin_scalars(hp, lin);
  hp.P.grad = lin->grad;
  hp.P.gd_step = lin->gd_step;
  const bool use_part = lin->owner && which != W_SINGLE && which != W_NEWTON && m > 1;
  hp.P.owner = use_part ? lin->owner : nullptr;
  apply_ranges(ctx, hp.P);
  hp.P.has_part = use_part ? 1 : 0;
  hp.P.rho = const_cast<double*>(rho_tilde);
  hp.P.delta_out = delta_out;
  hp.P.mask_out = mask_out;
  return project_common(ctx, hp, which, lower, upper, y_out, slacks_out, meta);
}

static int pgd_step_impl(topt_b200_ctx* ctx, Plan& hp, const topt_step_problem* prob,
                         const topt_pgd_settings* s, const topt_proj_options* opts,
                         topt_proj_meta* meta, double* y, double* slacks, double* ghat,
                         int job = JOB_PGD_STEP, const StreamIn* si = nullptr) {
  Problem& P = hp.P;
  P.job = job;
  P.which = W_AUTO;
  P.t = prob->t;
  P.violation = prob->violation;
  P.lower = prob->lower;
  P.upper = prob->upper;
  if (s) {
    P.set.alpha_max = s->alpha_max; P.set.alpha_fallback = s->alpha_fallback;
    P.set.omega = s->omega; P.set.eps_alpha = s->eps_alpha; P.set.tol_n = s->tol_n;
    P.set.t_warmup = s->t_warmup;
  } else {
    P.set.alpha_max = 1e2; P.set.alpha_fallback = 0.2; P.set.omega = 1.0;
    P.set.eps_alpha = 1e-6; P.set.tol_n = 1e-6; P.set.t_warmup = 50;
  }
  for (int j = 0; j < P.m; ++j) {
    P.G_minus_g[j] = prob->bounds_g[j] - prob->g_values[j];
    P.is_eq[j] = prob->is_equality ? (prob->is_equality[j] ? 1 : 0) : 0;
    if (prob->part_offsets)
      P.row_count[j] = (double)(prob->part_offsets[j + 1] - prob->part_offsets[j]);
  }
  int rc = run_plan(ctx, hp, si);
  if (rc) return rc;
  for (int j = 0; j < P.m; ++j) {
    if (y) y[j] = hp.res.y[j];
    if (slacks) slacks[j] = hp.res.slacks[j];
    if (ghat) ghat[j] = hp.res.ghat[j];
  }
  fill_meta(hp, meta);
  return TOPT_OK;
}

int topt_b200_pgd_step_ranks(topt_b200_ctx* ctx, const topt_step_problem* prob,
                             int64_t n_global, const int64_t* row_counts,
                             const topt_pgd_settings* settings, const topt_proj_options* opts,
                             const topt_step_outputs* out, topt_proj_meta* meta) {
  if (!ctx->comm && !ctx->lockstep)
    return fail(ctx, TOPT_ERR_PARAMETER, "context has no NCCL communicator");
  ctx->n_global_override = n_global;
  ctx->row_counts_override = row_counts;
  const int rc = topt_b200_pgd_step_dev(ctx, prob, settings, opts, out, meta);
  ctx->n_global_override = 0;
  ctx->row_counts_override = nullptr;
  return rc;
}

int topt_b200_pgd_step_dev(topt_b200_ctx* ctx, const topt_step_problem* prob,
                           const topt_pgd_settings* settings, const topt_proj_options* opts,
                           const topt_step_outputs* out, topt_proj_meta* meta) {
  cudaSetDevice(ctx->device);
  Plan& hp = ctx->h_plan;
  int rc = init_problem(ctx, hp, prob->n, prob->m, opts);
  if (rc) return rc;
  if (ctx->n_global_override > 0) {
    hp.P.n_global = ctx->n_global_override;
    for (int j = 0; j < prob->m; ++j)
      hp.P.row_count[j] = ctx->row_counts_override ? (double)ctx->row_counts_override[j]
                                                   : (double)ctx->n_global_override;
  }
  if (!out->rho_tilde || !out->d)
    return fail(ctx, TOPT_ERR_DOMAIN, "pgd_step_dev: rho_tilde and d outputs are required");
  Problem& P = hp.P;
  P.x = prob->x; P.x_prev = prob->x_prev; P.g = prob->g; P.g_prev = prob->g_prev;
  P.d_prev = prob->d_prev; P.grad = prob->grad;
  P.owner = (prob->owner && prob->m > 1) ? prob->owner : nullptr;
  apply_ranges(ctx, P);
  if ((rc = apply_structured(ctx, P))) return rc;
  P.has_part = P.owner ? 1 : 0;
  P.rho = out->rho_tilde; P.d_out = out->d; P.x_out = out->x_new; P.delta_out = out->delta;
  P.mask_out = out->mask;
  return pgd_step_impl(ctx, hp, prob, settings, opts, meta, out->y, out->slacks, out->g_hat);
}

static int pgd_step_host(topt_b200_ctx* ctx, const topt_step_problem* prob,
                         const topt_pgd_settings* settings, const topt_proj_options* opts,
                         const topt_step_outputs* out, topt_proj_meta* meta, bool allow_stream) {
  Plan& hp = ctx->h_plan;
  const int64_t n = prob->n;
  const int m = prob->m;
  int rc = init_problem(ctx, hp, n, m, opts);
  if (rc) return rc;
  const size_t nb = sizeof(double) * (size_t)std::max<int64_t>(n, 1);
  void *dx, *dxp, *dg, *dgp, *ddp, *dgrad;
  // Stream the inputs into the running kernel (copies overlap the BB/PR+ and
  // PREP passes) when the persistent path and the stream memory operations
  // are available; otherwise upload first.
  const bool streamed = allow_stream && ctx->stream_inputs && !ctx->comm && ctx->persistent &&
                        ctx->coop_grid > 0 && n > 0 && m >= 1 && memops().ok &&
                        prob->x && prob->x_prev && prob->g && prob->g_prev && prob->d_prev &&
                        prob->grad;
  if (streamed) {
    dx = buf(ctx, B_X, nb); dxp = buf(ctx, B_XP, nb); dg = buf(ctx, B_G, nb);
    dgp = buf(ctx, B_GP, nb); ddp = buf(ctx, B_DP, nb); dgrad = buf(ctx, B_GRAD, nb * (size_t)m);
    if (!dx || !dxp || !dg || !dgp || !ddp || !dgrad)
      return fail(ctx, TOPT_ERR_CUDA, "cudaMalloc failed");
  } else {
    if ((rc = upload(ctx, B_X, prob->x, nb, &dx))) return rc;
    if ((rc = upload(ctx, B_XP, prob->x_prev, nb, &dxp))) return rc;
    if ((rc = upload(ctx, B_G, prob->g, nb, &dg))) return rc;
    if ((rc = upload(ctx, B_GP, prob->g_prev, nb, &dgp))) return rc;
    if ((rc = upload(ctx, B_DP, prob->d_prev, nb, &ddp))) return rc;
    if ((rc = upload(ctx, B_GRAD, prob->grad, nb * (size_t)m, &dgrad))) return rc;
  }
  Problem& P = hp.P;
  P.x = (const double*)dx; P.x_prev = (const double*)dxp; P.g = (const double*)dg;
  P.g_prev = (const double*)dgp; P.d_prev = (const double*)ddp; P.grad = (const double*)dgrad;
  if (prob->part_offsets && m > 1) {
    int8_t* own = (int8_t*)buf(ctx, B_OWNER, (size_t)std::max<int64_t>(n, 1));
    if (!own) return fail(ctx, TOPT_ERR_CUDA, "cudaMalloc failed");
    if ((rc = owner_map_impl(ctx, n, m, prob->part_offsets, prob->part_indices, own))) return rc;
    P.owner = own;
    P.has_part = 1;
    apply_ranges(ctx, P);
    set_part_lists(ctx, P);
  }
  P.rho = (double*)buf(ctx, B_RHO, nb);
  P.d_out = (double*)buf(ctx, B_D, nb);
  P.x_out = (double*)buf(ctx, B_XNEW, nb);
  P.delta_out = out->delta ? (double*)buf(ctx, B_DELTA, nb) : nullptr;
  P.mask_out = out->mask ? (uint8_t*)buf(ctx, B_MASK, (size_t)std::max<int64_t>(n, 1)) : nullptr;
  if (!P.rho || !P.d_out || !P.x_out) return fail(ctx, TOPT_ERR_CUDA, "cudaMalloc failed");
  StreamIn si{};
  if (streamed) {
    int64_t nch = (n + (1 << 18) - 1) >> 18;   // ~2 MB per array per chunk
    nch = std::max<int64_t>(1, std::min<int64_t>(nch, MAX_STREAM_CHUNKS));
    P.chunk = (((n + nch - 1) / nch) + 63) & ~int64_t(63);   // even: 16-byte pairs
    P.nchunk = (int32_t)((n + P.chunk - 1) / P.chunk);
    P.epoch = ++ctx->epoch;
    P.in_flags = ctx->d_flags;
    P.out_flag = ctx->d_flags + 2 * MAX_STREAM_CHUNKS;
    si = StreamIn{prob->x, prob->x_prev, prob->g, prob->g_prev, prob->d_prev, prob->grad,
                  (double*)dx, (double*)dxp, (double*)dg, (double*)dgp, (double*)ddp,
                  (double*)dgrad, m, out->d, P.d_out};
  }
  rc = pgd_step_impl(ctx, hp, prob, settings, opts, meta, out->y, out->slacks, out->g_hat,
                     JOB_PGD_STEP, streamed ? &si : nullptr);
  if (rc) return rc;
  const size_t nbytes = sizeof(double) * (size_t)n;
  if (n > 0) {
    if (out->x_new) CUDA_TRY(ctx, cudaMemcpyAsync(out->x_new, P.x_out, nbytes, cudaMemcpyDeviceToHost, ctx->stream));
    if (out->d && !streamed) CUDA_TRY(ctx, cudaMemcpyAsync(out->d, P.d_out, nbytes, cudaMemcpyDeviceToHost, ctx->stream));
    if (out->rho_tilde) CUDA_TRY(ctx, cudaMemcpyAsync(out->rho_tilde, P.rho, nbytes, cudaMemcpyDeviceToHost, ctx->stream));
    if (out->delta) CUDA_TRY(ctx, cudaMemcpyAsync(out->delta, P.delta_out, nbytes, cudaMemcpyDeviceToHost, ctx->stream));
    if (out->mask) CUDA_TRY(ctx, cudaMemcpyAsync(out->mask, P.mask_out, (size_t)n, cudaMemcpyDeviceToHost, ctx->stream));
  }
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return TOPT_OK;
}

// Is host-buffer streaming usable on this context?  Probed once: a kernel
// spins on a flag the copy stream writes after the launch.
static bool stream_usable(topt_b200_ctx* ctx) {
  if (ctx->stream_probe >= 0) return ctx->stream_probe == 1;
  ctx->stream_probe = 0;
  MemOps& mo = memops();
  if (!mo.ok) return false;
  const uint32_t ep = ++ctx->epoch;
  unsigned* flag = ctx->d_flags + 3 * MAX_STREAM_CHUNKS;
  if (cudaMemsetAsync(ctx->d_probe, 0, sizeof(int), ctx->stream) != cudaSuccess) return false;
  if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return false;
  k_stream_probe<<<1, 32, 0, ctx->stream>>>(flag, ep, ctx->d_probe);
  ctx->launches++;
  if (mo.write32((CUstream)ctx->cstream, (CUdeviceptr)flag, ep, 0) != CUDA_SUCCESS) {
    cudaStreamSynchronize(ctx->stream);
    cudaGetLastError();
    return false;
  }
  int seen = 0;
  const bool ok = cudaStreamSynchronize(ctx->cstream) == cudaSuccess &&
                  cudaMemcpyAsync(&seen, ctx->d_probe, sizeof(int), cudaMemcpyDeviceToHost,
                                  ctx->stream) == cudaSuccess &&
                  cudaStreamSynchronize(ctx->stream) == cudaSuccess;
  cudaGetLastError();
  ctx->stream_probe = (ok && seen) ? 1 : 0;
  return ctx->stream_probe == 1;
}

int topt_b200_pgd_step(topt_b200_ctx* ctx, const topt_step_problem* prob,
                       const topt_pgd_settings* settings, const topt_proj_options* opts,
                       const topt_step_outputs* out, topt_proj_meta* meta) {
  cudaSetDevice(ctx->device);
  const bool try_stream = ctx->stream_inputs && ctx->persistent && ctx->coop_grid > 0 &&
                          !ctx->comm && stream_usable(ctx);
  const int rc = pgd_step_host(ctx, prob, settings, opts, out, meta, try_stream);
  if (rc == TOPT_ERR_CUDA && try_stream && ctx->stream_timeout) {
    // the copies did not overlap the running kernel after all (e.g. a
    // profiler serialized this launch): upload first from now on
    ctx->stream_timeout = 0;
    ctx->stream_probe = 0;
    return pgd_step_host(ctx, prob, settings, opts, out, meta, false);
  }
  return rc;
}

int topt_b200_step_direction(topt_b200_ctx* ctx, int64_t n, const double* x,
                             const double* x_prev, const double* g, const double* g_prev,
                             const double* d_prev, int32_t t, double violation,
                             const topt_pgd_settings* settings, double* d_out,
                             double* rho_tilde_out, double* alpha_out, double* beta_out,
                             int32_t* fallback_out) {
  cudaSetDevice(ctx->device);
  Plan& hp = ctx->h_plan;
  int rc = init_problem(ctx, hp, n, 0, nullptr);
  if (rc) return rc;
  const size_t nb = sizeof(double) * (size_t)std::max<int64_t>(n, 1);
  void *dx, *dxp, *dg, *dgp, *ddp;
  if ((rc = upload(ctx, B_X, x, nb, &dx))) return rc;
  if ((rc = upload(ctx, B_XP, x_prev, nb, &dxp))) return rc;
  if ((rc = upload(ctx, B_G, g, nb, &dg))) return rc;
  if ((rc = upload(ctx, B_GP, g_prev, nb, &dgp))) return rc;
  if ((rc = upload(ctx, B_DP, d_prev, nb, &ddp))) return rc;
  Problem& P = hp.P;
  P.x = (const double*)dx; P.x_prev = (const double*)dxp; P.g = (const double*)dg;
  P.g_prev = (const double*)dgp; P.d_prev = (const double*)ddp;
  P.rho = (double*)buf(ctx, B_RHO, nb);
  P.d_out = (double*)buf(ctx, B_D, nb);
  if (!P.rho || !P.d_out) return fail(ctx, TOPT_ERR_CUDA, "cudaMalloc failed");
  topt_step_problem pr;
  std::memset(&pr, 0, sizeof(pr));
  pr.n = n; pr.t = t; pr.violation = violation; pr.lower = 0.0; pr.upper = 1.0;
  rc = pgd_step_impl(ctx, hp, &pr, settings, nullptr, nullptr, nullptr, nullptr, nullptr,
                     JOB_DIRECTION);
  if (rc) return rc;
  if (n > 0) {
    if (d_out) CUDA_TRY(ctx, cudaMemcpyAsync(d_out, P.d_out, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
    if (rho_tilde_out) CUDA_TRY(ctx, cudaMemcpyAsync(rho_tilde_out, P.rho, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
  }
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  if (alpha_out) *alpha_out = hp.res.alpha;
  if (beta_out) *beta_out = hp.res.beta;
  if (fallback_out) *fallback_out = hp.res.fallback;
  return TOPT_OK;
}

// ---- single-process lockstep ranks (the multi-rank data plane without NCCL) ----
int topt_b200_ctx_create_lockstep(int device, int rank, int world, topt_b200_ctx** out) {
  *out = nullptr;
  if (world < 1 || rank < 0 || rank >= world) return TOPT_ERR_PARAMETER;
  topt_b200_ctx* ctx = nullptr;
  int rc = topt_b200_ctx_create(device, &ctx);
  if (rc) return rc;
  ctx->rank = rank;
  ctx->world = world;
  ctx->lockstep = 1;
  bool ok = cudaMalloc(&ctx->d_rank_tot, sizeof(double) * PMAX) == cudaSuccess;
  ok = ok && cudaMalloc(&ctx->d_gathered, sizeof(double) * PMAX * world) == cudaSuccess;
  ok = ok && cudaMemset(ctx->d_rank_tot, 0, sizeof(double) * PMAX) == cudaSuccess;
  ok = ok && cudaEventCreateWithFlags(&ctx->ev_pass, cudaEventDisableTiming) == cudaSuccess;
  ok = ok && cudaEventCreateWithFlags(&ctx->ev_copied, cudaEventDisableTiming) == cudaSuccess;
  if (!ok) { topt_b200_ctx_destroy(ctx); return TOPT_ERR_CUDA; }
  *out = ctx;
  return TOPT_OK;
}

int topt_b200_pgd_step_lockstep(int world, topt_b200_ctx* const* ctxs,
                                const topt_step_problem* probs, int64_t n_global,
                                const int64_t* row_counts, const topt_pgd_settings* settings,
                                const topt_proj_options* opts, const topt_step_outputs* outs,
                                topt_proj_meta* metas) {
  if (world < 1 || !ctxs) return TOPT_ERR_PARAMETER;
  for (int r = 0; r < world; ++r)
    if (!ctxs[r] || !ctxs[r]->lockstep || ctxs[r]->rank != r || ctxs[r]->world != world)
      return TOPT_ERR_PARAMETER;
  // every rank's plan: the ranks entry prepares it and stops before the passes
  for (int r = 0; r < world; ++r) {
    topt_b200_ctx* c = ctxs[r];
    c->defer = 1;
    const int rc = topt_b200_pgd_step_ranks(c, &probs[r], n_global, row_counts, settings, opts,
                                            &outs[r], metas ? &metas[r] : nullptr);
    c->defer = 0;
    if (rc != TOPT_DEFERRED) return rc ? rc : TOPT_ERR_INTERNAL;
  }
  int phase = ctxs[0]->h_plan.cmd.phase;
  for (int it = 0; phase != PH_DONE && it < 4096; it += RANK_BATCH) {
    for (int b = 0; b < RANK_BATCH; ++b) {
      for (int q = 0; q < world; ++q) {   // pass kernels (after last pass's copies of q's totals)
        topt_b200_ctx* c = ctxs[q];
        cudaSetDevice(c->device);
        if (it + b > 0)
          for (int r = 0; r < world; ++r) CUDA_TRY(c, cudaStreamWaitEvent(c->stream, ctxs[r]->ev_copied, 0));
        if (int rc = ranks_pass_kernel(c, c->h_plan)) return rc;
        CUDA_TRY(c, cudaEventRecord(c->ev_pass, c->stream));
      }
      for (int r = 0; r < world; ++r) {   // the all-gather, as device copies
        topt_b200_ctx* c = ctxs[r];
        cudaSetDevice(c->device);
        for (int q = 0; q < world; ++q) {
          CUDA_TRY(c, cudaStreamWaitEvent(c->stream, ctxs[q]->ev_pass, 0));
          CUDA_TRY(c, cudaMemcpyPeerAsync(c->d_gathered + (size_t)q * PMAX, c->device,
                                          ctxs[q]->d_rank_tot, ctxs[q]->device,
                                          sizeof(double) * PMAX, c->stream));
        }
        CUDA_TRY(c, cudaEventRecord(c->ev_copied, c->stream));
        if (int rc = ranks_control_kernel(c)) return rc;
      }
    }
    int ph0 = -1;
    for (int r = 0; r < world; ++r) {
      topt_b200_ctx* c = ctxs[r];
      cudaSetDevice(c->device);
      CUDA_TRY(c, cudaMemcpyAsync(c->h_phase, &c->d_plan->cmd.phase, sizeof(int),
                                  cudaMemcpyDeviceToHost, c->stream));
      CUDA_TRY(c, cudaStreamSynchronize(c->stream));
      if (r == 0) ph0 = *c->h_phase;
      else if (*c->h_phase != ph0)
        return fail(c, TOPT_ERR_INTERNAL, "lockstep ranks diverged");
    }
    phase = ph0;
  }
  for (int r = 0; r < world; ++r) {
    topt_b200_ctx* c = ctxs[r];
    cudaSetDevice(c->device);
    Plan& hp = c->h_plan;
    if (int rc = ranks_finish(c, hp, phase)) return rc;
    for (int j = 0; j < hp.P.m; ++j) {
      if (outs[r].y) outs[r].y[j] = hp.res.y[j];
      if (outs[r].slacks) outs[r].slacks[j] = hp.res.slacks[j];
      if (outs[r].g_hat) outs[r].g_hat[j] = hp.res.ghat[j];
    }
    if (metas) fill_meta(hp, &metas[r]);
  }
  return TOPT_OK;
}

}  // extern "C"
