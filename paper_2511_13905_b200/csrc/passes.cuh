// passes.cuh — the O(n) passes of the PGD-TO step (device code).
//
// Every pass is a grid-stride sweep over this rank's slab that produces a
// small vector of partial sums (<= PMAX slots) per CTA.  Reductions are
// deterministic: a fixed per-thread order, a fixed shuffle tree per warp, a
// fixed warp order per CTA, and a fixed CTA order in the final combine, so
// the same inputs on the same launch geometry give the same bits.
//
// Element arithmetic follows projection.cpp exactly (the library is built
// with -fmad=false, so every product and sum is separately rounded):
//   lo = lower - rho_i, hi = upper - rho_i             (:32, :207)
//   clip(v, lo, hi) = v < lo ? lo : (v > hi ? hi : v)   (:15-17)
//   term = a_i * clip(y * a_i, lo, hi)                  (:32, :35)
//   z_i = sum_{j: y_j != 0} y_j a_ji, ascending j, from 0.0  (:199-205)
#pragma once
#include <type_traits>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cooperative_groups.h>

#include "controller.h"
#include "topt_core.h"

namespace topt_b200 {
namespace cg = cooperative_groups;

constexpr int BLOCK = 512;
constexpr int NWARP = BLOCK / 32;

__device__ __forceinline__ double clipd(double v, double lo, double hi) {
  return v < lo ? lo : (v > hi ? hi : v);
}

__device__ __forceinline__ double apply_op(int op, double a, double b) {
  return op == 0 ? a + b : (op == 1 ? dmin_(a, b) : dmax_(a, b));
}

// Deterministic shuffle tree; lane 0 ends with the warp's value.
__device__ __forceinline__ double warp_reduce(int op, double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v = apply_op(op, v, __shfl_down_sync(0xffffffffu, v, off));
  return v;
}

__host__ __device__ constexpr int pow2_at_least(int n) { return n <= 1 ? 1 : 2 * pow2_at_least((n + 1) / 2); }

// Warp stage of a many-slot reduction by recursive halving: at each of the 5
// butterfly levels a lane keeps half of its slots and receives the partner's
// copy of them, so NS slots cost ~NS shuffles instead of 5 NS.  Every lane
// then writes the warp totals of the slots it ended with to wsum[slot]
// (slots < NS only; a slot held by several lanes is written by the lowest).
// The order of the additions is fixed, so results are deterministic.
// MINMAX: some slots reduce with min/max (slot_op(phase, slot0 + slot)).
template <int NS, bool MINMAX>
__device__ __forceinline__ void warp_reduce_slots(const double (&v)[NS], int phase, int slot0,
                                                  double* wsum) {
  constexpr int P = pow2_at_least(NS);
  const int lane = threadIdx.x & 31;
  double a[NS];   // slots >= NS of the padded power-of-two layout are zeros
#pragma unroll
  for (int s = 0; s < NS; ++s) a[s] = v[s];
  int base = 0;
  bool writer = true;
#pragma unroll
  for (int lev = 0; lev < 5; ++lev) {
    const int o = 16 >> lev;
    const int c = (P >> lev) > 1 ? (P >> lev) : 1;   // values held before this level
    const bool up = (lane & o) != 0;
    if (c > 1) {
      const int h = c / 2;
#pragma unroll
      for (int i = 0; i < h; ++i) {
        if (i >= NS) break;
        const double lo_v = a[i];
        const double hi_v = (h + i < NS) ? a[h + i] : 0.0;
        const double keep = up ? hi_v : lo_v;
        const double send = up ? lo_v : hi_v;
        const double recv = __shfl_xor_sync(0xffffffffu, send, o);
        const int op = MINMAX ? slot_op(phase, slot0 + base + (up ? h : 0) + i) : 0;
        // lower lane of the pair first: the same expression on both sides
        a[i] = up ? apply_op(op, recv, keep) : apply_op(op, keep, recv);
      }
      if (up) base += h;
    } else {
      const double recv = __shfl_xor_sync(0xffffffffu, a[0], o);
      const int op = MINMAX ? slot_op(phase, slot0 + base) : 0;
      a[0] = up ? apply_op(op, recv, a[0]) : apply_op(op, a[0], recv);
      if (up) writer = false;
    }
  }
  constexpr int F = P >= 32 ? P / 32 : 1;
  if (writer) {
#pragma unroll
    for (int i = 0; i < F && i < NS; ++i)
      if (base + i < NS) wsum[base + i] = a[i];
  }
}

// Reduce NS per-thread values (compile-time count) across the CTA and write
// them to out[slot0 + s] for s < ns (ns <= NS, runtime).
template <int NS>
__device__ __forceinline__ void block_reduce_store(const double (&v)[NS], int ns, int phase,
                                                   int slot0, double* out, double* smem) {
  const int warp = threadIdx.x >> 5;
  // phases with min / max slots (PREP breakpoints, STEP_REDUCE's max |g|)
  if (phase == PH_PREP || phase == PH_STEP_REDUCE)
    warp_reduce_slots<NS, true>(v, phase, slot0, smem + warp * NS);
  else warp_reduce_slots<NS, false>(v, phase, slot0, smem + warp * NS);
  __syncthreads();
  if (threadIdx.x < ns) {
    const int s = threadIdx.x;
    const int op = slot_op(phase, slot0 + s);
    double r = smem[s];
    for (int w = 1; w < NWARP; ++w) r = apply_op(op, r, smem[w * NS + s]);
    out[slot0 + s] = r;
  }
  __syncthreads();
}

struct PassCtx {
  const Plan* plan;
  const Cmd* cmd;      // shared-memory copy
  double* out;         // this CTA's partial slots
  double* smem;        // reduction scratch (NWARP * 160 doubles)
  int64_t i0, stride;  // grid-stride
  // persistent-kernel only (null otherwise): per-warp active element lists
  // and per-CTA fixed sums of the compacted bisection sweeps.
  uint32_t* list;      // [NWARP][list_cap]
  int* list_cnt;       // [NWARP]
  int* seg;            // [NWARP][MAX_M][2] range partitions: row j's (start, count) in a warp list
  double* fixC;        // [MAX_M]
  double* fixS;        // [MAX_M]
  int list_cap;
  // gather / local sweeps (persistent kernel only)
  int* blk_cnt;        // global [nb]: active items per CTA after a compacted sweep
  double* g_a;         // global [GATHER_CAP]
  double* g_r;
  int* g_row;
  double* g_fix;       // global [nb][MAX_M][2]
  double* it_a;        // shared [GATHER_CAP] gathered items
  double* it_r;
  int8_t* it_row;
  int* n_items;        // shared scalar
  int* timed_out;      // global flag: a streamed input chunk never arrived
  const double* rtab;  // shared centroid tables of structured rows (P.n_tab entries)
  void* ex_smem;       // chain ring + mbarriers in dynamic shared memory (strict parity)
  void* ms_smem;       // fused multi-row sweep queues / accumulators (or null)
};

// ---- Structured constraint rows ------------------------------------------------
// Rows the caller describes instead of storing:
// constant rows (the volume row, a_i = 1) and centroid rows
// a_i = sign * ((coord_axis(i) + 0.5) - center) / scale (the centre-of-mass
// rows, grid.hpp:29-33).  A pass then reads rho (and d) only.
// The centroid values come from a per-launch shared-memory table built with
// the same IEEE operations as the dense rows, so results are bit-identical.
struct GridIx {
  int64_t nx, ny, off;
  int sx, sy;          // log2 of nx / ny when powers of two, else -1
};
__device__ __forceinline__ GridIx grid_ix(const Problem& P) {
  GridIx G;
  G.nx = P.grid_n[0]; G.ny = P.grid_n[1]; G.off = P.idx_off;
  G.sx = (G.nx > 0 && (G.nx & (G.nx - 1)) == 0) ? __ffsll(G.nx) - 1 : -1;
  G.sy = (G.ny > 0 && (G.ny & (G.ny - 1)) == 0) ? __ffsll(G.ny) - 1 : -1;
  return G;
}
// x-fastest coordinates of global element gi
__device__ __forceinline__ void grid_coords(const GridIx& G, int64_t gi, int64_t (&co)[3]) {
  if (G.sx >= 0 && G.sy >= 0) {
    co[0] = gi & (G.nx - 1);
    const int64_t q = gi >> G.sx;
    co[1] = q & (G.ny - 1);
    co[2] = q >> G.sy;
  } else if (gi >= 0 && gi < (int64_t)0xffffffffLL) {
    const uint32_t g = (uint32_t)gi, nx = (uint32_t)G.nx, ny = (uint32_t)G.ny;
    const uint32_t q = g / nx;
    co[0] = g - q * nx;
    co[2] = q / ny;
    co[1] = q - (uint32_t)co[2] * ny;
  } else {
    const int64_t q = gi / G.nx;
    co[0] = gi - q * G.nx;
    co[2] = q / G.ny;
    co[1] = q - co[2] * G.ny;
  }
}
// Structured row k as one packed int, hoisted out of the element loops:
// table offset | table axis << 24 (3: constant row, entry 0) | negate << 27.
__device__ __forceinline__ int srow_code(const Problem& P, int k) {
  const int ax = P.row_kind[k] == RK_CONST ? 3 : P.row_axis[k];
  return P.row_tab[k] | (ax << 24) | ((P.row_sign[k] < 0.0 ? 1 : 0) << 27);
}
__device__ __forceinline__ double srow_fetch(const double* tab, int code, const int64_t (&co)[3]) {
  const int ax = (code >> 24) & 7;
  const int64_t ci = ax == 0 ? co[0] : (ax == 1 ? co[1] : (ax == 2 ? co[2] : 0));
  const double v = tab[(code & 0xffffff) + ci];
  return ((code >> 27) & 1) ? -v : v;
}

// The centre-of-mass pattern (P.axis_fast): per element four values --
// tv[a] = tab[axis_tab[a] + c_a] for the three axes and tv[3] = the constant
// row's entry -- and every structured row is +-tv[code & 3] (code: one int).
struct AxisRows {
  int tab[4];
  __device__ __forceinline__ void init(const Problem& P) {
    for (int a = 0; a < 3; ++a) tab[a] = P.axis_tab[a];
    tab[3] = P.const_tab;
  }
  __device__ __forceinline__ void values(const double* t, const int64_t (&co)[3],
                                         double (&tv)[4]) const {
#pragma unroll
    for (int a = 0; a < 3; ++a) tv[a] = tab[a] >= 0 ? t[tab[a] + co[a]] : 0.0;
    tv[3] = tab[3] >= 0 ? t[tab[3]] : 0.0;
  }
};
__device__ __forceinline__ int row_pick_code(const Problem& P, int k) {
  const int ax = P.row_kind[k] == RK_CONST ? 3 : P.row_axis[k];
  return ax | ((P.row_sign[k] < 0.0 && P.row_kind[k] != RK_CONST) ? 4 : 0);
}
__device__ __forceinline__ double row_pick(int code, const double (&tv)[4]) {
  const int ax = code & 3;
  const double v = ax == 0 ? tv[0] : (ax == 1 ? tv[1] : (ax == 2 ? tv[2] : tv[3]));
  return (code & 4) ? -v : v;
}

// Build the row tables (every CTA, at the start of a launch): one entry per
// constant row, one per grid coordinate for each distinct centroid row.
__device__ __forceinline__ void build_row_tables(const Problem& P, double* tab) {
  if (!P.structured) return;
  for (int k = 0; k < P.m; ++k) {
    if (P.row_kind[k] == RK_CONST) {
      if (threadIdx.x == 0) tab[P.row_tab[k]] = P.row_c[k];
      continue;
    }
    if (P.row_kind[k] != RK_CENTROID) continue;
    bool first = true;   // rows sharing (axis, center, scale) share one table
    for (int j = 0; j < k; ++j)
      if (P.row_kind[j] == RK_CENTROID && P.row_tab[j] == P.row_tab[k]) first = false;
    if (!first) continue;
    const int64_t len = P.grid_n[P.row_axis[k]];
    const double ctr = P.row_c[k], sc = P.row_scale[k];
    for (int64_t t = threadIdx.x; t < len; t += blockDim.x)
      tab[P.row_tab[k] + t] = (((double)t + 0.5) - ctr) / sc;
  }
}

// 16-byte vector access is used when every array of a pass is 16-byte
// aligned (torch / cudaMalloc buffers are; an offset user pointer may not be).
__device__ __forceinline__ bool al16(const void* p) {
  return (reinterpret_cast<uintptr_t>(p) & 15u) == 0;
}

// L2 prefetch of a CTA's upcoming slice of a streamed array: one bulk
// prefetch instruction (TMA unit) per array and step, issued PF_AHEAD loop
// steps ahead by one thread, so the vector loads of that step hit L2 instead
// of waiting a full HBM round trip -- the passes are latency-limited with 16
// warps per SM (ncu: long_scoreboard on the loads).  Clamped to the array.
constexpr int PF_AHEAD = 3;
__device__ __forceinline__ void prefetch_l2(const void* base, int64_t off_bytes, int64_t bytes,
                                            int64_t limit_bytes) {
  if (off_bytes >= limit_bytes || bytes <= 0) return;
  if (off_bytes + bytes > limit_bytes) bytes = limit_bytes - off_bytes;
  bytes &= ~int64_t(15);
  if (bytes <= 0) return;
  const char* p = reinterpret_cast<const char*>(base) + off_bytes;
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"((unsigned)bytes) : "memory");
}

__device__ __forceinline__ void prefetch_line_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// ---- Row-pair streaming -------------------------------------------------------
// Passes that read several element-aligned rows (rho, A rows, x, g, ...) for
// every element load them as 16-byte pairs: each thread takes element pairs
// (2q, 2q+1), q = i0, i0 + stride, ..., with every row's pair load issued
// before any arithmetic (nr x 16 bytes in flight per thread).  Measured on
// the B200 (tools/streambench.cu, 8 rows of 8.4M doubles, 1 CTA of 512
// threads per SM): 5.5 TB/s, ahead of a 3-stage cp.async.bulk (TMA) +
// mbarrier pipeline through shared memory at 4.3 TB/s, so the passes use
// this.  Misaligned rows or an odd count fall back to one element at a time.
constexpr int RP_MAXR = 9;
struct StreamRows {
  const double* row[RP_MAXR];
  int nr;
  // structured rows: gen[r] >= 0 -> row r is structured row gen[r] of *P
  const Problem* P = nullptr;
  const double* tab = nullptr;
  int gen[RP_MAXR] = {-1, -1, -1, -1, -1, -1, -1, -1, -1};
};

// Row r of a pass = A row k: dense pointer or, for a structured row, generated.
__device__ __forceinline__ void set_arow(StreamRows& R, int r, const PassCtx& c, const Problem& P,
                                         int k) {
  if (P.structured && P.row_kind[k] != RK_DENSE) {
    R.P = &P;
    R.tab = c.rtab;
    R.gen[r] = k;
    R.row[r] = nullptr;
  } else {
    R.row[r] = P.grad + (int64_t)k * P.ld;
  }
}

// f(i, v): element i with v[r] = row r at i (r < nr; v[r] = 0 beyond).
// Per thread the elements come in a fixed order (deterministic sums).
template <int NR, typename F>
__device__ __forceinline__ void rows_pairs(const PassCtx& c, const StreamRows& R, int64_t n,
                                           F&& f) {
  const int nr = R.nr;
  const int64_t st = c.stride;
  bool vec = (n & 1) == 0;
  for (int r = 0; r < nr; ++r) vec = vec && (R.gen[r] >= 0 || al16(R.row[r]));
  if (vec && R.P && R.P->axis_fast) {   // structured rows, centre-of-mass pattern
    const GridIx G = grid_ix(*R.P);
    const int64_t n2 = n >> 1;
    AxisRows AX;
    AX.init(*R.P);
    int pk[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) pk[r] = (r < nr && R.gen[r] >= 0) ? row_pick_code(*R.P, R.gen[r]) : 0;
    const double* __restrict__ tab = R.tab;
    for (int64_t q = c.i0; q < n2; q += st) {
      double2 v2[NR];
#pragma unroll
      for (int r = 0; r < NR; ++r)
        v2[r] = (r < nr && R.gen[r] < 0) ? reinterpret_cast<const double2*>(R.row[r])[q]
                                         : make_double2(0.0, 0.0);
      int64_t c0[3], c1[3];
      grid_coords(G, 2 * q + G.off, c0);
      grid_coords(G, 2 * q + 1 + G.off, c1);
      double t0[4], t1[4];
      AX.values(tab, c0, t0);
      AX.values(tab, c1, t1);
#pragma unroll
      for (int r = 0; r < NR; ++r)
        if (r < nr && R.gen[r] >= 0) v2[r] = make_double2(row_pick(pk[r], t0), row_pick(pk[r], t1));
      double v[NR];
#pragma unroll
      for (int r = 0; r < NR; ++r) v[r] = v2[r].x;
      f(2 * q, v);
#pragma unroll
      for (int r = 0; r < NR; ++r) v[r] = v2[r].y;
      f(2 * q + 1, v);
    }
    return;
  }
  if (vec && R.P) {   // some rows are generated (structured rows)
    const GridIx G = grid_ix(*R.P);
    const int64_t n2 = n >> 1;
    int code[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) code[r] = (r < nr && R.gen[r] >= 0) ? srow_code(*R.P, R.gen[r]) : 0;
    const double* __restrict__ tab = R.tab;
    for (int64_t q = c.i0; q < n2; q += st) {
      double2 v2[NR];
#pragma unroll
      for (int r = 0; r < NR; ++r)
        v2[r] = (r < nr && R.gen[r] < 0) ? reinterpret_cast<const double2*>(R.row[r])[q]
                                         : make_double2(0.0, 0.0);
      int64_t c0[3], c1[3];
      grid_coords(G, 2 * q + G.off, c0);
      grid_coords(G, 2 * q + 1 + G.off, c1);
#pragma unroll
      for (int r = 0; r < NR; ++r)
        if (r < nr && R.gen[r] >= 0)
          v2[r] = make_double2(srow_fetch(tab, code[r], c0), srow_fetch(tab, code[r], c1));
      double v[NR];
#pragma unroll
      for (int r = 0; r < NR; ++r) v[r] = v2[r].x;
      f(2 * q, v);
#pragma unroll
      for (int r = 0; r < NR; ++r) v[r] = v2[r].y;
      f(2 * q + 1, v);
    }
    return;
  }
  if (vec) {
    const int64_t n2 = n >> 1;
    for (int64_t q = c.i0; q < n2; q += st) {
      double2 v2[NR];
#pragma unroll
      for (int r = 0; r < NR; ++r)
        v2[r] = r < nr ? reinterpret_cast<const double2*>(R.row[r])[q] : make_double2(0.0, 0.0);
      double v[NR];
#pragma unroll
      for (int r = 0; r < NR; ++r) v[r] = v2[r].x;
      f(2 * q, v);
#pragma unroll
      for (int r = 0; r < NR; ++r) v[r] = v2[r].y;
      f(2 * q + 1, v);
    }
    return;
  }
  for (int64_t i = c.i0; i < n; i += st) {
    double v[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) v[r] = r < nr ? R.row[r][i] : 0.0;
    f(i, v);
  }
}

// Fill each warp's active list with all of its grid-stride elements (this
// CTA owns i = blockIdx*BLOCK + tid + k*stride) and clear the fixed sums.
__device__ void compact_init(const PassCtx& c) {
  if (!c.list) return;
  const int64_t n = c.plan->P.n;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* L = c.list + (size_t)warp * c.list_cap;
  const int64_t base = c.i0 - lane;   // warp's first element
  int cnt = 0;
  const int8_t* __restrict__ owner = c.plan->P.owner;
  for (int64_t b = base; b < n; b += c.stride) {   // 32 consecutive elements per step
    const int64_t i = b + lane;
    const bool take = i < n && (owner == nullptr || owner[i] >= 0);
    const unsigned ok = __ballot_sync(0xffffffffu, take);
    if (take) L[cnt + __popc(ok & ((1u << lane) - 1u))] = (uint32_t)i;
    cnt += __popc(ok);
  }
  if (lane == 0) c.list_cnt[warp] = cnt;
  const Problem& P = c.plan->P;
  if (P.part_ranges && c.seg) {
    // the list is ascending and every set a contiguous range: row j's items
    // are one segment [lower_bound(lo_j), lower_bound(hi_j)); lane j finds it
    __syncwarp();
    if (lane < P.m) {
      auto lb = [&](int64_t v) {
        int lo = 0, hi = cnt;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if ((int64_t)L[mid] < v) lo = mid + 1; else hi = mid;
        }
        return lo;
      };
      const int s0 = lb(P.row_lo[lane]), s1 = lb(P.row_hi[lane]);
      c.seg[(warp * MAX_M + lane) * 2] = s0;
      c.seg[(warp * MAX_M + lane) * 2 + 1] = s1 - s0;
    }
  }
  if (threadIdx.x < MAX_M) { c.fixC[threadIdx.x] = 0.0; c.fixS[threadIdx.x] = 0.0; }
  __syncthreads();
}

// ---- host-buffer streaming: wait for an input chunk ------------------------
// One thread per CTA polls the flag the copy stream writes after the chunk's
// copies (stream-ordered, so the data is in memory once the flag is seen);
// the CTA then reads the chunk through L2 (it never touched it before).  A
// copy that never lands stops the wait after ~4 s with *err set, so a broken
// stream cannot hang the GPU.
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __noinline__ void wait_chunk(const unsigned* flag, unsigned epoch, int* timed_out) {
  if (threadIdx.x == 0) {
    // after a first timeout (any CTA) nothing will arrive in time: the launch's
    // results are discarded and the host re-runs the step upload-first
    if (*(volatile int*)timed_out == 0 && (int)(ld_acquire_u32(flag) - epoch) < 0) {
      const unsigned long long t0 = global_ns();
      while ((int)(ld_acquire_u32(flag) - epoch) < 0) {
        __nanosleep(256);
        if (global_ns() - t0 > 4000000000ull || *(volatile int*)timed_out) {
          *(volatile int*)timed_out = 1;
          break;
        }
      }
    }
  }
  __syncthreads();
}

// Element range [lo, hi) of chunk k (the whole slab when not streaming).
struct ChunkRange {
  int64_t lo, hi;
};
__device__ __forceinline__ int num_chunks(const Problem& P) { return P.chunk > 0 ? P.nchunk : 1; }
__device__ __forceinline__ ChunkRange chunk_range(const Problem& P, int k) {
  if (P.chunk <= 0) return {0, P.n};
  const int64_t lo = (int64_t)k * P.chunk;
  return {lo, lo + P.chunk < P.n ? lo + P.chunk : P.n};
}

// ---- PH_STEP_REDUCE: BB / PR+ sums --------------------
struct StepAcc {
  double v[6];
  __device__ __forceinline__ void add(double x0, double q0, double g0, double h0) {
    const double s0 = x0 - q0, y0 = g0 - h0;
    v[0] += s0 * s0; v[1] += s0 * y0; v[2] += y0 * y0; v[3] += g0 * y0; v[4] += h0 * h0;
    v[5] = dmax_(v[5], fabs(g0));
  }
};

__device__ __noinline__ void pass_step_reduce(const PassCtx& c) {
  const Problem& P = c.plan->P;
  const int64_t st = c.stride;
  const double* __restrict__ x = P.x;
  const double* __restrict__ xp = P.x_prev;
  const double* __restrict__ g = P.g;
  const double* __restrict__ gp = P.g_prev;
  StepAcc A = {{0, 0, 0, 0, 0, 0}};
  const int nch = num_chunks(P);
  const bool vec = al16(x) && al16(xp) && al16(g) && al16(gp);
  for (int k = 0; k < nch; ++k) {
    if (P.chunk > 0) wait_chunk(P.in_flags + k, P.epoch, c.timed_out);
    const ChunkRange cr = chunk_range(P, k);
    if (vec) {   // element pairs (chunk starts are even), two pairs in flight
      const double2* __restrict__ X = reinterpret_cast<const double2*>(x);
      const double2* __restrict__ Q = reinterpret_cast<const double2*>(xp);
      const double2* __restrict__ Gv = reinterpret_cast<const double2*>(g);
      const double2* __restrict__ H = reinterpret_cast<const double2*>(gp);
      const int64_t q1 = cr.hi >> 1;
      int64_t q = (cr.lo >> 1) + c.i0;
      for (; q + st < q1; q += 2 * st) {
        const double2 x0 = X[q], p0 = Q[q], g0 = Gv[q], h0 = H[q];
        const double2 x1 = X[q + st], p1 = Q[q + st], g1 = Gv[q + st], h1 = H[q + st];
        A.add(x0.x, p0.x, g0.x, h0.x); A.add(x0.y, p0.y, g0.y, h0.y);
        A.add(x1.x, p1.x, g1.x, h1.x); A.add(x1.y, p1.y, g1.y, h1.y);
      }
      if (q < q1) {
        const double2 x0 = X[q], p0 = Q[q], g0 = Gv[q], h0 = H[q];
        A.add(x0.x, p0.x, g0.x, h0.x); A.add(x0.y, p0.y, g0.y, h0.y);
      }
      if ((cr.hi & 1) && c.i0 == 0) {   // odd tail element
        const int64_t i = cr.hi - 1;
        A.add(x[i], xp[i], g[i], gp[i]);
      }
      continue;
    }
    const int64_t n = cr.hi;
    int64_t i = cr.lo + c.i0;
    for (; i + st < n; i += 2 * st) {   // two independent elements in flight
      const double x0 = x[i], q0 = xp[i], g0 = g[i], h0 = gp[i];
      const double x1 = x[i + st], q1 = xp[i + st], g1 = g[i + st], h1 = gp[i + st];
      A.add(x0, q0, g0, h0);
      A.add(x1, q1, g1, h1);
    }
    if (i < n) A.add(x[i], xp[i], g[i], gp[i]);
  }
  block_reduce_store<6>(A.v, 6, PH_STEP_REDUCE, 0, c.out, c.smem);
}

// ---- PH_PREP: direction, rho_tilde, g_hat dots, r(0), slope(0), bounds,
//      breakpoints (projection.cpp:53-73, :139-145, :150-181) ---------------
struct PrepAcc {
  double v[PREP_SLOTS];
};

__device__ __forceinline__ void prep_elem(PrepAcc& A, double a, double r, double gd, bool dot,
                                          double L, double U) {
  const double lo = L - r, hi = U - r;
  if (dot) {
    const double p = gd * a;
    A.v[PS_DOT] += p;
    A.v[PS_DABS] += fabs(p);
  }
  A.v[PS_S0] += a * (0.0 < lo ? lo : (0.0 > hi ? hi : 0.0));
  if (!(0.0 < lo || 0.0 > hi)) A.v[PS_SLOPE0] += a * a;
  A.v[PS_T] += fabs(a) * dmax_(fabs(lo), fabs(hi));
  if (fabs(a) >= kGradFloor) {
    A.v[PS_ANY] += 1.0;
    // Exact IEEE divisions only where they can move the running min / max:
    // a float estimate (rel. error < 1e-6 in the checked range) filters out
    // the rest.  min(c1,c2) = (a > 0 ? lo : hi) / a, max = (a > 0 ? hi : lo) / a.
    const double nmin = a > 0.0 ? lo : hi, nmax = a > 0.0 ? hi : lo;
    const double fa = fabs(a);
    bool do_min = true, do_max = true;
    if (fa > 1e-30 && fa < 1e30 && fabs(nmin) < 1e30 && fabs(nmax) < 1e30) {
      const float ra = __frcp_rn((float)a);
      const double qmin = (double)((float)nmin * ra), qmax = (double)((float)nmax * ra);
      do_min = qmin - 1e-5 * fabs(qmin) - 1e-300 < A.v[PS_BPLO];
      do_max = qmax + 1e-5 * fabs(qmax) + 1e-300 > A.v[PS_BPHI];
    }
    if (do_min) A.v[PS_BPLO] = dmin_(A.v[PS_BPLO], dmin_(lo / a, hi / a));
    if (do_max) A.v[PS_BPHI] = dmax_(A.v[PS_BPHI], dmax_(lo / a, hi / a));
  }
}

// Does an element's breakpoint fl(num / a) possibly lie below the filter
// value m (MAX: above it)?  It is skipped only when a STRICT comparison with
// the correctly rounded product t = fl(m a) proves it cannot: for a > 0,
// num > t means num >= succ(t) > m a (round-to-nearest puts m a within half
// an ulp of t), so num / a > m and, the division rounding monotonically,
// fl(num / a) >= m -- it cannot be a new minimum.  a < 0 flips the test, MAX
// mirrors it.  Overflow (t = +-inf) and NaN make every comparison false:
// "maybe", the division runs.  (-fmad=false: t is one rounded product.)
template <bool MAX>
__device__ __forceinline__ bool bp_may_beat(double num, double a, double m) {
  const double t = m * a;
  const bool flip = (a > 0.0) == MAX;
  return flip ? !(num < t) : !(num > t);
}

// prep_elem with the breakpoint divisions filtered against (fmin, fmax):
// exact breakpoint values already seen by this warp (refreshed by the caller
// with a warp min / max), so that records of one lane stop the divisions of
// the others.  Elements that cannot beat them cannot be the global extremum
// (the filter values are themselves element breakpoints).
__device__ __forceinline__ void prep_elem_w(PrepAcc& A, double a, double r, double gd, bool dot,
                                            double L, double U, double& fmin, double& fmax) {
  const double lo = L - r, hi = U - r;
  if (dot) {
    const double p = gd * a;
    A.v[PS_DOT] += p;
    A.v[PS_DABS] += fabs(p);
  }
  const bool b0 = 0.0 < lo, a0 = 0.0 > hi;
  A.v[PS_S0] += a * (b0 ? lo : (a0 ? hi : 0.0));
  A.v[PS_SLOPE0] += (b0 || a0) ? 0.0 : a * a;
  A.v[PS_T] += fabs(a) * dmax_(fabs(lo), fabs(hi));
  if (fabs(a) >= kGradFloor) {
    A.v[PS_ANY] += 1.0;
    const bool pos = a > 0.0;
    const double nmin = pos ? lo : hi, nmax = pos ? hi : lo;
    if (bp_may_beat<false>(nmin, a, fmin) || bp_may_beat<true>(nmax, a, fmax)) {
      const double c1 = lo / a, c2 = hi / a;
      A.v[PS_BPLO] = dmin_(A.v[PS_BPLO], dmin_(c1, c2));
      A.v[PS_BPHI] = dmax_(A.v[PS_BPHI], dmax_(c1, c2));
      fmin = dmin_(fmin, A.v[PS_BPLO]);
      fmax = dmax_(fmax, A.v[PS_BPHI]);
    }
  }
}

__device__ __forceinline__ void warp_minmax(double& fmin, double& fmax) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    fmin = dmin_(fmin, __shfl_xor_sync(0xffffffffu, fmin, o));
    fmax = dmax_(fmax, __shfl_xor_sync(0xffffffffu, fmax, o));
  }
}

// PREP row sums of G dense rows j0 .. j0+G-1 in ONE sweep over
// (a_j0 .. a_j0+G-1, rho, d): rho and d are read once per group instead of
// once per row (C4/C5, m = 7: 26 -> 16 streamed n-vectors).  FUSE folds the
// direction pass into the group (g, d_prev, x read; d, rho computed in
// registers and written).  Pair q is handled by thread q mod stride, in
// increasing q, exactly like the one-row loop and rows_pairs, so every row's
// per-thread sums and the stores of rho / d are those of the unfused passes
// (the warp breakpoint filter only skips divisions that cannot move the
// min / max).  Needs 16-byte aligned vectors and even n.
template <int G, bool FUSE>
__device__ __forceinline__ void prep_group(const PassCtx& c, int j0, int64_t n, bool dot, bool use_dp,
                                           double beta, double wa, double L, double U_) {
  const Problem& P = c.plan->P;
  const int64_t st = c.stride, n2 = n >> 1;
  const int lane = threadIdx.x & 31;
  const double2* __restrict__ R2 = reinterpret_cast<const double2*>(P.rho);
  const double2* __restrict__ D2 = reinterpret_cast<const double2*>(P.d_out);
  const double2* __restrict__ G2 = reinterpret_cast<const double2*>(P.g);
  const double2* __restrict__ P2 = reinterpret_cast<const double2*>(use_dp ? P.d_prev : P.g);
  const double2* __restrict__ X2 = reinterpret_cast<const double2*>(P.x);
  double2* __restrict__ RO = reinterpret_cast<double2*>(P.rho);
  double2* __restrict__ DO = reinterpret_cast<double2*>(P.d_out);
  const double2* __restrict__ A2[G];
#pragma unroll
  for (int r = 0; r < G; ++r)
    A2[r] = reinterpret_cast<const double2*>(P.grad + (int64_t)(j0 + r) * P.ld);
  PrepAcc A[G];
  double fmin[G], fmax[G], aref[G];
  // row-structure detection (single rank): a constant row, and row r the
  // exact negation of row r - 1 within the group
  const bool detect = P.n_global == P.n;
#pragma unroll
  for (int r = 0; r < G; ++r) {
#pragma unroll
    for (int s = 0; s < PREP_SLOTS; ++s) A[r].v[s] = 0.0;   // bp_lo = bp_hi = 0 (:58)
    fmin[r] = 0.0;
    fmax[r] = 0.0;
    aref[r] = (detect && n > 0) ? P.grad[(int64_t)(j0 + r) * P.ld] : 0.0;
    if (!detect) A[r].v[PS_NCONST] = 1.0;
    if (!detect || r == 0) A[r].v[PS_NNEG] = 1.0;
    if (detect && c.i0 == 0) A[r].v[PS_AREF] = aref[r];
  }
  // pairs in flight per thread: enough bytes per SM to cover HBM latency
  // (Little's law) without spilling the G rows' accumulators
  constexpr int UP = G == 1 ? 3 : 2;
  int step = 0;
  for (int64_t qb = c.i0 - lane; qb < n2; qb += UP * st, ++step) {   // warp-uniform trip count
    double2 a2[UP][G], r2[UP], d2[UP];
    const double2 z2 = make_double2(0.0, 0.0);
#pragma unroll
    for (int u = 0; u < UP; ++u) {
      const int64_t q = qb + u * st + lane;
      const bool ok = q < n2;
#pragma unroll
      for (int r = 0; r < G; ++r) a2[u][r] = ok ? A2[r][q] : z2;
      if (FUSE) {
        const double2 gv = ok ? G2[q] : z2, pv = (ok && use_dp) ? P2[q] : z2;
        const double2 xv = ok ? X2[q] : z2;
        // d = g + beta d_prev ; rho = x - (omega alpha) d
        d2[u].x = use_dp ? gv.x + beta * pv.x : gv.x;
        d2[u].y = use_dp ? gv.y + beta * pv.y : gv.y;
        r2[u].x = xv.x - wa * d2[u].x;
        r2[u].y = xv.y - wa * d2[u].y;
        if (ok) {
          DO[q] = d2[u];
          RO[q] = r2[u];
        }
      } else {
        r2[u] = ok ? R2[q] : z2;
        d2[u] = (ok && dot) ? D2[q] : z2;
      }
    }
#pragma unroll
    for (int u = 0; u < UP; ++u) {
      if (qb + u * st + lane < n2) {
        const double g0 = dot ? wa * d2[u].x : 0.0, g1 = dot ? wa * d2[u].y : 0.0;
#pragma unroll
        for (int r = 0; r < G; ++r) {
          prep_elem_w(A[r], a2[u][r].x, r2[u].x, g0, dot, L, U_, fmin[r], fmax[r]);
          prep_elem_w(A[r], a2[u][r].y, r2[u].y, g1, dot, L, U_, fmin[r], fmax[r]);
          if (detect) {
            A[r].v[PS_NCONST] += (double)((a2[u][r].x != aref[r]) + (a2[u][r].y != aref[r]));
            if (r > 0)
              A[r].v[PS_NNEG] += (double)((a2[u][r].x != -a2[u][r - 1].x) +
                                          (a2[u][r].y != -a2[u][r - 1].y));
          }
        }
      }
    }
    // the filter may be stale (any breakpoint seen earlier is a valid bound):
    // refreshed every 4th step (20 shuffles per row and refresh)
    if ((step & 3) == 3) {
#pragma unroll
      for (int r = 0; r < G; ++r) warp_minmax(fmin[r], fmax[r]);
    }
  }
#pragma unroll
  for (int r = 0; r < G; ++r)
    block_reduce_store<PREP_SLOTS>(A[r].v, PREP_SLOTS, PH_PREP, (j0 + r) * PREP_SLOTS, c.out, c.smem);
}

// Pattern PREP (cmd.pat_hint: the previous step on these buffers found rows
// 2k the exact negations of rows 2k - 1): one sweep computes NP base rows in
// full and only VERIFIES their negations element by element; a verified
// negated row's sums follow from its base row's by exact sign flips (every
// term negated, min and max breakpoints swapped), so the slots written are
// bit for bit those of the general PREP.  FUSE0 folds the direction pass and
// row 0 (computed in full) into the sweep.  m = 7: rows 0 | (1, 2) and then
// (3, 4), (5, 6) -- 14 streamed n-vectors and 4 rows of arithmetic instead of
// 18 and 7.  A failed verification (PS_NNEG != 0) makes the controller run
// the general PREP again.
template <bool FUSE0, int NP>
__device__ __noinline__ void prep_pairs(const PassCtx& c, int jb0, int64_t n, bool dot,
                                           bool use_dp, double beta, double wa, double L,
                                           double U_) {
  constexpr int NB = NP + (FUSE0 ? 1 : 0);   // rows computed in full
  const Problem& P = c.plan->P;
  const int64_t st = c.stride, n2 = n >> 1;
  const int lane = threadIdx.x & 31;
  const double2* __restrict__ R2 = reinterpret_cast<const double2*>(P.rho);
  const double2* __restrict__ D2 = reinterpret_cast<const double2*>(P.d_out);
  const double2* __restrict__ G2 = reinterpret_cast<const double2*>(P.g);
  const double2* __restrict__ P2 = reinterpret_cast<const double2*>(use_dp ? P.d_prev : P.g);
  const double2* __restrict__ X2 = reinterpret_cast<const double2*>(P.x);
  double2* __restrict__ RO = reinterpret_cast<double2*>(P.rho);
  double2* __restrict__ DO = reinterpret_cast<double2*>(P.d_out);
  int rowf[NB];   // the full rows' indices; negated row of full row r (r >= NB - NP): rowf[r] + 1
#pragma unroll
  for (int r = 0; r < NB; ++r) rowf[r] = (FUSE0 && r == 0) ? 0 : jb0 + 2 * (r - (FUSE0 ? 1 : 0));
  const double2* __restrict__ F2[NB];
  const double2* __restrict__ N2[NP];
#pragma unroll
  for (int r = 0; r < NB; ++r)
    F2[r] = reinterpret_cast<const double2*>(P.grad + (int64_t)rowf[r] * P.ld);
#pragma unroll
  for (int p = 0; p < NP; ++p)
    N2[p] = reinterpret_cast<const double2*>(P.grad + (int64_t)(jb0 + 2 * p + 1) * P.ld);
  PrepAcc A[NB];
  double fmin[NB], fmax[NB], aref[NB], nneg[NP];
#pragma unroll
  for (int r = 0; r < NB; ++r) {
#pragma unroll
    for (int s = 0; s < PREP_SLOTS; ++s) A[r].v[s] = 0.0;
    fmin[r] = 0.0;
    fmax[r] = 0.0;
    aref[r] = n > 0 ? P.grad[(int64_t)rowf[r] * P.ld] : 0.0;
    A[r].v[PS_NNEG] = 1.0;   // a full row is not examined as a negation
    if (c.i0 == 0) A[r].v[PS_AREF] = aref[r];
  }
#pragma unroll
  for (int p = 0; p < NP; ++p) nneg[p] = 0.0;
  constexpr int UP = 1;   // (two pairs in flight spill: 2 x 6 loads + 25 accumulators)
  int step = 0;
  for (int64_t qb = c.i0 - lane; qb < n2; qb += UP * st, ++step) {   // warp-uniform trip count
    {   // the next step's lines into L2 (one lane per 128-byte line, no registers held):
        // one pair in flight per thread does not cover the HBM latency by itself
      const int64_t qn = qb + 2 * UP * st + lane;   // two steps ahead
      if ((lane & 7) == 0 && qn < n2) {
#pragma unroll
        for (int r = 0; r < NB; ++r) prefetch_line_l2(F2[r] + qn);
#pragma unroll
        for (int p = 0; p < NP; ++p) prefetch_line_l2(N2[p] + qn);
        if (FUSE0) {
          prefetch_line_l2(G2 + qn);
          if (use_dp) prefetch_line_l2(P2 + qn);
          prefetch_line_l2(X2 + qn);
        } else {
          prefetch_line_l2(R2 + qn);
          if (dot) prefetch_line_l2(D2 + qn);
        }
      }
    }
    double2 f2[UP][NB], m2[UP][NP], r2[UP], d2[UP];
    const double2 z2 = make_double2(0.0, 0.0);
#pragma unroll
    for (int u = 0; u < UP; ++u) {
      const int64_t q = qb + u * st + lane;
      const bool ok = q < n2;
#pragma unroll
      for (int r = 0; r < NB; ++r) f2[u][r] = ok ? F2[r][q] : z2;
#pragma unroll
      for (int p = 0; p < NP; ++p) m2[u][p] = ok ? N2[p][q] : z2;
      if (FUSE0) {
        const double2 gv = ok ? G2[q] : z2, pv = (ok && use_dp) ? P2[q] : z2;
        const double2 xv = ok ? X2[q] : z2;
        // d = g + beta d_prev ; rho = x - (omega alpha) d
        d2[u].x = use_dp ? gv.x + beta * pv.x : gv.x;
        d2[u].y = use_dp ? gv.y + beta * pv.y : gv.y;
        r2[u].x = xv.x - wa * d2[u].x;
        r2[u].y = xv.y - wa * d2[u].y;
        if (ok) {
          DO[q] = d2[u];
          RO[q] = r2[u];
        }
      } else {
        r2[u] = ok ? R2[q] : z2;
        d2[u] = (ok && dot) ? D2[q] : z2;
      }
    }
#pragma unroll
    for (int u = 0; u < UP; ++u) {
      if (qb + u * st + lane < n2) {
        const double g0 = dot ? wa * d2[u].x : 0.0, g1 = dot ? wa * d2[u].y : 0.0;
#pragma unroll
        for (int r = 0; r < NB; ++r) {
          prep_elem_w(A[r], f2[u][r].x, r2[u].x, g0, dot, L, U_, fmin[r], fmax[r]);
          prep_elem_w(A[r], f2[u][r].y, r2[u].y, g1, dot, L, U_, fmin[r], fmax[r]);
          A[r].v[PS_NCONST] += (double)((f2[u][r].x != aref[r]) + (f2[u][r].y != aref[r]));
        }
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          const double2 b = f2[u][NB - NP + p];
          nneg[p] += (double)((m2[u][p].x != -b.x) + (m2[u][p].y != -b.y));
        }
      }
    }
    if ((step & 7) == 7) {   // (stale filters are valid: see prep_group)
#pragma unroll
      for (int r = 0; r < NB; ++r) warp_minmax(fmin[r], fmax[r]);
    }
  }
#pragma unroll
  for (int r = 0; r < NB; ++r)
    block_reduce_store<PREP_SLOTS>(A[r].v, PREP_SLOTS, PH_PREP, rowf[r] * PREP_SLOTS, c.out, c.smem);
#pragma unroll
  for (int p = 0; p < NP; ++p) {   // the negated rows' slots from their base rows'
    const PrepAcc& B = A[NB - NP + p];
    PrepAcc Dn;
    Dn.v[PS_DOT] = -B.v[PS_DOT];
    Dn.v[PS_DABS] = B.v[PS_DABS];
    Dn.v[PS_S0] = -B.v[PS_S0];
    Dn.v[PS_SLOPE0] = B.v[PS_SLOPE0];
    Dn.v[PS_T] = B.v[PS_T];
    Dn.v[PS_NZOUT] = B.v[PS_NZOUT];
    Dn.v[PS_BPLO] = -B.v[PS_BPHI];
    Dn.v[PS_BPHI] = -B.v[PS_BPLO];
    Dn.v[PS_ANY] = B.v[PS_ANY];
    Dn.v[PS_NCONST] = B.v[PS_NCONST];
    Dn.v[PS_AREF] = -B.v[PS_AREF];
    Dn.v[PS_NNEG] = nneg[p];
    block_reduce_store<PREP_SLOTS>(Dn.v, PREP_SLOTS, PH_PREP, (jb0 + 2 * p + 1) * PREP_SLOTS, c.out,
                                   c.smem);
  }
}

// Dense rows, no partition, device-resident aligned inputs: the direction
// pass fused with the first row group, then groups of PREP_GROUP rows.
constexpr int PREP_GROUP = 2;
__device__ __forceinline__ bool P_detect_single_rank(const PassCtx& c) {
  return c.plan->P.n_global == c.plan->P.n;
}
__device__ __noinline__ void prep_dense_grouped(const PassCtx& c, int m, int64_t n, bool dir,
                                                bool dot, bool use_dp, double beta, double wa,
                                                double L, double U_) {
  // row 0 with the direction pass, then pairs (1,2), (3,4), ...: the +- rows
  // of two-sided constraints (a row and its negation, adjacent) share a group,
  // where the negation is detected (same 2m + 4 streamed vectors as before)
  if (c.cmd->pat_hint && dir && m == 7 && P_detect_single_rank(c)) {
    prep_pairs<true, 1>(c, 1, n, dot, use_dp, beta, wa, L, U_);
    prep_pairs<false, 2>(c, 3, n, dot, use_dp, beta, wa, L, U_);
    return;
  }
  int j = 0;
  if (dir) {
    prep_group<1, true>(c, 0, n, dot, use_dp, beta, wa, L, U_);
    j = 1;
  }
  for (; j + PREP_GROUP <= m; j += PREP_GROUP)
    prep_group<PREP_GROUP, false>(c, j, n, dot, use_dp, beta, wa, L, U_);
  for (; j < m; ++j) prep_group<1, false>(c, j, n, dot, use_dp, beta, wa, L, U_);
}

__device__ __noinline__ void pass_prep(const PassCtx& c) {
  const Plan& pl = *c.plan;
  const Problem& P = pl.P;
  const Cmd& cmd = *c.cmd;
  const int64_t n = P.n, st = c.stride, ld = P.ld;
  const int m = P.m;
  double* __restrict__ rho = P.rho;
  double* __restrict__ dout = P.d_out;
  const double* __restrict__ x = P.x;
  const double* __restrict__ g = P.g;
  const double* __restrict__ dp = P.d_prev;
  const double* __restrict__ gd_in = P.gd_step;
  const int8_t* __restrict__ owner = P.owner;
  const bool dir = cmd.compute_dir, dot = cmd.compute_dot, use_dp = cmd.use_dprev;
  const double beta = cmd.beta, wa = cmd.wa;
  constexpr int U = 4;   // elements in flight per thread
  const double L = P.lower, U_ = P.upper;
  if (dir && m == 1 && !owner) {
    // One row, no partition (C1/C2): direction and row sums in one sweep, so
    // rho and d are not read back.
    PrepAcc A;
#pragma unroll
    for (int s = 0; s < PREP_SLOTS; ++s) A.v[s] = 0.0;   // bp_lo = bp_hi = 0 (:58)
    A.v[PS_NCONST] = A.v[PS_NNEG] = 1.0;   // (structure not examined here)
    const double* __restrict__ ar = P.grad;
    const int nch = num_chunks(P);
    const bool vec = al16(g) && al16(x) && al16(ar) && al16(dout) && al16(rho) &&
                     (!use_dp || al16(dp));
    // d = g + beta d_prev ; gd = (omega alpha) d ; rho = x - gd
    double fmin = 0.0, fmax = 0.0;   // warp-shared breakpoint filter (prep_elem_w)
    auto elem = [&](double gv, double dv, double xv, double av, double& d, double& r) {
      d = use_dp ? gv + beta * dv : gv;
      const double gd = wa * d;
      r = xv - gd;
      prep_elem_w(A, av, r, gd, dot, L, U_, fmin, fmax);
    };
    for (int k = 0; k < nch; ++k) {
      if (P.chunk > 0) wait_chunk(P.in_flags + P.nchunk + k, P.epoch, c.timed_out);
      const ChunkRange cr = chunk_range(P, k);
      if (vec) {   // element pairs, two pairs in flight per thread
        const double2* __restrict__ G2 = reinterpret_cast<const double2*>(g);
        const double2* __restrict__ D2 = reinterpret_cast<const double2*>(dp);
        const double2* __restrict__ X2 = reinterpret_cast<const double2*>(x);
        const double2* __restrict__ A2 = reinterpret_cast<const double2*>(ar);
        double2* __restrict__ DO = reinterpret_cast<double2*>(dout);
        double2* __restrict__ RO = reinterpret_cast<double2*>(rho);
        const int64_t q1 = cr.hi >> 1;
        const int lane = threadIdx.x & 31;
        // warp-uniform trip count (the filter refresh is a warp shuffle)
        for (int64_t qb = (cr.lo >> 1) + c.i0 - lane; qb < q1; qb += 2 * st) {
          const int64_t q = qb + lane;
          const bool ok0 = q < q1, ok1 = q + st < q1;
          const double2 z2 = make_double2(0.0, 0.0);
          const double2 g0 = ok0 ? G2[q] : z2, x0 = ok0 ? X2[q] : z2, a0 = ok0 ? A2[q] : z2;
          const double2 d0 = (ok0 && use_dp) ? D2[q] : z2;
          const double2 g1 = ok1 ? G2[q + st] : z2, x1 = ok1 ? X2[q + st] : z2;
          const double2 a1 = ok1 ? A2[q + st] : z2;
          const double2 d1 = (ok1 && use_dp) ? D2[q + st] : z2;
          double2 dd, rr;
          if (ok0) {
            elem(g0.x, d0.x, x0.x, a0.x, dd.x, rr.x);
            elem(g0.y, d0.y, x0.y, a0.y, dd.y, rr.y);
            DO[q] = dd;
            RO[q] = rr;
          }
          if (ok1) {
            elem(g1.x, d1.x, x1.x, a1.x, dd.x, rr.x);
            elem(g1.y, d1.y, x1.y, a1.y, dd.y, rr.y);
            DO[q + st] = dd;
            RO[q + st] = rr;
          }
          warp_minmax(fmin, fmax);
        }
        if ((cr.hi & 1) && c.i0 == 0) {   // odd tail element
          const int64_t i = cr.hi - 1;
          double dd, rr;
          elem(g[i], use_dp ? dp[i] : 0.0, x[i], ar[i], dd, rr);
          dout[i] = dd;
          rho[i] = rr;
        }
        continue;
      }
      for (int64_t i = cr.lo + c.i0; i < cr.hi; i += st) {
        double dd, rr;
        elem(g[i], use_dp ? dp[i] : 0.0, x[i], ar[i], dd, rr);
        dout[i] = dd;
        rho[i] = rr;
      }
    }
    block_reduce_store<PREP_SLOTS>(A.v, PREP_SLOTS, PH_PREP, 0, c.out, c.smem);
    compact_init(c);
    return;
  }
  // device-resident inputs, no partition or a partition of contiguous index
  // ranges: the direction pass and one pass per row over (a_j, rho, d) as
  // 16-byte pairs (a range row only over its own range; outside it only a_j
  // is read, for the validation count), same per-element arithmetic
  if ((!owner || P.part_ranges) && P.chunk <= 0) {
    if (dir && m >= 1 && !owner && !P.structured && (n & 1) == 0 && (ld & 1) == 0 && al16(P.grad) &&
        al16(g) && al16(x) && al16(dout) && al16(rho) && (!use_dp || al16(dp))) {
      prep_dense_grouped(c, m, n, dir, dot, use_dp, beta, wa, L, U_);
      compact_init(c);
      return;
    }
    if (dir) {
      StreamRows D;
      D.nr = 3;
      D.row[0] = g; D.row[1] = use_dp ? dp : g; D.row[2] = x;
      const bool vo = al16(dout) && al16(rho);
      if (vo && (n & 1) == 0) {
        rows_pairs<3>(c, D, n, [&](int64_t i, const double (&v)[3]) {
          const double d = use_dp ? v[0] + beta * v[1] : v[0];
          dout[i] = d;
          rho[i] = v[2] - wa * d;
        });
      } else {
        for (int64_t i = c.i0; i < n; i += st) {
          const double d = use_dp ? g[i] + beta * dp[i] : g[i];
          dout[i] = d;
          rho[i] = x[i] - wa * d;
        }
      }
    }
    for (int j = 0; j < m; ++j) {
      PrepAcc A;
#pragma unroll
      for (int s2 = 0; s2 < PREP_SLOTS; ++s2) A.v[s2] = 0.0;   // bp_lo = bp_hi = 0 (:58)
      A.v[PS_NCONST] = A.v[PS_NNEG] = 1.0;   // (structure not examined here)
      StreamRows Rj;
      Rj.nr = 3;
      Rj.row[0] = P.grad + (int64_t)j * ld; Rj.row[1] = rho;
      Rj.row[2] = dot ? (dir ? dout : gd_in) : rho;
      // rho and d of element i were written by this same thread above (same
      // element-to-thread map), so no barrier is needed between the loops
      const bool gen = P.structured && P.row_kind[j] != RK_DENSE;
      const int gcode = gen ? srow_code(P, j) : 0;
      const double* __restrict__ ar = gen ? rho : Rj.row[0];   // (not read when generated)
      const double* __restrict__ gdr = Rj.row[2];
      const int64_t rlo = owner ? P.row_lo[j] : 0, rhi = owner ? P.row_hi[j] : n;
      const GridIx G = grid_ix(P);
      if (owner) {   // validation (projection.cpp:173-180): a_j must vanish outside its set
        int nz = 0;
        auto scan = [&](int64_t b, int64_t e) {   // count a_ji != 0 for i in [b, e)
          if (((b | e) & 1) == 0 && al16(ar)) {
            const double2* __restrict__ A2 = reinterpret_cast<const double2*>(ar);
            const int64_t e2 = e >> 1;
            for (int64_t q = (b >> 1) + c.i0; q < e2; q += 4 * st) {
              double2 v[4];
#pragma unroll
              for (int u = 0; u < 4; ++u)
                v[u] = q + u * st < e2 ? A2[q + u * st] : make_double2(0.0, 0.0);
#pragma unroll
              for (int u = 0; u < 4; ++u) nz += (v[u].x != 0.0) + (v[u].y != 0.0);
            }
          } else {
            for (int64_t i = b + c.i0; i < e; i += st) nz += ar[i] != 0.0;
          }
        };
        scan(0, rlo);
        scan(rhi, n);
        A.v[PS_NZOUT] = (double)nz;
      }
      if (((rlo | rhi) & 1) == 0 && al16(ar) && al16(rho) && al16(gdr)) {
        // 16-byte pairs, warp-uniform trip count: the breakpoint filter is
        // refreshed with the warp's min / max every step
        const int lane = threadIdx.x & 31;
        const int64_t q0 = rlo >> 1, n2 = rhi >> 1;
        const double2* __restrict__ A2 = reinterpret_cast<const double2*>(ar);
        const double2* __restrict__ R2 = reinterpret_cast<const double2*>(rho);
        const double2* __restrict__ D2 = reinterpret_cast<const double2*>(gdr);
        double fmin = 0.0, fmax = 0.0;
        constexpr int UP = 4;   // pairs in flight per thread
        for (int64_t qb = q0 + c.i0 - lane; qb < n2; qb += UP * st) {
          double2 a2[UP], r2[UP], d2[UP];
#pragma unroll
          for (int u = 0; u < UP; ++u) {
            const int64_t q = qb + u * st + lane;
            const bool ok = q < n2;
            a2[u] = (ok && !gen) ? A2[q] : make_double2(0.0, 0.0);
            r2[u] = ok ? R2[q] : make_double2(0.0, 0.0);
            d2[u] = (ok && dot) ? D2[q] : make_double2(0.0, 0.0);
            if (ok && gen) {
              int64_t c0[3], c1[3];
              grid_coords(G, 2 * q + G.off, c0);
              grid_coords(G, 2 * q + 1 + G.off, c1);
              a2[u] = make_double2(srow_fetch(c.rtab, gcode, c0), srow_fetch(c.rtab, gcode, c1));
            }
          }
#pragma unroll
          for (int u = 0; u < UP; ++u) {
            if (qb + u * st + lane < n2) {
              const double g0 = dot ? (dir ? wa * d2[u].x : d2[u].x) : 0.0;
              const double g1 = dot ? (dir ? wa * d2[u].y : d2[u].y) : 0.0;
              prep_elem_w(A, a2[u].x, r2[u].x, g0, dot, L, U_, fmin, fmax);
              prep_elem_w(A, a2[u].y, r2[u].y, g1, dot, L, U_, fmin, fmax);
            }
          }
          warp_minmax(fmin, fmax);
        }
      } else {
        for (int64_t i = rlo + c.i0; i < rhi; i += st) {
          const double gdv = dot ? (dir ? wa * gdr[i] : gdr[i]) : 0.0;
          prep_elem(A, ar[i], rho[i], gdv, dot, L, U_);
        }
      }
      block_reduce_store<PREP_SLOTS>(A.v, PREP_SLOTS, PH_PREP, j * PREP_SLOTS, c.out, c.smem);
    }
    compact_init(c);
    return;
  }
  if (dir) {  // d = g + beta d_prev ; gd = (omega alpha) d ; rho = x - gd
   const int nch = num_chunks(P);
   for (int k = 0; k < nch; ++k) {
    if (P.chunk > 0) wait_chunk(P.in_flags + P.nchunk + k, P.epoch, c.timed_out);
    const ChunkRange cr = chunk_range(P, k);
    for (int64_t i0 = cr.lo + c.i0; i0 < cr.hi; i0 += U * st) {
      double gv[U], dv[U], xv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t i = i0 + u * st;
        const bool ok = i < cr.hi;
        gv[u] = ok ? g[i] : 0.0;
        dv[u] = (ok && use_dp) ? dp[i] : 0.0;
        xv[u] = ok ? x[i] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t i = i0 + u * st;
        if (i < cr.hi) {
          const double d = use_dp ? gv[u] + beta * dv[u] : gv[u];
          dout[i] = d;
          rho[i] = xv[u] - wa * d;
        }
      }
    }
   }
  } else if (P.chunk > 0) {   // streamed PROJECT-style input: wait for everything
    for (int k = 0; k < P.nchunk; ++k) wait_chunk(P.in_flags + P.nchunk + k, P.epoch, c.timed_out);
  }
  for (int j = 0; j < m; ++j) {
    PrepAcc A;
#pragma unroll
    for (int s = 0; s < PREP_SLOTS; ++s) A.v[s] = 0.0;   // bp_lo = bp_hi = 0 (:58)
    A.v[PS_NCONST] = A.v[PS_NNEG] = 1.0;   // (structure not examined here)
    const double* __restrict__ ar = P.grad + (int64_t)j * ld;
    for (int64_t i0 = c.i0; i0 < n; i0 += U * st) {
      double av[U], rv[U], gdv[U];
      int ov[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t i = i0 + u * st;
        const bool ok = i < n;
        av[u] = ok ? ar[i] : 0.0;
        rv[u] = ok ? rho[i] : 0.0;
        gdv[u] = (ok && dot) ? (dir ? wa * dout[i] : gd_in[i]) : 0.0;
        ov[u] = (ok && owner) ? (int)owner[i] : j;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (i0 + u * st >= n) continue;
        if (ov[u] != j) {
          A.v[PS_NZOUT] += (av[u] != 0.0) ? 1.0 : 0.0;
          continue;
        }
        prep_elem(A, av[u], rv[u], gdv[u], dot, L, U_);
      }
    }
    block_reduce_store<PREP_SLOTS>(A.v, PREP_SLOTS, PH_PREP, j * PREP_SLOTS, c.out, c.smem);
  }
  compact_init(c);
}

// ---- PH_SWEEP: r_j(y_k) and slope at up to MAX_K candidates per row -------
// 1/a to full precision without the IEEE division subroutine: hardware
// reciprocal estimate + two Newton steps (< 1 ulp off before the final
// product).  |a| outside the normal range falls back to the IEEE division.
__device__ __forceinline__ double rcp_full(double a) {
  const double fa = fabs(a);
  if (!(fa > 1e-300 && fa < 1e300)) return 1.0 / a;
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a));
  r = __fma_rn(r, __fma_rn(-a, r, 1.0), r);
  r = __fma_rn(r, __fma_rn(-a, r, 1.0), r);
  return r;
}

// One element's contribution to r(y_k) at the SORTED candidates y[0..cnt):
// its clip region is L for y < bl, free for bl <= y <= bh, U for y > bh
// (bl, bh = its two breakpoints in y), so two binary searches give the region
// of every candidate, and the sweep accumulates per candidate only the
// clipped constants C_k and the free slope S_k (r_k = C_k + y_k S_k).  An
// element whose breakpoint lies within a few ulps of a candidate may be
// classified differently from the reference's fl(y a) test; its term then
// differs by <= 4u|a| max(|lo|,|hi|) and the free terms by 2u|t|: both are
// inside the certification bound E (+16u T, controller.h).
template <int KC>
__device__ __forceinline__ void sweep_elem(double a, double r, const double* y, int cnt,
                                           double L, double U, double* C, double* S) {
  if (a == 0.0) return;   // every term is an exact zero
  const double lo = L - r, hi = U - r;
  const double ra = rcp_full(a);
  const double b1 = lo * ra, b2 = hi * ra;
  const bool pos = a > 0.0;
  const double bl = pos ? b1 : b2, bh = pos ? b2 : b1;
  const double cl = a * (pos ? lo : hi), ch = a * (pos ? hi : lo), aa = a * a;
  // the candidates are ascending: k < p1 = #{y_k < bl} below the free window,
  // k >= p2 = #{y_k <= bh} above it -- one compare pair per candidate
  // (independent, no search chain through shared memory)
#pragma unroll
  for (int k = 0; k < KC; ++k) {
    const double yk = y[k];
    const bool below = yk < bl, above = !(yk <= bh);
    C[k] += below ? cl : (above ? ch : 0.0);
    S[k] += (below || above) ? 0.0 : aa;
  }
  (void)cnt;
}

// Most elements have no candidate inside their free window [bl, bh] and none
// between their two breakpoints' positions: every candidate then sees the
// same clipped constant, or the element is free at every candidate -- one of
// three running sums per lane.  The others are queued per warp (a, rho) and
// run through the per-candidate evaluation 32 at a time, TRANSPOSED: lane l
// owns candidate l & 15 and walks half (l >> 4) of the batch, reading the
// queued elements from shared memory (broadcast) -- two accumulators per lane
// for any number of candidates.  (One accumulator pair per candidate and lane,
// the earlier layout, is 2 x 16 doubles per lane: pass_sweep_row<16> spilled
// them to local memory inside the candidate loop; C5's first sweep spent 5 of
// its 8.5 ms there.)  The sums per candidate get the same terms, in a
// different, still fixed, order.
constexpr int SQ_CAP = 64;   // NWARP * 2 * SQ_CAP doubles fit the reduction scratch
static_assert(MAX_K <= 16, "the transposed candidate evaluation maps candidates to 16 lanes");
template <int KC>
struct SweepAcc {
  double Cq, Sq;     // queued elements' sums at this lane's candidate (lane & 15)
  double Sall;       // slopes of elements free at every candidate (p1 = 0, p2 = cnt)
  double Clo, Chi;   // constants of elements clipped alike at every candidate
  double y0, yl;     // the row's first and last candidate
  double yk;         // this lane's candidate
  double* qa;        // this warp's queue (shared memory, SQ_CAP entries)
  double* qr;
  int qn;
  const double* y;
  int cnt;
  double L, U;
  __device__ __forceinline__ void init(double* qa_, double* qr_, const double* y_, int cnt_,
                                       double L_, double U_) {
    Cq = 0.0; Sq = 0.0;
    Sall = 0.0; Clo = 0.0; Chi = 0.0;
    qa = qa_; qr = qr_; qn = 0; y = y_; cnt = cnt_; L = L_; U = U_;
    y0 = y_[0]; yl = y_[cnt_ - 1];
    const int k = threadIdx.x & 15;
    yk = y_[k < cnt_ ? k : cnt_ - 1];
  }
  // entries [from, from + nq) of the queue at every candidate (all 32 lanes)
  __device__ __forceinline__ void batch(int from, int nq) {
    const int half = (threadIdx.x & 31) >> 4;
#pragma unroll 4
    for (int e = 0; e < 16; ++e) {
      const int idx = half * 16 + e;
      if (idx < nq) {   // (uniform within each half-warp)
        const double a = qa[from + idx], r = qr[from + idx];
        const double lo = L - r, hi = U - r;
        const double ra = rcp_full(a);
        const double b1 = lo * ra, b2 = hi * ra;
        const bool pos = a > 0.0;
        const double bl = pos ? b1 : b2, bh = pos ? b2 : b1;
        const double cl = a * (pos ? lo : hi), ch = a * (pos ? hi : lo), aa = a * a;
        const bool below = yk < bl, above = !(yk <= bh);
        Cq += below ? cl : (above ? ch : 0.0);
        Sq += (below || above) ? 0.0 : aa;
      }
    }
  }
  // all 32 lanes call push together (valid = this lane holds an element)
  __device__ __forceinline__ void push(bool valid, double a, double r) {
    const int lane = threadIdx.x & 31;
    bool need = false;
    if (valid && a != 0.0) {
      const double lo = L - r, hi = U - r;
      const double ra = rcp_full(a);
      const double b1 = lo * ra, b2 = hi * ra;
      const bool pos = a > 0.0;
      const double bl = pos ? b1 : b2, bh = pos ? b2 : b1;
      // window endpoints decide most elements without a search: both
      // breakpoints outside (y_0, y_last] means p1, p2 in {0, cnt}
      const bool outl = bl <= y0 || bl > yl, outh = bh < y0 || bh >= yl;
      if (outl && outh) {
        const bool p1z = !(bl > yl), p2z = !(bh >= yl);   // p1 == 0, p2 == 0
        if (p1z == p2z) {
          // clipped alike at every candidate: one sum, added to every C_k at
          // the end, instead of a select + add per candidate
          if (p1z) Chi += a * (pos ? hi : lo);
          else Clo += a * (pos ? lo : hi);
        } else if (p1z) {
          // free at every candidate (a small |a| makes the window wide): its
          // term is y_k a^2 for all k -- one slope sum
          Sall += a * a;
        } else {
          need = true;
        }
      } else {
        need = true;   // a breakpoint inside the window: the per-candidate evaluation
      }
    }
    const unsigned nm = __ballot_sync(0xffffffffu, need);
    if (nm) {
      if (need) {
        const int slot = qn + __popc(nm & ((1u << lane) - 1u));
        qa[slot] = a;
        qr[slot] = r;
      }
      qn += __popc(nm);
      __syncwarp();
      if (qn >= 32) {
        batch(qn - 32, 32);
        qn -= 32;
        __syncwarp();
      }
    }
  }
  // Drain the queue and leave this warp's (R_k, S_k) pairs, k < 16, in
  // out32[2k], out32[2k + 1] (shared memory; may alias the queue).
  __device__ __forceinline__ void finish(double* out32) {
    const int lane = threadIdx.x & 31;
    __syncwarp();
    if (qn > 0) batch(0, qn);
    qn = 0;
    __syncwarp();
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {   // fixed xor tree: every lane gets the warp's sums
      Sall += __shfl_xor_sync(0xffffffffu, Sall, o);
      Clo += __shfl_xor_sync(0xffffffffu, Clo, o);
      Chi += __shfl_xor_sync(0xffffffffu, Chi, o);
    }
    const double C2 = Cq + __shfl_down_sync(0xffffffffu, Cq, 16);
    const double S2 = Sq + __shfl_down_sync(0xffffffffu, Sq, 16);
    if (lane < 16) {
      const double Sk = S2 + Sall, Ck = (C2 + Chi) + Clo;
      out32[2 * lane] = Ck + yk * Sk;   // r_k = C_k + y_k S_k
      out32[2 * lane + 1] = Sk;
    }
    __syncwarp();
  }
};

// The per-lane layout (one accumulator pair per candidate and lane): fewer
// instructions per queued element than the transposed batch, but 2 KC + 5
// live doubles -- used for the WIDE sweeps (a walk's first full sweep and the
// sketches, where a large share of the elements has a breakpoint inside the
// window), one pair of loads in flight so the accumulators stay in registers.
template <int KC>
struct SweepAccW {
  double C[KC], S[KC];
  double Sall;   // slopes of elements free at every candidate (p1 = 0, p2 = cnt)
  double Clo, Chi;   // constants of elements clipped alike at every candidate
  double y0, yl;     // the row's first and last candidate
  double* qa;    // this warp's queue (shared memory, SQ_CAP entries)
  double* qr;
  int qn;
  const double* y;
  int cnt;
  double L, U;
  __device__ __forceinline__ void init(double* qa_, double* qr_, const double* y_, int cnt_,
                                       double L_, double U_) {
#pragma unroll
    for (int k = 0; k < KC; ++k) { C[k] = 0.0; S[k] = 0.0; }
    Sall = 0.0; Clo = 0.0; Chi = 0.0;
    qa = qa_; qr = qr_; qn = 0; y = y_; cnt = cnt_; L = L_; U = U_;
    y0 = y_[0]; yl = y_[cnt_ - 1];
  }
  // all 32 lanes call push together (valid = this lane holds an element)
  __device__ __forceinline__ void push(bool valid, double a, double r) {
    const int lane = threadIdx.x & 31;
    bool need = false;
    if (valid && a != 0.0) {
      const double lo = L - r, hi = U - r;
      const double ra = rcp_full(a);
      const double b1 = lo * ra, b2 = hi * ra;
      const bool pos = a > 0.0;
      const double bl = pos ? b1 : b2, bh = pos ? b2 : b1;
      // window endpoints decide most elements without a search: both
      // breakpoints outside (y_0, y_last] means p1, p2 in {0, cnt}
      const bool outl = bl <= y0 || bl > yl, outh = bh < y0 || bh >= yl;
      int p1 = 0, p2 = 0;
      if (outl && outh) {
        p1 = bl > yl ? cnt : 0;
        p2 = bh >= yl ? cnt : 0;
      } else {
        p1 = -1;   // a breakpoint inside the window: the full per-candidate loop
      }
      if (p1 < 0) {
        need = true;
      } else if (p1 == p2) {
        const double cl = a * (pos ? lo : hi), ch = a * (pos ? hi : lo);
        // the walk window is narrow after the first sweep: nearly every
        // element is clipped alike at every candidate -- one sum, added to
        // every C_k at the end, instead of a select + add per candidate
        if (p1 == 0) {
          Chi += ch;
        } else if (p1 >= cnt) {
          Clo += cl;
        } else {
#pragma unroll
          for (int k = 0; k < KC; ++k) C[k] += (k < p1) ? cl : ch;
        }
      } else if (p1 == 0 && p2 == cnt) {
        // free at every candidate (a small |a| makes the window wide): its
        // term is y_k a^2 for all k -- one slope sum, added to every S_k at
        // the end (no clipped constant)
        Sall += a * a;
      } else {
        need = true;
      }
    }
    const unsigned nm = __ballot_sync(0xffffffffu, need);
    if (need) {
      const int slot = qn + __popc(nm & ((1u << lane) - 1u));
      qa[slot] = a;
      qr[slot] = r;
    }
    qn += __popc(nm);
    __syncwarp();
    if (qn >= 32) {
      const int s2 = qn - 32 + lane;
      sweep_elem<KC>(qa[s2], qr[s2], y, cnt, L, U, C, S);
      qn -= 32;
      __syncwarp();
    }
  }
  __device__ __forceinline__ void flush() {
    const int lane = threadIdx.x & 31;
    if (lane < qn) sweep_elem<KC>(qa[lane], qr[lane], y, cnt, L, U, C, S);
    qn = 0;
    __syncwarp();
#pragma unroll
    for (int k = 0; k < KC; ++k) {
      S[k] += Sall;
      C[k] = (C[k] + Chi) + Clo;
    }
    Sall = 0.0; Clo = 0.0; Chi = 0.0;
  }
};

// r_k = C_k + y_k S_k into the (R, S) slot pair layout
template <int KC>
__device__ __forceinline__ void sweep_finish(const double* y, int cnt, double* C,
                                             const double* S) {
#pragma unroll
  for (int k = 0; k < KC; ++k)
    if (k < cnt) C[k] = C[k] + y[k] * S[k];
}

// cmd.sample = s > 0 (a sketch, controller.h: consume_sketch): only every
// 2^s-th step of the loop below runs; `count_slot` >= 0 then receives the
// number of elements visited.
template <int KC, bool WIDE>
__device__ __noinline__ void pass_sweep_row(const PassCtx& c, int j, int b, int cnt,
                                            int count_slot = -1) {
  const Problem& P = c.plan->P;
  const int64_t n = P.n, st = c.stride;
  const int shift = c.cmd->sample;
  const bool pf_l2 = n >= ((int64_t)1 << 22);   // (an L2-resident problem gains nothing: C2 + 2 us)
  double visited = 0.0, r0s = 0.0;   // sketch: elements visited, their sum of a clip(0, lo, hi)
  auto term0 = [&](bool ok, double a, double r) {
    const double lo = P.lower - r, hi = P.upper - r;
    return ok ? a * (0.0 < lo ? lo : (0.0 > hi ? hi : 0.0)) : 0.0;
  };
  const double* __restrict__ rho = P.rho;
  const double* __restrict__ ar = P.grad + (int64_t)j * P.ld;
  const int8_t* __restrict__ owner = P.owner;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // the warps' queues live in the reduction scratch (free until the end)
  typename std::conditional<WIDE, SweepAccW<KC>, SweepAcc<KC>>::type acc;
  acc.init(c.smem + warp * 2 * SQ_CAP, c.smem + warp * 2 * SQ_CAP + SQ_CAP, c.cmd->cand_y + b,
           cnt, P.lower, P.upper);
  StreamRows R;
  R.nr = 2;
  R.row[0] = ar;
  R.row[1] = rho;
  const int64_t rlo = owner ? P.row_lo[j] : 0, rhi = owner ? P.row_hi[j] : n;
  const bool gen = P.structured && P.row_kind[j] != RK_DENSE;
  const int gcode = gen ? srow_code(P, j) : 0;
  const GridIx G = grid_ix(P);
  // a constant row found by PREP (the volume row) is not read again
  const bool cst = !gen && P.n_alias && P.alias_kind[j] == AK_CONST;
  const double cv = cst ? P.alias_c[j] : 0.0;
  if ((!owner || P.part_ranges) && ((rlo | rhi) & 1) == 0 && (gen || cst || al16(ar)) &&
      al16(rho)) {
    // 16-byte pairs over the row's elements (its own range for a range
    // partition); the trip count is warp-uniform (push is warp-collective)
    const int64_t n2 = rhi >> 1;
    const double2* __restrict__ A2 = reinterpret_cast<const double2*>(ar);
    const double2* __restrict__ R2 = reinterpret_cast<const double2*>(rho);
    for (int64_t q0 = (rlo >> 1) + c.i0 - lane; q0 < n2; q0 += (2 * st) << shift) {
      const int64_t qa = q0 + lane, qb = q0 + st + lane;
      const bool oa = qa < n2, ob = qb < n2;
      if (pf_l2 && (lane & 7) == 0) {   // the next step's lines into L2 (see prep_pairs)
        const int64_t na = qa + ((2 * st) << shift), nb2 = na + st;
        if (na < n2) {
          prefetch_line_l2(R2 + na);
          if (!gen && !cst) prefetch_line_l2(A2 + na);
        }
        if (nb2 < n2) {
          prefetch_line_l2(R2 + nb2);
          if (!gen && !cst) prefetch_line_l2(A2 + nb2);
        }
      }
      if (WIDE) {   // one pair at a time (same elements, same order per lane)
        visited += (double)(2 * ((int)oa + (int)ob));
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
          const int64_t qq = h ? qb : qa;
          const bool oo = h ? ob : oa;
          double2 av = (oo && !gen && !cst) ? A2[qq] : make_double2(cv, cv);
          const double2 rv = oo ? R2[qq] : make_double2(0.0, 0.0);
          if (gen && oo) {
            int64_t c0[3], c1[3];
            grid_coords(G, 2 * qq + G.off, c0);
            grid_coords(G, 2 * qq + 1 + G.off, c1);
            av = make_double2(srow_fetch(c.rtab, gcode, c0), srow_fetch(c.rtab, gcode, c1));
          }
          if (shift) r0s += term0(oo, av.x, rv.x) + term0(oo, av.y, rv.y);
          acc.push(oo, av.x, rv.x);
          acc.push(oo, av.y, rv.y);
        }
        continue;
      }
      visited += (double)(2 * ((int)oa + (int)ob));
      double2 a0 = (oa && !gen && !cst) ? A2[qa] : make_double2(cv, cv);
      double2 a1 = (ob && !gen && !cst) ? A2[qb] : make_double2(cv, cv);
      const double2 r0 = oa ? R2[qa] : make_double2(0.0, 0.0), r1 = ob ? R2[qb] : make_double2(0.0, 0.0);
      if (gen) {   // structured row: generated from the element coordinates
        int64_t c0[3], c1[3];
        if (oa) {
          grid_coords(G, 2 * qa + G.off, c0);
          grid_coords(G, 2 * qa + 1 + G.off, c1);
          a0 = make_double2(srow_fetch(c.rtab, gcode, c0), srow_fetch(c.rtab, gcode, c1));
        }
        if (ob) {
          grid_coords(G, 2 * qb + G.off, c0);
          grid_coords(G, 2 * qb + 1 + G.off, c1);
          a1 = make_double2(srow_fetch(c.rtab, gcode, c0), srow_fetch(c.rtab, gcode, c1));
        }
      }
      if (shift)
        r0s += (term0(oa, a0.x, r0.x) + term0(oa, a0.y, r0.y)) +
               (term0(ob, a1.x, r1.x) + term0(ob, a1.y, r1.y));
      acc.push(oa, a0.x, r0.x);
      acc.push(oa, a0.y, r0.y);
      acc.push(ob, a1.x, r1.x);
      acc.push(ob, a1.y, r1.y);
    }
  } else {
  constexpr int UL = 4;   // elements' loads in flight per lane
  for (int64_t i0 = c.i0 - lane; i0 < n; i0 += (UL * st) << shift) {   // warp-uniform trip count
    double av[UL], rv[UL];
    bool ok[UL];
#pragma unroll
    for (int u = 0; u < UL; ++u) {
      const int64_t i = i0 + u * st + lane;
      ok[u] = i < n && (owner == nullptr || owner[i] == j);
      visited += ok[u] ? 1.0 : 0.0;
      av[u] = ok[u] ? ar[i] : 0.0;
      rv[u] = ok[u] ? rho[i] : 0.0;
    }
    if (shift) {
#pragma unroll
      for (int u = 0; u < UL; ++u) r0s += term0(ok[u], av[u], rv[u]);
    }
#pragma unroll
    for (int u = 0; u < UL; ++u) acc.push(ok[u], av[u], rv[u]);
  }
  }
  if constexpr (WIDE) {
    acc.flush();
    __syncthreads();   // queues (in c.smem) drained before the reduction reuses it
    sweep_finish<KC>(acc.y, cnt, acc.C, acc.S);
    double v[2 * KC];
#pragma unroll
    for (int k = 0; k < KC; ++k) { v[2 * k] = acc.C[k]; v[2 * k + 1] = acc.S[k]; }
    block_reduce_store<2 * KC>(v, 2 * cnt, PH_SWEEP, 2 * b, c.out, c.smem);
  } else {
  // per warp (R_k, S_k) into the head of its own queue region, then the
  // warps in order (the second stage of block_reduce_store)
  acc.finish(c.smem + warp * 2 * SQ_CAP);
  __syncthreads();
  if (threadIdx.x < 2 * cnt) {
    const int sl = threadIdx.x;
    double r = c.smem[sl];
    for (int w = 1; w < NWARP; ++w) r += c.smem[w * 2 * SQ_CAP + sl];
    c.out[2 * b + sl] = r;
  }
  __syncthreads();
  }
  if (shift) {   // sketch slots: [2 ncand] elements visited, [2 ncand + 1 + j] row j's sampled r(0) sum
    const double cv1[1] = {r0s};
    block_reduce_store<1>(cv1, 1, PH_SWEEP, 2 * c.cmd->ncand + 1 + j, c.out, c.smem);
  }
  if (count_slot >= 0) {
    const double cv1[1] = {visited};
    block_reduce_store<1>(cv1, 1, PH_SWEEP, count_slot, c.out, c.smem);
  }
}

// Compacted sweep of row j over the warps' active lists.  An element whose
// clip region (the reference's own predicate on fl(y a)) is the same at both
// ends of the walk interval keeps that region for every candidate in it
// (fl(y a) is monotone in y): its term is folded into the CTA's fixed sums --
// exactly a*lo or a*hi when clipped, y * a^2 when free -- and it leaves the
// list for good (the walk interval only shrinks).
template <int KC>
__device__ __noinline__ void pass_sweep_row_compact(const PassCtx& c, int j, int b, int cnt) {
  const Problem& P = c.plan->P;
  const Cmd& cmd = *c.cmd;
  const double* __restrict__ rho = P.rho;
  const double* __restrict__ ar = P.grad + (int64_t)j * P.ld;
  const int8_t* owner = P.owner;
  const double L = P.lower, U_ = P.upper;
  const double wlo = cmd.wlo[j], whi = cmd.whi[j];
  const double* y = cmd.cand_y + b;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // range partition: row j's own segment of the warp list (no owner tests)
  const bool segs = P.part_ranges && c.seg;
  int* sg = segs ? c.seg + (warp * MAX_M + j) * 2 : nullptr;
  uint32_t* Lst = c.list + (size_t)warp * c.list_cap + (segs ? sg[0] : 0);
  const int n_items = segs ? sg[1] : c.list_cnt[warp];
  if (segs) owner = nullptr;
  double R[KC], S[KC];
#pragma unroll
  for (int k = 0; k < KC; ++k) { R[k] = 0.0; S[k] = 0.0; }
  double nC = 0.0, nS = 0.0;
  int kept = 0;
  // Phase 1: classify every listed element against the window (loads of UC
  // entries in flight per lane), fold the fixed ones and compact the list in
  // order.  Phase 2 then evaluates the kept elements only, 32 per warp step,
  // so a warp is not held by one active lane.
  constexpr int UC = 4;
  for (int base = 0; base < n_items; base += 32 * UC) {
    uint32_t iv[UC];
    double av[UC], rv[UC];
    bool rel[UC];
#pragma unroll
    for (int u = 0; u < UC; ++u) {
      const int idx = base + u * 32 + lane;
      const bool valid = idx < n_items;
      iv[u] = valid ? Lst[idx] : 0u;
      rel[u] = valid && (owner == nullptr || owner[iv[u]] == j);
      av[u] = rel[u] ? ar[iv[u]] : 0.0;
      rv[u] = rel[u] ? rho[iv[u]] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < UC; ++u) {
      const int idx = base + u * 32 + lane;
      const bool valid = idx < n_items;
      bool fixed = false;
      if (rel[u]) {
        const double a = av[u], r = rv[u];
        const double lo = L - r, hi = U_ - r;
        const double v1 = wlo * a, v2 = whi * a;
        const int g1 = v1 < lo ? 0 : (v1 > hi ? 2 : 1);
        const int g2 = v2 < lo ? 0 : (v2 > hi ? 2 : 1);
        if (g1 == g2) {
          fixed = true;
          if (g1 == 0) nC += a * lo;
          else if (g1 == 2) nC += a * hi;
          else nS += a * a;
        }
      }
      // rows other than j keep their items (partitioned problems)
      const bool keep = valid && !(rel[u] && fixed);
      const unsigned km = __ballot_sync(0xffffffffu, keep);
      if (keep) Lst[kept + __popc(km & ((1u << lane) - 1u))] = iv[u];
      kept += __popc(km);
    }
  }
  __syncwarp();
  // Phase 2: the window's active elements of row j
  for (int k = lane; k < kept; k += 32) {
    const uint32_t i = Lst[k];
    if (owner && owner[i] != j) continue;
    sweep_elem<KC>(ar[i], rho[i], y, cnt, L, U_, R, S);
  }
  __syncwarp();
  if (lane == 0) {
    if (segs) sg[1] = kept; else c.list_cnt[warp] = kept;
  }
  sweep_finish<KC>(y, cnt, R, S);
  // CTA totals of this sweep's active sums and newly fixed sums
  double v[2 * KC + 2];
#pragma unroll
  for (int k = 0; k < KC; ++k) { v[2 * k] = R[k]; v[2 * k + 1] = S[k]; }
  v[2 * KC] = nC;
  v[2 * KC + 1] = nS;
  double* sred = c.smem;
  warp_reduce_slots<2 * KC + 2, false>(v, PH_SWEEP, 0, sred + warp * (2 * KC + 2));
  __syncthreads();
  double* tot = c.smem + NWARP * (2 * KC + 2);
  if (threadIdx.x < 2 * KC + 2) {
    double r = sred[threadIdx.x];
    for (int w = 1; w < NWARP; ++w) r += sred[w * (2 * KC + 2) + threadIdx.x];
    tot[threadIdx.x] = r;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    c.fixC[j] += tot[2 * KC];
    c.fixS[j] += tot[2 * KC + 1];
  }
  __syncthreads();
  if (threadIdx.x < cnt) {
    const int k = threadIdx.x;
    c.out[2 * (b + k)] = tot[2 * k] + (c.fixC[j] + y[k] * c.fixS[j]);
    c.out[2 * (b + k) + 1] = tot[2 * k + 1] + c.fixS[j];
  }
  __syncthreads();
}

// ---- fused multi-row sweep (rows found structured by PREP) ------------------
// The stage-1 sweeps of C4/C5 walk up to 4 rows at once.  pass_sweep_row
// reads rho and the row once PER ROW; here one pass over the elements reads
// rho and each walking row's data once (a constant row -- the volume row --
// not at all; a negated row as its base) and serves every walking row.
//
// Per element and row the clip region of the reference's own predicate on
// fl(y a) is taken at the two ends of the row's candidate window [y_first,
// y_last] (two products, four compares, no reciprocal): fl(y a) is monotone
// in y, so an element with the same region at both ends has it at every
// candidate in between and adds its exact term -- a lo, a hi, or a^2 for the
// slope of y a^2 -- to one of two running sums.  Only elements whose region
// changes inside the window are queued per (warp, row) and, 32 at a time, run
// through the per-candidate loop (sweep_elem) in ms_flush, whose per-lane
// sums are folded into the warp's shared-memory accumulators by a fixed
// shuffle tree.  With the root sketch (controller.h) every full sweep has a
// narrow window, so the queue path is rare.  Deterministic; the sums differ
// from the per-row sweep only in (certified) rounding.
constexpr int MS_ROWS = 4;      // walking rows per fused sweep
constexpr int MS_Q = 64;        // queue entries per (warp, row)
__host__ __device__ constexpr size_t multi_sweep_bytes() {
  return sizeof(double) * (size_t)NWARP * MS_ROWS * (2 * MAX_K + 2 * MS_Q);
}

// lanes < cntq hold queued items qa[from + lane] (a), qa[MS_Q + from + lane] (rho)
template <int KC>
__device__ __noinline__ void ms_flush_k(const double* qa, double* acc, const double* y, int cn,
                                        double L, double U, int from, int cntq) {
  const int lane = threadIdx.x & 31;
  double C[KC], S[KC];
#pragma unroll
  for (int k = 0; k < KC; ++k) { C[k] = 0.0; S[k] = 0.0; }
  if (lane < cntq) sweep_elem<KC>(qa[from + lane], qa[MS_Q + from + lane], y, cn, L, U, C, S);
#pragma unroll
  for (int k = 0; k < KC; ++k) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      C[k] += __shfl_down_sync(0xffffffffu, C[k], o);
      S[k] += __shfl_down_sync(0xffffffffu, S[k], o);
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < KC; ++k) { acc[2 * k] += C[k]; acc[2 * k + 1] += S[k]; }
  }
  __syncwarp();
}
__device__ __noinline__ void ms_flush(int kc, const double* qa, double* acc, const double* y,
                                      int cn, double L, double U, int from, int cntq) {
  if (kc <= 8) ms_flush_k<8>(qa, acc, y, cn, L, U, from, cntq);
  else if (kc <= 12) ms_flush_k<12>(qa, acc, y, cn, L, U, from, cntq);
  else ms_flush_k<MAX_K>(qa, acc, y, cn, L, U, from, cntq);
}

// Candidates far outside the others -- in a walk's first sweep the
// infeasibility probe at the bracket end (projection.cpp:80-94) and the first
// midpoints of a bracket much wider than the root's neighbourhood -- would
// stretch the window over nearly every element's breakpoints.  Up to two of
// them at one end are kept out of the window: ms_outliers finds them (their
// gap to the next candidate more than 4x the span of the rest), and the OUTL
// instantiation evaluates each for every un-queued element with its own
// region test and sums.  Returns their count; *low: at the low end.
__device__ __forceinline__ int ms_outliers(const double* y, int cn, bool* low) {
  *low = true;
  if (cn < 4) return 0;
  const double y1 = y[0], y2 = y[1], y3 = y[2], yz = y[cn - 1], yy = y[cn - 2], yx = y[cn - 3];
  const int nlo = (y3 - y2) > 4.0 * (yz - y3) ? 2 : ((y2 - y1) > 4.0 * (yz - y2) ? 1 : 0);
  const int nhi = (yy - yx) > 4.0 * (yx - y1) ? 2 : ((yz - yy) > 4.0 * (yy - y1) ? 1 : 0);
  if (nlo >= nhi) return nlo;
  *low = false;
  return nhi;
}

template <int NW, bool OUTL>
__device__ __noinline__ void pass_sweep_multi_t(const PassCtx& c, const int* wrow, int kmax) {
  constexpr int nw = NW;
  const Problem& P = c.plan->P;
  const Cmd& cmd = *c.cmd;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double L = P.lower, U = P.upper;
  const int64_t n2 = P.n >> 1, st = c.stride, ld2 = P.ld >> 1;
  const double2* __restrict__ R2 = reinterpret_cast<const double2*>(P.rho);
  const double2* __restrict__ A2 = reinterpret_cast<const double2*>(P.grad);
  double* wacc = reinterpret_cast<double*>(c.ms_smem) + (size_t)warp * MS_ROWS * 2 * MAX_K;
  double* qbase = reinterpret_cast<double*>(c.ms_smem) + (size_t)NWARP * MS_ROWS * 2 * MAX_K +
                  (size_t)warp * MS_ROWS * 2 * MS_Q;
  // per walking row: data source, candidate window, running sums
  int64_t off[NW];
  int qn[NW];
  unsigned negm = 0u, cstm = 0u;   // bit w: row w is a negated / a constant row
  double cst = 0.0;                // (constant rows of one problem share their value: one volume row)
  double y0[NW], yl[NW], Sall[NW], Cfix[NW];
  constexpr int NO = OUTL ? 2 * NW : 1;
  double yo[NO], So[NO], Co[NO];   // the outlier candidates (two slots per row)
  int no[NW];                      // their count, negated when they sit at the high end
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const int j = wrow[w];
    const int ak = P.alias_kind[j];
    const int cb = cmd.row_start[j];
    const int cn = cmd.row_start[j + 1] - cb;
    if (ak == AK_NEG) negm |= 1u << w;
    if (ak == AK_CONST) { cstm |= 1u << w; cst = P.alias_c[j]; }
    off[w] = (int64_t)(ak == AK_NEG ? j - 1 : j) * ld2;
    bool olow = true;
    const int nout = OUTL ? ms_outliers(cmd.cand_y + cb, cn, &olow) : 0;
    no[w] = olow ? nout : -nout;
    y0[w] = cmd.cand_y[cb + (olow ? nout : 0)];
    yl[w] = cmd.cand_y[cb + (cn > 0 ? cn - 1 : 0) - (olow ? 0 : nout)];
    if (OUTL) {
#pragma unroll
      for (int u = 0; u < 2; ++u) {   // outlier u = candidate u (low end) / cn - nout + u (high end)
        yo[2 * w + u] = u < nout ? cmd.cand_y[cb + (olow ? u : cn - nout + u)] : y0[w];
        So[2 * w + u] = Co[2 * w + u] = 0.0;
      }
    }
    Sall[w] = Cfix[w] = 0.0;
    qn[w] = 0;
  }
  for (int k = lane; k < MS_ROWS * 2 * MAX_K; k += 32) wacc[k] = 0.0;
  __syncwarp();
  auto flush = [&](int w, int from, int cntq) {
    const int j = wrow[w];
    const int cb = cmd.row_start[j];
    ms_flush(kmax, qbase + (size_t)w * 2 * MS_Q, wacc + (size_t)w * 2 * MAX_K, cmd.cand_y + cb,
             cmd.row_start[j + 1] - cb, L, U, from, cntq);
  };
  // row w's value at an element from the loaded pair value
  auto rowval = [&](int w, double v) {
    return ((cstm >> w) & 1u) ? cst : (((negm >> w) & 1u) ? -v : v);
  };
  // queue the lanes whose bit is set in their needmask for row w
  auto enqueue = [&](int w, bool need, double a, double r) {
    const unsigned nm = __ballot_sync(0xffffffffu, need);
    if (nm) {
      double* qa = qbase + (size_t)w * 2 * MS_Q;
      if (need) {
        const int slot = qn[w] + __popc(nm & ((1u << lane) - 1u));
        qa[slot] = a;
        qa[MS_Q + slot] = r;
      }
      qn[w] += __popc(nm);
      __syncwarp();
      if (qn[w] >= 32) {
        flush(w, qn[w] - 32, 32);
        qn[w] -= 32;
      }
    }
  };
  // One pair per thread and step, the next step's loads issued before this
  // step's arithmetic (the classification is branch-free: every (element,
  // row) is independent work for the fp64 pipe while the loads are in flight).
  const double2 z2 = make_double2(0.0, 0.0);
  int64_t q0 = c.i0 - lane;   // warp-uniform trip count
  double2 r2 = z2, v2[NW];
  {
    const int64_t q = q0 + lane;
    const bool ok = q < n2;
    r2 = ok ? R2[q] : z2;
#pragma unroll
    for (int w = 0; w < NW; ++w) v2[w] = (ok && !((cstm >> w) & 1u)) ? A2[off[w] + q] : z2;
  }
  for (; q0 < n2; q0 += st) {
    const bool ok = q0 + lane < n2;
    const int64_t qn1 = q0 + st + lane;
    const bool ok1 = qn1 < n2;
    const double2 r2n = ok1 ? R2[qn1] : z2;
    double2 v2n[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) v2n[w] = (ok1 && !((cstm >> w) & 1u)) ? A2[off[w] + qn1] : z2;
    const double lo0 = L - r2.x, hi0 = U - r2.x, lo1 = L - r2.y, hi1 = U - r2.y;
    unsigned needmask = 0u;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const double a = rowval(w, e ? v2[w].y : v2[w].x);
        const double lo = e ? lo1 : lo0, hi = e ? hi1 : hi0;
        const double t0 = y0[w] * a, tl = yl[w] * a;
        const bool b0 = t0 < lo, a0 = t0 > hi, bl = tl < lo, al = tl > hi;
        const bool live = ok && a != 0.0;
        const bool same = (b0 == bl) && (a0 == al);   // one region over the whole window
        const double term = b0 ? a * lo : (a0 ? a * hi : 0.0);
        Cfix[w] += (live && same) ? term : 0.0;
        Sall[w] += (live && same && !b0 && !a0) ? a * a : 0.0;
        needmask |= (live && !same) ? (1u << (2 * w + e)) : 0u;
        if (OUTL) {   // the outlier candidates' own regions (queued elements get them in ms_flush)
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const double to = yo[2 * w + u] * a;
            const bool bo = to < lo, ao = to > hi;
            Co[2 * w + u] += (live && same) ? (bo ? a * lo : (ao ? a * hi : 0.0)) : 0.0;
            So[2 * w + u] += (live && same && !bo && !ao) ? a * a : 0.0;
          }
        }
      }
    }
    if (__any_sync(0xffffffffu, needmask != 0u)) {   // rare once the window is narrow
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        enqueue(w, (needmask >> (2 * w)) & 1u, rowval(w, v2[w].x), r2.x);
        enqueue(w, (needmask >> (2 * w + 1)) & 1u, rowval(w, v2[w].y), r2.y);
      }
    }
    r2 = r2n;
#pragma unroll
    for (int w = 0; w < NW; ++w) v2[w] = v2n[w];
  }
#pragma unroll
  for (int w = 0; w < NW; ++w)
    if (qn[w] > 0) flush(w, 0, qn[w]);
  __syncthreads();   // the reduction scratch is reused below
  // per row: thread sums + (lane 0) the warp's queued sums, then the CTA reduction
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const int j = wrow[w];
    const int cb = cmd.row_start[j], cn = cmd.row_start[j + 1] - cb;
    const double* acc = wacc + (size_t)w * 2 * MAX_K;
    for (int k0 = 0; k0 < cn; k0 += 4) {   // 4 candidates (8 slots) per reduction
      double v[8];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k = k0 + u;
        double Ck = Cfix[w], Sk = Sall[w];
        if (OUTL) {
          const int nout = no[w] < 0 ? -no[w] : no[w];
          const int u = no[w] >= 0 ? k : k - (cn - nout);   // outlier slot of candidate k, if any
          if (u >= 0 && u < nout && k < cn) {
            Ck = u == 0 ? Co[2 * w] : Co[2 * w + 1];
            Sk = u == 0 ? So[2 * w] : So[2 * w + 1];
          }
        }
        if (lane == 0 && k < cn) { Ck = Ck + acc[2 * k]; Sk = Sk + acc[2 * k + 1]; }
        const double yk = k < cn ? cmd.cand_y[cb + k] : 0.0;
        v[2 * u] = Ck + yk * Sk;
        v[2 * u + 1] = Sk;
      }
      const int ns = 2 * (cn - k0 < 4 ? cn - k0 : 4);
      block_reduce_store<8>(v, ns, PH_SWEEP, 2 * (cb + k0), c.out, c.smem);
    }
  }
}

__device__ void pass_sweep_multi(const PassCtx& c, int nw, const int* wrow, int kmax) {
  const Cmd& cmd = *c.cmd;
  bool outl = false;
  for (int w = 0; w < nw; ++w) {
    const int cb = cmd.row_start[wrow[w]];
    bool low;
    outl = outl || ms_outliers(cmd.cand_y + cb, cmd.row_start[wrow[w] + 1] - cb, &low) > 0;
  }
  if (outl) {   // (the outlier sums cost registers: two rows per pass over the elements)
    for (int w = 0; w < nw; w += 2) {
      if (w + 1 < nw) pass_sweep_multi_t<2, true>(c, wrow + w, kmax);
      else pass_sweep_multi_t<1, true>(c, wrow + w, kmax);
      __syncthreads();
    }
  } else {
    if (nw == 2) pass_sweep_multi_t<2, false>(c, wrow, kmax);
    else if (nw == 3) pass_sweep_multi_t<3, false>(c, wrow, kmax);
    else pass_sweep_multi_t<4, false>(c, wrow, kmax);
  }
}

__device__ void pass_sweep(const PassCtx& c) {
  const Cmd& cmd = *c.cmd;
  const int m = c.plan->P.m;
  {   // rows with detected structure: one fused pass for all walking rows
    const Problem& P = c.plan->P;
    int wrow[MS_ROWS], nw = 0, kmax = 0;
    bool fit = !cmd.compact && !cmd.sample && c.ms_smem && P.n_alias && !P.owner && !P.structured &&
               (P.n & 1) == 0 && (P.ld & 1) == 0 && al16(P.rho) && al16(P.grad);
    int ncst = 0;
    for (int j = 0; j < m && fit; ++j) {
      const int cnt = cmd.row_start[j + 1] - cmd.row_start[j];
      if (cnt <= 0) continue;
      if (nw == MS_ROWS) { fit = false; break; }
      if (P.alias_kind[j] == AK_CONST && ++ncst > 1) { fit = false; break; }   // one constant row
      wrow[nw++] = j;
      kmax = cnt > kmax ? cnt : kmax;
    }
    if (fit && nw >= 2) {
      pass_sweep_multi(c, nw, wrow, kmax);
      return;
    }
  }
  bool counted = false;
  for (int j = 0; j < m; ++j) {
    const int b = cmd.row_start[j], cnt = cmd.row_start[j + 1] - b;
    if (cnt <= 0) continue;
    if (cmd.compact && c.list) {
      if (cnt <= 4) pass_sweep_row_compact<4>(c, j, b, cnt);
      else if (cnt <= 8) pass_sweep_row_compact<8>(c, j, b, cnt);
      else pass_sweep_row_compact<MAX_K>(c, j, b, cnt);
      continue;
    }
    // (10 / 12: the multi-row stage-1 sweeps, MAX_CAND / rows candidates per
    // row -- the per-element work is one select + add per template slot)
    // a sketch: the first row with candidates also counts the sampled elements
    const int cslot = (cmd.sample && !counted) ? 2 * cmd.ncand : -1;
    counted = counted || cslot >= 0;
    // a walk's first full sweep and the sketches have wide windows: the
    // per-lane candidate loop; later sweeps: the lean transposed batch
    if (cmd.sample || c.plan->res.sweeps <= 1) {
      if (cnt <= 4) pass_sweep_row<4, true>(c, j, b, cnt, cslot);
      else if (cnt <= 8) pass_sweep_row<8, true>(c, j, b, cnt, cslot);
      else if (cnt <= 10) pass_sweep_row<10, true>(c, j, b, cnt, cslot);
      else if (cnt <= 12) pass_sweep_row<12, true>(c, j, b, cnt, cslot);
      else pass_sweep_row<MAX_K, true>(c, j, b, cnt, cslot);
    } else {
      pass_sweep_row<MAX_K, false>(c, j, b, cnt, cslot);
    }
  }
  if (cmd.compact && c.list) {   // active elements left in this CTA
    __shared__ int s_woff[NWARP + 1];
    if (c.plan->P.part_ranges && c.seg) {
      // close the gaps the per-row compactions left: segments back to back in
      // row order (every move goes to a lower address, in increasing order)
      __syncthreads();
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
      uint32_t* Lw = c.list + (size_t)warp * c.list_cap;
      int off = 0;
      for (int j = 0; j < m; ++j) {
        int* sg = c.seg + (warp * MAX_M + j) * 2;
        const int s0 = sg[0], n0 = sg[1];
        for (int k0 = 0; k0 < n0; k0 += 32) {
          const int k = k0 + lane;
          const uint32_t v = k < n0 ? Lw[s0 + k] : 0u;
          __syncwarp();
          if (k < n0) Lw[off + k] = v;
          __syncwarp();
        }
        __syncwarp();
        if (lane == 0) sg[0] = off;
        off += n0;
      }
      if (lane == 0) c.list_cnt[warp] = off;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int tot = 0;
      for (int w = 0; w < NWARP; ++w) { s_woff[w] = tot; tot += c.list_cnt[w]; }
      s_woff[NWARP] = tot;
      c.out[2 * cmd.ncand] = (double)tot;
      c.out[2 * cmd.ncand + 1] = tot > GATHER_BLK ? 1.0 : 0.0;
      c.blk_cnt[blockIdx.x] = tot;
    }
    __syncthreads();
    if (s_woff[NWARP] <= GATHER_BLK) {
      // publish this CTA's items and fixed sums in its own region: when the
      // total is small enough, every CTA loads them after the barrier and
      // the walk continues CTA-locally without a separate gather pass
      const Problem& P = c.plan->P;
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
      const uint32_t* __restrict__ Lst = c.list + (size_t)warp * c.list_cap;
      const int cnt = c.list_cnt[warp];
      const size_t base = (size_t)blockIdx.x * GATHER_BLK + s_woff[warp];
      double* __restrict__ g_a = c.g_a;
      double* __restrict__ g_r = c.g_r;
      int* __restrict__ g_row = c.g_row;
      const int8_t* __restrict__ owner = P.owner;
      const double* __restrict__ grad = P.grad;
      const double* __restrict__ rho = P.rho;
      const int64_t ld = P.ld;
      for (int k = lane; k < cnt; k += 32) {
        const uint32_t i = Lst[k];
        const int row = owner ? (int)owner[i] : 0;
        g_a[base + k] = grad[(int64_t)row * ld + i];
        g_r[base + k] = rho[i];
        g_row[base + k] = row;
      }
      if (threadIdx.x < m) {
        c.g_fix[((size_t)blockIdx.x * MAX_M + threadIdx.x) * 2] = c.fixC[threadIdx.x];
        c.g_fix[((size_t)blockIdx.x * MAX_M + threadIdx.x) * 2 + 1] = c.fixS[threadIdx.x];
      }
    }
  }
}

// ---- PH_GATHER: write this CTA's active items and fixed sums ---------------
__device__ __noinline__ void pass_gather(const PassCtx& c) {
  const Problem& P = c.plan->P;
  const int m = P.m;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ int s_off[NWARP + 1];
  if (warp == 0) {   // items of the CTAs before this one: loads issued together
    int off = 0;
    for (int b0 = 0; b0 < (int)blockIdx.x; b0 += 32) {
      const int b = b0 + lane;
      off += __reduce_add_sync(0xffffffffu, b < (int)blockIdx.x ? __ldcg(c.blk_cnt + b) : 0);
    }
    if (lane == 0) {
      s_off[0] = off;
      for (int w = 0; w < NWARP; ++w) s_off[w + 1] = s_off[w] + c.list_cnt[w];
    }
  }
  __syncthreads();
  const uint32_t* Lst = c.list + (size_t)warp * c.list_cap;
  const int cnt = c.list_cnt[warp], base = s_off[warp];
  for (int k = lane; k < cnt; k += 32) {
    const uint32_t i = Lst[k];
    const int row = P.owner ? (int)P.owner[i] : 0;
    const int dst = base + k;
    if (dst < GATHER_CAP) {
      c.g_a[dst] = P.grad[(int64_t)row * P.ld + i];
      c.g_r[dst] = P.rho[i];
      c.g_row[dst] = row;
    }
  }
  if (threadIdx.x < m) {
    c.g_fix[((size_t)blockIdx.x * MAX_M + threadIdx.x) * 2] = c.fixC[threadIdx.x];
    c.g_fix[((size_t)blockIdx.x * MAX_M + threadIdx.x) * 2 + 1] = c.fixS[threadIdx.x];
  }
  __syncthreads();
}

// After the gather barrier: every CTA loads all items and the fixed totals
// (summed over CTAs in index order) into its shared memory.
__device__ __noinline__ void gather_load(const PassCtx& c, int nb) {
  const int m = c.plan->P.m;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ int s_total;
  if (warp == 0) {
    int t = 0;
    for (int b0 = 0; b0 < nb; b0 += 32) {
      const int b = b0 + lane;
      t += __reduce_add_sync(0xffffffffu, b < nb ? __ldcg(c.blk_cnt + b) : 0);
    }
    if (lane == 0) {
      s_total = t < GATHER_CAP ? t : GATHER_CAP;
      *c.n_items = s_total;
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < s_total; k += BLOCK) {
    c.it_a[k] = __ldcg(c.g_a + k);
    c.it_r[k] = __ldcg(c.g_r + k);
    c.it_row[k] = (int8_t)__ldcg(c.g_row + k);
  }
  // fixed sums over the CTAs: warp w takes slot w (C_j, S_j interleaved);
  // lane l sums CTAs l, l+32, ... then a fixed shuffle tree (deterministic)
  for (int sl = warp; sl < 2 * m; sl += NWARP) {
    double v = 0.0;
    for (int b = lane; b < nb; b += 32) v += __ldcg(c.g_fix + (size_t)b * MAX_M * 2 + sl);
    v = warp_reduce(0, v);
    if (lane == 0) {
      if (sl & 1) c.fixS[sl >> 1] = v; else c.fixC[sl >> 1] = v;
    }
  }
  __syncthreads();
}

// Fused gather: after the barrier of a compacted sweep in which every CTA
// published its (<= GATHER_BLK) items in its own region, every CTA loads all
// of them in CTA order (the order pass_gather + gather_load would give) and
// sums the fixed totals over the CTAs in index order.
__device__ __noinline__ void gather_load_fused(const PassCtx& c, int nb) {
  const int m = c.plan->P.m;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // locals: stores through the (generic) item pointers would otherwise force
  // a reload of every context field after each store
  int* __restrict__ s_off = reinterpret_cast<int*>(c.smem);   // [nb + 1] item offsets
  const int* __restrict__ blk_cnt = c.blk_cnt;
  const double* __restrict__ g_a = c.g_a;
  const double* __restrict__ g_r = c.g_r;
  const int* __restrict__ g_row = c.g_row;
  const double* __restrict__ g_fix = c.g_fix;
  double* __restrict__ it_a = c.it_a;
  double* __restrict__ it_r = c.it_r;
  int8_t* __restrict__ it_row = c.it_row;
  double* __restrict__ fixC = c.fixC;
  double* __restrict__ fixS = c.fixS;
  int* __restrict__ n_items = c.n_items;
  if (warp == 0) {
    int run = 0;
    for (int b0 = 0; b0 < nb; b0 += 32) {
      const int b = b0 + lane;
      const int v = b < nb ? __ldcg(blk_cnt + b) : 0;
      int incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
      }
      if (b < nb) s_off[b] = run + incl - v;
      run += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) {
      s_off[nb] = run;
      *n_items = run < GATHER_CAP ? run : GATHER_CAP;
    }
  }
  __syncthreads();
  // destination-major: item t sits in the CTA b with s_off[b] <= t < s_off[b+1]
  // (binary search); four items' loads are issued together per thread
  const int total = *n_items;
  for (int t0 = threadIdx.x; t0 < total; t0 += 4 * BLOCK) {
    double va[4], vr[4];
    int vw[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int t = t0 + u * BLOCK;
      va[u] = 0.0; vr[u] = 0.0; vw[u] = 0;
      if (t < total) {
        int lo = 0, hi = nb;   // s_off[lo] <= t < s_off[hi]
        while (hi - lo > 1) {
          const int mid = (lo + hi) >> 1;
          if (s_off[mid] <= t) lo = mid; else hi = mid;
        }
        const size_t src = (size_t)lo * GATHER_BLK + (t - s_off[lo]);
        va[u] = __ldcg(g_a + src);
        vr[u] = __ldcg(g_r + src);
        vw[u] = __ldcg(g_row + src);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int t = t0 + u * BLOCK;
      if (t < total) { it_a[t] = va[u]; it_r[t] = vr[u]; it_row[t] = (int8_t)vw[u]; }
    }
  }
  for (int sl = warp; sl < 2 * m; sl += NWARP) {
    double v = 0.0;
    for (int b = lane; b < nb; b += 32) v += __ldcg(g_fix + (size_t)b * MAX_M * 2 + sl);
    v = warp_reduce(0, v);
    if (lane == 0) {
      if (sl & 1) fixS[sl >> 1] = v; else fixC[sl >> 1] = v;
    }
  }
  __syncthreads();
}

// CTA-local compaction of row j's gathered items against the walk window
// (same predicate and folding as pass_sweep_row_compact): fixed items go
// into fixC / fixS, the rest are compacted in order.  Every CTA holds the
// same items and does the same arithmetic in the same order.
__device__ __noinline__ void local_compact_row(const PassCtx& c, int j) {
  const Problem& P = c.plan->P;
  const double L = P.lower, U = P.upper;
  const double wlo = c.cmd->wlo[j], whi = c.cmd->whi[j];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ int s_wc[NWARP];
  __shared__ int s_base;
  double* __restrict__ it_a = c.it_a;
  double* __restrict__ it_r = c.it_r;
  int8_t* __restrict__ it_row = c.it_row;
  double* __restrict__ sm = c.smem;
  const int nit = *c.n_items;
  if (threadIdx.x == 0) s_base = 0;
  double nC = 0.0, nS = 0.0;
  for (int c0 = 0; c0 < nit; c0 += BLOCK) {
    const int k = c0 + threadIdx.x;
    const bool valid = k < nit;
    const double a = valid ? it_a[k] : 0.0, r = valid ? it_r[k] : 0.0;
    const int8_t row = valid ? it_row[k] : (int8_t)-1;
    bool fixed = false;
    if (valid && row == j) {
      const double lo = L - r, hi = U - r;
      const double v1 = wlo * a, v2 = whi * a;
      const int g1 = v1 < lo ? 0 : (v1 > hi ? 2 : 1);
      const int g2 = v2 < lo ? 0 : (v2 > hi ? 2 : 1);
      if (g1 == g2) {
        fixed = true;
        if (g1 == 0) nC += a * lo;
        else if (g1 == 2) nC += a * hi;
        else nS += a * a;
      }
    }
    const bool keep = valid && !fixed;
    const unsigned km = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) s_wc[warp] = __popc(km);
    __syncthreads();   // every read of this chunk is done before any write
    int off = s_base;
    for (int w = 0; w < warp; ++w) off += s_wc[w];
    if (keep) {
      const int dst = off + __popc(km & ((1u << lane) - 1u));
      it_a[dst] = a; it_r[dst] = r; it_row[dst] = row;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int tot = 0;
      for (int w = 0; w < NWARP; ++w) tot += s_wc[w];
      s_base += tot;
    }
  }
  // fixed sums: fixed shuffle tree, warps in order
  nC = warp_reduce(0, nC);
  nS = warp_reduce(0, nS);
  if (lane == 0) { sm[warp] = nC; sm[NWARP + warp] = nS; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double C = sm[0], S = sm[NWARP];
    for (int w = 1; w < NWARP; ++w) { C += sm[w]; S += sm[NWARP + w]; }
    c.fixC[j] += C;
    c.fixS[j] += S;
    *c.n_items = s_base;
  }
  __syncthreads();
}

// CTA-local sweep over the gathered items: totals go straight to tot[]
// (no partials, no grid barrier; every CTA computes the same bits).
template <int KC>
__device__ __noinline__ void local_sweep_row(const PassCtx& c, int j, int b, int cnt,
                                             double* tot) {
  const Problem& P = c.plan->P;
  const double L = P.lower, U = P.upper;
  const double* y = c.cmd->cand_y + b;
  const int nit = *c.n_items;
  double R[KC], S[KC];
#pragma unroll
  for (int k = 0; k < KC; ++k) { R[k] = 0.0; S[k] = 0.0; }
  const double* __restrict__ it_a = c.it_a;
  const double* __restrict__ it_r = c.it_r;
  const int8_t* __restrict__ it_row = c.it_row;
  for (int k = threadIdx.x; k < nit; k += BLOCK)
    if (it_row[k] == j) sweep_elem<KC>(it_a[k], it_r[k], y, cnt, L, U, R, S);
  sweep_finish<KC>(y, cnt, R, S);
  const int warp = threadIdx.x >> 5;
  double* sred = c.smem;
  {
    double v[2 * KC];
#pragma unroll
    for (int k = 0; k < KC; ++k) { v[2 * k] = R[k]; v[2 * k + 1] = S[k]; }
    warp_reduce_slots<2 * KC, false>(v, PH_SWEEP, 0, sred + warp * 2 * KC);
  }
  __syncthreads();
  if (threadIdx.x < 2 * cnt) {
    double r = sred[threadIdx.x];
    for (int w = 1; w < NWARP; ++w) r += sred[w * 2 * KC + threadIdx.x];
    const int k = threadIdx.x >> 1;
    tot[2 * b + threadIdx.x] = (threadIdx.x & 1) ? r + c.fixS[j]
                                                  : r + (c.fixC[j] + y[k] * c.fixS[j]);
  }
  __syncthreads();
}

__device__ void local_sweep(const PassCtx& c, double* tot) {
  const Cmd& cmd = *c.cmd;
  const int m = c.plan->P.m;
  for (int j = 0; j < m; ++j) {
    const int b = cmd.row_start[j], cnt = cmd.row_start[j + 1] - b;
    if (cnt <= 0) continue;
    if (cmd.compact) local_compact_row(c, j);
    if (cnt <= 4) local_sweep_row<4>(c, j, b, cnt, tot);
    else if (cnt <= 8) local_sweep_row<8>(c, j, b, cnt, tot);
    else local_sweep_row<MAX_K>(c, j, b, cnt, tot);
  }
}

// ---- PH_FEAS: stage-1 dots a_k . clip(y_j a_j) (projection.cpp:320-333) ---
// Streamed: up to FEAS_GROUP candidates per pass over (rho, A), their m dots
// each accumulated per thread in the reference's row order.
constexpr int FEAS_GROUP = 4;
__device__ __noinline__ void pass_feas_streamed(const PassCtx& c) {
  constexpr int M = 8;
  const Plan& pl = *c.plan;
  const Problem& P = pl.P;
  const Cmd& cmd = *c.cmd;
  const double L = P.lower, U = P.upper;
  const int m = P.m;
  const int64_t n = P.n;
  StreamRows R;
  R.nr = m + 1;
  R.row[0] = P.rho;
  for (int k = 0; k < m && k + 1 < RP_MAXR; ++k) set_arow(R, 1 + k, c, P, k);
  for (int f0 = 0; f0 < cmd.nfeas; f0 += FEAS_GROUP) {
    double acc[FEAS_GROUP][M];
    int rj[FEAS_GROUP];
    double yj[FEAS_GROUP];
#pragma unroll
    for (int g = 0; g < FEAS_GROUP; ++g) {
      const bool on = f0 + g < cmd.nfeas;
      rj[g] = on ? cmd.feas_row[f0 + g] : -1;
      yj[g] = on ? cmd.feas_y[f0 + g] : 0.0;
#pragma unroll
      for (int k = 0; k < M; ++k) acc[g][k] = 0.0;
    }
    rows_pairs<M + 1>(c, R, n, [&](int64_t, const double (&v)[M + 1]) {
      const double r = v[0];
      const double lo = L - r, hi = U - r;
#pragma unroll
      for (int g = 0; g < FEAS_GROUP; ++g) {
        double z = 0.0;
        if (rj[g] >= 0 && yj[g] != 0.0) {
          double arj = 0.0;
#pragma unroll
          for (int k = 0; k < M; ++k)
            if (k == rj[g]) arj = v[1 + k];
          z = 0.0 + yj[g] * arj;
        }
        const double dl = clipd(z, lo, hi);
#pragma unroll
        for (int k = 0; k < M; ++k)
          if (k < m) acc[g][k] += v[1 + k] * dl;
      }
    });
#pragma unroll
    for (int g = 0; g < FEAS_GROUP; ++g)
      if (f0 + g < cmd.nfeas) block_reduce_store<M>(acc[g], m, PH_FEAS, (f0 + g) * m, c.out, c.smem);
  }
}

// Dense rows, exact m = M (C4/C5): pass_feas_streamed with one base pointer
// for the rows and the candidates' (row, dual) re-read from the shared-memory
// command per element (register-lean: no spills in the loop).  Same element
// order per thread and the same per-element arithmetic; the zero-padded warp
// reduction of M and of pass_feas_streamed's 8 slots are the same.
template <int M>
__device__ __noinline__ void pass_feas_dense(const PassCtx& c) {
  const Plan& pl = *c.plan;
  const Problem& P = pl.P;
  const Cmd& cmd = *c.cmd;
  const double L = P.lower, U = P.upper;
  const int64_t n2 = P.n >> 1, st = c.stride, ld2 = P.ld >> 1;
  const double2* __restrict__ R2 = reinterpret_cast<const double2*>(P.rho);
  const double2* __restrict__ A2 = reinterpret_cast<const double2*>(P.grad);
  const volatile int* frow = cmd.feas_row;
  const volatile double* fy = cmd.feas_y;
  for (int f0 = 0; f0 < cmd.nfeas; f0 += FEAS_GROUP) {
    const int ng = cmd.nfeas - f0 < FEAS_GROUP ? cmd.nfeas - f0 : FEAS_GROUP;
    double acc[FEAS_GROUP][M];
#pragma unroll
    for (int g = 0; g < FEAS_GROUP; ++g)
#pragma unroll
      for (int k = 0; k < M; ++k) acc[g][k] = 0.0;
    auto one = [&](const double (&a)[M], double r) {
      const double lo = L - r, hi = U - r;
#pragma unroll
      for (int g = 0; g < FEAS_GROUP; ++g) {
        const int rj = g < ng ? frow[f0 + g] : -1;
        const double yj = g < ng ? fy[f0 + g] : 0.0;
        double z = 0.0;
        if (rj >= 0 && yj != 0.0) {
          double arj = 0.0;
#pragma unroll
          for (int k = 0; k < M; ++k)
            if (k == rj) arj = a[k];
          z = 0.0 + yj * arj;
        }
        const double dl = clipd(z, lo, hi);
#pragma unroll
        for (int k = 0; k < M; ++k) acc[g][k] += a[k] * dl;
      }
    };
    for (int64_t q = c.i0; q < n2; q += st) {
      double2 v2[M + 1];
      v2[0] = R2[q];
#pragma unroll
      for (int k = 0; k < M; ++k) v2[1 + k] = A2[(int64_t)k * ld2 + q];
      double a[M];
#pragma unroll
      for (int k = 0; k < M; ++k) a[k] = v2[1 + k].x;
      one(a, v2[0].x);
#pragma unroll
      for (int k = 0; k < M; ++k) a[k] = v2[1 + k].y;
      one(a, v2[0].y);
    }
#pragma unroll
    for (int g = 0; g < FEAS_GROUP; ++g)
      if (g < ng) block_reduce_store<M>(acc[g], M, PH_FEAS, (f0 + g) * M, c.out, c.smem);
  }
}

__device__ __noinline__ void pass_feas_pat7(const PassCtx& c);

__device__ __noinline__ void pass_feas(const PassCtx& c) {
  const Plan& pl = *c.plan;
  const Problem& P = pl.P;
  const Cmd& cmd = *c.cmd;
  const double L = P.lower, U = P.upper;
  const int m = P.m;
  const int64_t n = P.n, st = c.stride, ld = P.ld;
  const double* __restrict__ rho = P.rho;
  const double* __restrict__ grad = P.grad;
  if (m == 7 && !P.structured && (n & 1) == 0 && (ld & 1) == 0 && al16(rho) && al16(grad)) {
    if (P.pat7) pass_feas_pat7(c);
    else pass_feas_dense<7>(c);
    return;
  }
  if (m <= 8) {   // 16-byte pairs, FEAS_GROUP candidates per pass
    pass_feas_streamed(c);
    return;
  }
  for (int f = 0; f < cmd.nfeas; ++f) {
    const int rj = cmd.feas_row[f];
    const double yj = cmd.feas_y[f];
    double acc[MAX_M];
#pragma unroll
    for (int k = 0; k < MAX_M; ++k) acc[k] = 0.0;
    for (int64_t i = c.i0; i < n; i += st) {
      const double r = rho[i];
      const double lo = L - r, hi = U - r;
      double z = 0.0;
      if (rj >= 0 && yj != 0.0) z = 0.0 + yj * grad[(int64_t)rj * ld + i];
      const double dl = clipd(z, lo, hi);
#pragma unroll
      for (int k = 0; k < MAX_M; ++k)
        if (k < m) acc[k] += grad[(int64_t)k * ld + i] * dl;
    }
    block_reduce_store<MAX_M>(acc, m, PH_FEAS, f * m, c.out, c.smem);
  }
}

// ---- PH_NEWTON: delta(y), h-dots and the free-set Gram A D A^T ------------
// (eval_phi projection.cpp:279-298 and J_h projection.cpp:359-376)
//
// Register version: per thread the h-dots and the packed Gram triangle (M
// exact for m = 7: 28 accumulators); the rows come as 16-byte pairs
// (rows_pairs), two elements' loads in flight per thread.
// Dense rows, exact m = M (C4/C5): a register-lean copy of pass_newton_m's
// rows_pairs loop -- one base pointer for the rows and the duals re-read
// from the shared-memory command per element, so the m + m(m+1)/2
// accumulators and the m + 1 pair loads fit without spilling.  Same elements
// per thread in the same order and the same per-element arithmetic.
template <int M>
__device__ __noinline__ void pass_newton_dense(const PassCtx& c) {
  const Plan& pl = *c.plan;
  const Problem& P = pl.P;
  const Cmd& cmd = *c.cmd;
  const double L = P.lower, U = P.upper;
  const int64_t n = P.n, st = c.stride, ld = P.ld;
  const double* __restrict__ rho = P.rho;
  const double* __restrict__ grad = P.grad;
  const bool want_gram = cmd.want_gram;
  constexpr int NG = M * (M + 1) / 2;
  double h[M], G[NG];
#pragma unroll
  for (int k = 0; k < M; ++k) h[k] = 0.0;
#pragma unroll
  for (int k = 0; k < NG; ++k) G[k] = 0.0;
  const volatile double* ys = cmd.y;
  const double2* __restrict__ R2 = reinterpret_cast<const double2*>(rho);
  const double2* __restrict__ A2 = reinterpret_cast<const double2*>(grad);
  const int64_t n2 = n >> 1, ld2 = ld >> 1;
  auto one = [&](const double (&a)[M], double r) {
    const double lo = L - r, hi = U - r;
    double z = 0.0;
#pragma unroll
    for (int k = 0; k < M; ++k) {
      const double yk = ys[k];
      if (yk != 0.0) z += yk * a[k];
    }
    const bool clipped = (z < lo) || (z > hi);
    const double dl = clipd(z, lo, hi);
#pragma unroll
    for (int k = 0; k < M; ++k) h[k] += a[k] * dl;
    if (want_gram && !clipped) {
      int q = 0;
#pragma unroll
      for (int j = 0; j < M; ++j)
#pragma unroll
        for (int k = j; k < M; ++k) { G[q] = __fma_rn(a[j], a[k], G[q]); ++q; }
    }
  };
  for (int64_t q = c.i0; q < n2; q += st) {
    double2 v2[M + 1];
    v2[0] = R2[q];
#pragma unroll
    for (int k = 0; k < M; ++k) v2[1 + k] = A2[(int64_t)k * ld2 + q];
    double a[M];
#pragma unroll
    for (int k = 0; k < M; ++k) a[k] = v2[1 + k].x;
    one(a, v2[0].x);
#pragma unroll
    for (int k = 0; k < M; ++k) a[k] = v2[1 + k].y;
    one(a, v2[0].y);
  }
  double v[M + NG];
#pragma unroll
  for (int k = 0; k < M; ++k) v[k] = h[k];
#pragma unroll
  for (int k = 0; k < NG; ++k) v[M + k] = G[k];   // m = M: gram_idx is the packed order
  block_reduce_store<M + NG>(v, M + NG, PH_NEWTON, 0, c.out, c.smem);
}

// The C4/C5 row layout detected by PREP (P.pat7): row 0 constant (volume),
// rows 2, 4, 6 the exact negations of rows 1, 3, 5 (the two-sided centre-of-
// mass bands).  Only rho and rows 1, 3, 5 are read (32 instead of 64 bytes
// per element), h is accumulated for rows 0, 1, 3, 5 and the Gram for their
// 10 distinct products; the rest follow by exact sign flips:
// h_{2k} = -h_{2k-1}; G(j, k) = s_j s_k G(b_j, b_k) (an FMA chain with
// negated operands rounds to the negated value).  Bit-identical to
// pass_newton_dense<7> (same elements per thread, same order, same ops).
__device__ __forceinline__ int p7_base(int k) { return (k >= 2 && (k & 1) == 0) ? k - 1 : k; }
__device__ __forceinline__ bool p7_neg(int k) { return k >= 2 && (k & 1) == 0; }

__device__ __noinline__ void pass_newton_pat7(const PassCtx& c) {
  constexpr int M = 7;
  const Plan& pl = *c.plan;
  const Problem& P = pl.P;
  const Cmd& cmd = *c.cmd;
  const double L = P.lower, U = P.upper;
  const double a0 = P.alias_c[0];
  const bool want_gram = cmd.want_gram;
  constexpr int NB = 4;                 // distinct rows 0, 1, 3, 5
  double h[NB], G[NB * (NB + 1) / 2];
#pragma unroll
  for (int k = 0; k < NB; ++k) h[k] = 0.0;
#pragma unroll
  for (int k = 0; k < NB * (NB + 1) / 2; ++k) G[k] = 0.0;
  double ys[M];   // duals in registers (14 of the 28 doubles the dense kernel keeps)
#pragma unroll
  for (int k = 0; k < M; ++k) ys[k] = cmd.y[k];
  const double2* __restrict__ R2 = reinterpret_cast<const double2*>(P.rho);
  const double2* __restrict__ A2 = reinterpret_cast<const double2*>(P.grad);
  const int64_t n2 = P.n >> 1, st = c.stride, ld2 = P.ld >> 1;
  auto one = [&](double u, double v, double w, double r) {
    const double a[M] = {a0, u, -u, v, -v, w, -w};
    const double lo = L - r, hi = U - r;
    double z = 0.0;
#pragma unroll
    for (int k = 0; k < M; ++k) {
      const double yk = ys[k];
      if (yk != 0.0) z += yk * a[k];
    }
    const bool clipped = (z < lo) || (z > hi);
    const double dl = clipd(z, lo, hi);
    const double b[NB] = {a0, u, v, w};
#pragma unroll
    for (int k = 0; k < NB; ++k) h[k] += b[k] * dl;
    if (want_gram && !clipped) {
      int q = 0;
#pragma unroll
      for (int j = 0; j < NB; ++j)
#pragma unroll
        for (int k = j; k < NB; ++k) { G[q] = __fma_rn(b[j], b[k], G[q]); ++q; }
    }
  };
  // two pairs per thread in flight (8 x 16-byte loads): the pass is HBM-bound
  // only with enough bytes in flight per SM; same per-thread element order
  int64_t q = c.i0;
  const int64_t cta0 = c.i0 - threadIdx.x;
  for (; q + st < n2; q += 2 * st) {
    if (threadIdx.x == 0) {   // L2 prefetch of rho and rows 1, 3, 5, PF_AHEAD steps ahead
      const int64_t lim = n2 * 16;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int64_t off = (cta0 + (q - c.i0) + (int64_t)PF_AHEAD * 2 * st + u * st) * 16;
        prefetch_l2(R2, off, BLOCK * 16, lim);
        prefetch_l2(A2 + ld2, off, BLOCK * 16, lim);
        prefetch_l2(A2 + 3 * ld2, off, BLOCK * 16, lim);
        prefetch_l2(A2 + 5 * ld2, off, BLOCK * 16, lim);
      }
    }
    const double2 r2 = R2[q], u2 = A2[ld2 + q], v2 = A2[3 * ld2 + q], w2 = A2[5 * ld2 + q];
    const double2 r3 = R2[q + st], u3 = A2[ld2 + q + st], v3 = A2[3 * ld2 + q + st],
                  w3 = A2[5 * ld2 + q + st];
    one(u2.x, v2.x, w2.x, r2.x);
    one(u2.y, v2.y, w2.y, r2.y);
    one(u3.x, v3.x, w3.x, r3.x);
    one(u3.y, v3.y, w3.y, r3.y);
  }
  if (q < n2) {
    const double2 r2 = R2[q], u2 = A2[ld2 + q], v2 = A2[3 * ld2 + q], w2 = A2[5 * ld2 + q];
    one(u2.x, v2.x, w2.x, r2.x);
    one(u2.y, v2.y, w2.y, r2.y);
  }
  // expand to the m = 7 layout: slots [0, 7) h, [7, 35) packed Gram
  constexpr int NG = M * (M + 1) / 2;
  double vv[M + NG];
  const int bi[M] = {0, 1, 1, 2, 2, 3, 3};   // row -> distinct row
#pragma unroll
  for (int k = 0; k < M; ++k) vv[k] = p7_neg(k) ? -h[bi[k]] : h[bi[k]];
  int s = 0;
#pragma unroll
  for (int j = 0; j < M; ++j)
#pragma unroll
    for (int k = j; k < M; ++k) {
      const int x = bi[j] < bi[k] ? bi[j] : bi[k], y = bi[j] < bi[k] ? bi[k] : bi[j];
      const int gi = x * NB - x * (x - 1) / 2 + (y - x);
      vv[M + s] = (p7_neg(j) != p7_neg(k)) ? -G[gi] : G[gi];
      ++s;
    }
  block_reduce_store<M + NG>(vv, M + NG, PH_NEWTON, 0, c.out, c.smem);
}

// FEAS for the P.pat7 layout (see pass_newton_pat7): rho and rows 1, 3, 5.
__device__ __noinline__ void pass_feas_pat7(const PassCtx& c) {
  constexpr int M = 7, NB = 4;
  const Plan& pl = *c.plan;
  const Problem& P = pl.P;
  const Cmd& cmd = *c.cmd;
  const double L = P.lower, U = P.upper;
  const double a0 = P.alias_c[0];
  const int64_t n2 = P.n >> 1, st = c.stride, ld2 = P.ld >> 1;
  const double2* __restrict__ R2 = reinterpret_cast<const double2*>(P.rho);
  const double2* __restrict__ A2 = reinterpret_cast<const double2*>(P.grad);
  // cmd.feas_gram0: Newton's first evaluation (y = 0) rides on the first
  // group's sweep -- h-dots of clip(0, lo, hi) and the free-set Gram of the 4
  // distinct rows, exactly pass_newton_pat7's per-element arithmetic at y = 0
  double h0[NB], G0[NB * (NB + 1) / 2];
#pragma unroll
  for (int k = 0; k < NB; ++k) h0[k] = 0.0;
#pragma unroll
  for (int k = 0; k < NB * (NB + 1) / 2; ++k) G0[k] = 0.0;
  for (int f0 = 0; f0 < cmd.nfeas; f0 += FEAS_GROUP) {
    const bool gram0 = cmd.feas_gram0 && f0 == 0;
    const int ng = cmd.nfeas - f0 < FEAS_GROUP ? cmd.nfeas - f0 : FEAS_GROUP;
    int frow[FEAS_GROUP];     // the group's candidates in registers
    double fy[FEAS_GROUP];
#pragma unroll
    for (int g = 0; g < FEAS_GROUP; ++g) {
      frow[g] = g < ng ? cmd.feas_row[f0 + g] : -1;
      fy[g] = g < ng ? cmd.feas_y[f0 + g] : 0.0;
    }
    double acc[FEAS_GROUP][NB];
#pragma unroll
    for (int g = 0; g < FEAS_GROUP; ++g)
#pragma unroll
      for (int k = 0; k < NB; ++k) acc[g][k] = 0.0;
    auto one = [&](double u, double v, double w, double r) {
      const double a[M] = {a0, u, -u, v, -v, w, -w};
      const double b[NB] = {a0, u, v, w};
      const double lo = L - r, hi = U - r;
#pragma unroll
      for (int g = 0; g < FEAS_GROUP; ++g) {
        const int rj = frow[g];
        const double yj = fy[g];
        double z = 0.0;
        if (rj >= 0 && yj != 0.0) {
          double arj = 0.0;
#pragma unroll
          for (int k = 0; k < M; ++k)
            if (k == rj) arj = a[k];
          z = 0.0 + yj * arj;
        }
        const double dl = clipd(z, lo, hi);
#pragma unroll
        for (int k = 0; k < NB; ++k) acc[g][k] += b[k] * dl;
      }
      if (gram0) {
        const bool clipped = (0.0 < lo) || (0.0 > hi);
        const double dl = clipd(0.0, lo, hi);
#pragma unroll
        for (int k = 0; k < NB; ++k) h0[k] += b[k] * dl;
        if (!clipped) {
          int qq = 0;
#pragma unroll
          for (int j = 0; j < NB; ++j)
#pragma unroll
            for (int k = j; k < NB; ++k) { G0[qq] = __fma_rn(b[j], b[k], G0[qq]); ++qq; }
        }
      }
    };
    int64_t q = c.i0;
    for (; q + st < n2; q += 2 * st) {   // two pairs in flight (see pass_newton_pat7)
      const double2 r2 = R2[q], u2 = A2[ld2 + q], v2 = A2[3 * ld2 + q], w2 = A2[5 * ld2 + q];
      const double2 r3 = R2[q + st], u3 = A2[ld2 + q + st], v3 = A2[3 * ld2 + q + st],
                    w3 = A2[5 * ld2 + q + st];
      one(u2.x, v2.x, w2.x, r2.x);
      one(u2.y, v2.y, w2.y, r2.y);
      one(u3.x, v3.x, w3.x, r3.x);
      one(u3.y, v3.y, w3.y, r3.y);
    }
    if (q < n2) {
      const double2 r2 = R2[q], u2 = A2[ld2 + q], v2 = A2[3 * ld2 + q], w2 = A2[5 * ld2 + q];
      one(u2.x, v2.x, w2.x, r2.x);
      one(u2.y, v2.y, w2.y, r2.y);
    }
    const int bi[M] = {0, 1, 1, 2, 2, 3, 3};
#pragma unroll
    for (int g = 0; g < FEAS_GROUP; ++g) {
      if (g >= ng) continue;
      double vv[M];
#pragma unroll
      for (int k = 0; k < M; ++k) vv[k] = p7_neg(k) ? -acc[g][bi[k]] : acc[g][bi[k]];
      block_reduce_store<M>(vv, M, PH_FEAS, (f0 + g) * M, c.out, c.smem);
    }
  }
  if (cmd.feas_gram0) {   // expand to the m = 7 layout: 7 h-dots, then the packed 28-entry Gram
    constexpr int NG = M * (M + 1) / 2;
    const int bi[M] = {0, 1, 1, 2, 2, 3, 3};
    double vv[M + NG];
#pragma unroll
    for (int k = 0; k < M; ++k) vv[k] = p7_neg(k) ? -h0[bi[k]] : h0[bi[k]];
    int sidx = 0;
#pragma unroll
    for (int j = 0; j < M; ++j)
#pragma unroll
      for (int k = j; k < M; ++k) {
        const int x = bi[j] < bi[k] ? bi[j] : bi[k], y = bi[j] < bi[k] ? bi[k] : bi[j];
        const int gi = x * NB - x * (x - 1) / 2 + (y - x);
        vv[M + sidx] = (p7_neg(j) != p7_neg(k)) ? -G0[gi] : G0[gi];
        ++sidx;
      }
    block_reduce_store<M + NG>(vv, M + NG, PH_FEAS, cmd.nfeas * M, c.out, c.smem);
  }
}

template <int M>
__device__ __noinline__ void pass_newton_m(const PassCtx& c) {
  const Plan& pl = *c.plan;
  const Problem& P = pl.P;
  const Cmd& cmd = *c.cmd;
  const double L = P.lower, U = P.upper;
  const int m = P.m;
  const int64_t n = P.n, st = c.stride, ld = P.ld;
  const double* __restrict__ rho = P.rho;
  const double* __restrict__ grad = P.grad;
  const bool want_gram = cmd.want_gram;
  constexpr int NG = M * (M + 1) / 2;
  double h[M], G[NG], y[M];
#pragma unroll
  for (int k = 0; k < M; ++k) { h[k] = 0.0; y[k] = (k < m) ? cmd.y[k] : 0.0; }
#pragma unroll
  for (int k = 0; k < NG; ++k) G[k] = 0.0;
  auto elem = [&](const double (&a)[M], double r) {
    const double lo = L - r, hi = U - r;
    double z = 0.0;
#pragma unroll
    for (int k = 0; k < M; ++k)
      if (k < m && y[k] != 0.0) z += y[k] * a[k];
    const bool clipped = (z < lo) || (z > hi);
    const double dl = clipd(z, lo, hi);
#pragma unroll
    for (int k = 0; k < M; ++k) h[k] += a[k] * dl;
    if (want_gram && !clipped) {
      int q = 0;
#pragma unroll
      for (int j = 0; j < M; ++j)
#pragma unroll
        for (int k = j; k < M; ++k) { G[q] = __fma_rn(a[j], a[k], G[q]); ++q; }
    }
  };
  if (m + 1 <= RP_MAXR && M + 1 <= RP_MAXR) {
    StreamRows R;
    R.nr = m + 1;
    R.row[0] = rho;
    for (int k = 0; k < m; ++k) set_arow(R, 1 + k, c, P, k);
    rows_pairs<(M + 1 <= RP_MAXR ? M + 1 : RP_MAXR)>(c, R, n, [&](int64_t, const auto& v) {
      double a[M];
#pragma unroll
      for (int k = 0; k < M; ++k) a[k] = (k < m && k + 1 < RP_MAXR) ? v[1 + k] : 0.0;
      elem(a, v[0]);
    });
  } else {
    for (int64_t i = c.i0; i < n; i += st) {
      double a[M];
#pragma unroll
      for (int k = 0; k < M; ++k) a[k] = (k < m) ? grad[(int64_t)k * ld + i] : 0.0;
      elem(a, rho[i]);
    }
  }
  // pack: slots [0, m) h ; [m, m + m(m+1)/2) upper-triangle of the m x m Gram
  double v[M + NG];
#pragma unroll
  for (int k = 0; k < M; ++k) v[k] = h[k];
  {
    int q = 0;
#pragma unroll
    for (int j = 0; j < M; ++j)
#pragma unroll
      for (int k = j; k < M; ++k) {
        if (j < m && k < m) v[m + gram_idx(m, j, k)] = G[q];
        ++q;
      }
  }
  block_reduce_store<M + NG>(v, m + m * (m + 1) / 2, PH_NEWTON, 0, c.out, c.smem);
}

// ---- PH_FINAL: delta / x_{t+1} / mask writes and residual dots ------------
// M: compile-time row bound (>= m); OWN: partition owner map present.
template <int M, bool OWN>
__device__ __noinline__ void pass_final_m(const PassCtx& c) {
  const Plan& pl = *c.plan;
  const Problem& P = pl.P;
  const Cmd& cmd = *c.cmd;
  const double L = P.lower, Up = P.upper;
  const int m = P.m;
  const int64_t n = P.n, st = c.stride, ld = P.ld;
  const double* __restrict__ rho = P.rho;
  const double* __restrict__ grad = P.grad;
  const int8_t* __restrict__ owner = P.owner;
  double* __restrict__ dout = cmd.write_delta ? P.delta_out : nullptr;
  double* __restrict__ xout = cmd.write_x ? P.x_out : nullptr;
  uint8_t* __restrict__ mout = cmd.write_mask ? P.mask_out : nullptr;
  const bool resid = cmd.resid_rows;
  double yv[M], acc[M];
#pragma unroll
  for (int k = 0; k < M; ++k) { yv[k] = (k < m) ? cmd.y[k] : 0.0; acc[k] = 0.0; }
  if (!OWN && M + 1 <= RP_MAXR && (n & 1) == 0) {
    // 16-byte pairs in and out (x_{t+1} / delta as double2, the mask as 2 bytes)
    bool vec = al16(rho) && (!dout || al16(dout)) && (!xout || al16(xout)) &&
               (!mout || (reinterpret_cast<uintptr_t>(mout) & 1u) == 0);
    const double* rows[M];
#pragma unroll
    for (int k = 0; k < M; ++k) {
      const bool gen = k < m && P.structured && P.row_kind[k] != RK_DENSE;
      rows[k] = (k < m && !gen) ? grad + (int64_t)k * ld : rho;
      vec = vec && al16(rows[k]);
    }
    if (vec) {
      const int64_t n2 = n >> 1;
      auto one = [&](double r, const double (&a)[M], bool& below, bool& above) {
        double z = 0.0;
#pragma unroll
        for (int k = 0; k < M; ++k)
          if (k < m && yv[k] != 0.0) z += yv[k] * a[k];
        const double lo = L - r, hi = Up - r;
        below = z < lo; above = z > hi;
        const double dl = below ? lo : (above ? hi : z);
        if (resid) {
#pragma unroll
          for (int k = 0; k < M; ++k)
            if (k < m) acc[k] += a[k] * dl;
        }
        return dl;
      };
      const bool sr = P.structured;
      const GridIx G = grid_ix(P);
      int scode[M], ak[M];
      bool need[M];
#pragma unroll
      for (int k = 0; k < M; ++k) {
        scode[k] = (sr && k < m && P.row_kind[k] != RK_DENSE) ? srow_code(P, k) : -1;
        ak[k] = (P.n_alias && k < m) ? P.alias_kind[k] : AK_DENSE;
        need[k] = k < m && (resid || yv[k] != 0.0);   // rows with y_k = 0: no read
      }
#pragma unroll
      for (int k = M - 1; k >= 1; --k)   // a negated row reads its predecessor
        if (ak[k] == AK_NEG && need[k]) need[k - 1] = true;
      // loads of one element pair; derived rows filled in (exact copies)
      auto load = [&](int64_t q, double2& r2, double2 (&a2)[M]) {
        r2 = reinterpret_cast<const double2*>(rho)[q];
#pragma unroll
        for (int k = 0; k < M; ++k)
          a2[k] = (need[k] && scode[k] < 0 && ak[k] == AK_DENSE)
                      ? reinterpret_cast<const double2*>(rows[k])[q] : make_double2(0.0, 0.0);
      };
      auto finish = [&](int64_t q, const double2 r2, double2 (&a2)[M]) {
#pragma unroll
        for (int k = 0; k < M; ++k) {   // structure found by PREP: exact copies
          if (ak[k] == AK_CONST) a2[k] = make_double2(P.alias_c[k], P.alias_c[k]);
          if (k > 0 && ak[k] == AK_NEG) a2[k] = make_double2(-a2[k - 1].x, -a2[k - 1].y);
        }
        if (sr) {   // structured rows: generated from the element coordinates
          int64_t c0[3], c1[3];
          grid_coords(G, 2 * q + G.off, c0);
          grid_coords(G, 2 * q + 1 + G.off, c1);
#pragma unroll
          for (int k = 0; k < M; ++k)
            if (scode[k] >= 0)
              a2[k] = make_double2(srow_fetch(c.rtab, scode[k], c0), srow_fetch(c.rtab, scode[k], c1));
        }
        double ax[M], ay[M];
#pragma unroll
        for (int k = 0; k < M; ++k) { ax[k] = a2[k].x; ay[k] = a2[k].y; }
        bool b0, u0, b1, u1;
        const double d0 = one(r2.x, ax, b0, u0);
        const double d1 = one(r2.y, ay, b1, u1);
        if (dout) reinterpret_cast<double2*>(dout)[q] = make_double2(d0, d1);
        if (xout) reinterpret_cast<double2*>(xout)[q] = make_double2(r2.x + d0, r2.y + d1);
        if (mout) {
          uchar2 mk;
          mk.x = b0 ? 1 : (u0 ? 2 : 0);
          mk.y = b1 ? 1 : (u1 ? 2 : 0);
          reinterpret_cast<uchar2*>(mout)[q] = mk;
        }
      };
      int64_t q = c.i0;
      // two pairs' loads in flight per thread where the registers allow it
      // (m = 7 / 8 would spill: pass_final_pat7 covers the C4/C5 layout)
      if (M <= 4)
        for (; q + st < n2; q += 2 * st) {
          double2 r2, r3, a2[M], a3[M];
          load(q, r2, a2);
          load(q + st, r3, a3);
          finish(q, r2, a2);
          finish(q + st, r3, a3);
        }
      for (; q < n2; q += st) {
        double2 r2, a2[M];
        load(q, r2, a2);
        finish(q, r2, a2);
      }
      if (resid) block_reduce_store<M>(acc, m, PH_FINAL, 0, c.out, c.smem);
      return;
    }
  }
  for (int64_t i = c.i0; i < n; i += st) {
    const double r = rho[i];
    double z = 0.0;
    int o = -1;
    if (OWN) {
      o = owner[i];
      double yo = 0.0;
#pragma unroll
      for (int k = 0; k < M; ++k)
        if (k == o) yo = yv[k];
      if (o >= 0 && yo != 0.0) z = 0.0 + yo * grad[(int64_t)o * ld + i];
    } else {
#pragma unroll
      for (int k = 0; k < M; ++k)
        if (k < m && yv[k] != 0.0) z += yv[k] * grad[(int64_t)k * ld + i];
    }
    const double lo = L - r, hi = Up - r;
    const bool below = z < lo, above = z > hi;
    const double dl = below ? lo : (above ? hi : z);
    if (dout) dout[i] = dl;
    if (xout) xout[i] = r + dl;
    if (mout) mout[i] = below ? 1 : (above ? 2 : 0);
    if (resid) {
      if (OWN) {
        if (o >= 0) {
          const double t = grad[(int64_t)o * ld + i] * dl;
#pragma unroll
          for (int k = 0; k < M; ++k)
            if (k == o) acc[k] += t;
        }
      } else {
#pragma unroll
        for (int k = 0; k < M; ++k)
          if (k < m) acc[k] += grad[(int64_t)k * ld + i] * dl;
      }
    }
  }
  if (resid) block_reduce_store<M>(acc, m, PH_FINAL, 0, c.out, c.smem);
}

// FINAL for the P.pat7 layout (see pass_newton_pat7): rho and rows 1, 3, 5
// (the rows of the dual's non-zero entries only, unless residuals are
// wanted); x_{t+1} / delta / mask as 16-byte pairs, two pairs in flight.
__device__ __noinline__ void pass_final_pat7(const PassCtx& c) {
  constexpr int M = 7;
  const Plan& pl = *c.plan;
  const Problem& P = pl.P;
  const Cmd& cmd = *c.cmd;
  const double L = P.lower, Up = P.upper;
  const double a0 = P.alias_c[0];
  const int64_t n2 = P.n >> 1, st = c.stride, ld2 = P.ld >> 1;
  const double2* __restrict__ R2 = reinterpret_cast<const double2*>(P.rho);
  const double2* __restrict__ A2 = reinterpret_cast<const double2*>(P.grad);
  double2* __restrict__ DO = cmd.write_delta ? reinterpret_cast<double2*>(P.delta_out) : nullptr;
  double2* __restrict__ XO = cmd.write_x ? reinterpret_cast<double2*>(P.x_out) : nullptr;
  uchar2* __restrict__ MO = cmd.write_mask ? reinterpret_cast<uchar2*>(P.mask_out) : nullptr;
  const bool resid = cmd.resid_rows;
  double yv[M];
#pragma unroll
  for (int k = 0; k < M; ++k) yv[k] = cmd.y[k];
  // base rows 1, 3, 5 are read when their pair has a non-zero dual
  const bool nu = resid || yv[1] != 0.0 || yv[2] != 0.0;
  const bool nv = resid || yv[3] != 0.0 || yv[4] != 0.0;
  const bool nw = resid || yv[5] != 0.0 || yv[6] != 0.0;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  auto one = [&](double r, double u, double v, double w, bool& below, bool& above) {
    const double a[M] = {a0, u, -u, v, -v, w, -w};
    double z = 0.0;
#pragma unroll
    for (int k = 0; k < M; ++k)
      if (yv[k] != 0.0) z += yv[k] * a[k];
    const double lo = L - r, hi = Up - r;
    below = z < lo; above = z > hi;
    const double dl = below ? lo : (above ? hi : z);
    if (resid) {
      acc[0] += a0 * dl; acc[1] += u * dl; acc[2] += v * dl; acc[3] += w * dl;
    }
    return dl;
  };
  auto put = [&](int64_t q, double2 r2, double2 u2, double2 v2, double2 w2) {
    bool b0, o0, b1, o1;
    const double d0 = one(r2.x, u2.x, v2.x, w2.x, b0, o0);
    const double d1 = one(r2.y, u2.y, v2.y, w2.y, b1, o1);
    if (DO) DO[q] = make_double2(d0, d1);
    if (XO) XO[q] = make_double2(r2.x + d0, r2.y + d1);
    if (MO) {
      uchar2 mk;
      mk.x = b0 ? 1 : (o0 ? 2 : 0);
      mk.y = b1 ? 1 : (o1 ? 2 : 0);
      MO[q] = mk;
    }
  };
  const double2 z2 = make_double2(0.0, 0.0);
  int64_t q = c.i0;
  for (; q + st < n2; q += 2 * st) {
    const double2 r2 = R2[q], r3 = R2[q + st];
    const double2 u2 = nu ? A2[ld2 + q] : z2, u3 = nu ? A2[ld2 + q + st] : z2;
    const double2 v2 = nv ? A2[3 * ld2 + q] : z2, v3 = nv ? A2[3 * ld2 + q + st] : z2;
    const double2 w2 = nw ? A2[5 * ld2 + q] : z2, w3 = nw ? A2[5 * ld2 + q + st] : z2;
    put(q, r2, u2, v2, w2);
    put(q + st, r3, u3, v3, w3);
  }
  if (q < n2)
    put(q, R2[q], nu ? A2[ld2 + q] : z2, nv ? A2[3 * ld2 + q] : z2, nw ? A2[5 * ld2 + q] : z2);
  if (resid) {
    double vv[M] = {acc[0], acc[1], -acc[1], acc[2], -acc[2], acc[3], -acc[3]};
    block_reduce_store<M>(vv, M, PH_FINAL, 0, c.out, c.smem);
  }
}

// FINAL for a contiguous-range partition: row j's range as 16-byte pairs
// (z = 0.0 + y_j a_j, the OWN path's expression), then the elements in no
// set (owner -1, z = 0) if the ranges do not cover the slab.
__device__ __noinline__ void pass_final_ranges(const PassCtx& c) {
  const Problem& P = c.plan->P;
  const Cmd& cmd = *c.cmd;
  const double L = P.lower, Up = P.upper;
  const int m = P.m;
  const int64_t n = P.n, st = c.stride, ld = P.ld;
  const double* __restrict__ rho = P.rho;
  double* __restrict__ dout = cmd.write_delta ? P.delta_out : nullptr;
  double* __restrict__ xout = cmd.write_x ? P.x_out : nullptr;
  uint8_t* __restrict__ mout = cmd.write_mask ? P.mask_out : nullptr;
  const bool resid = cmd.resid_rows;
  double acc[MAX_M];
#pragma unroll
  for (int k = 0; k < MAX_M; ++k) acc[k] = 0.0;
  auto one = [&](int64_t i, double r, double a, double yj, double& accj) {
    const double z = (yj != 0.0) ? 0.0 + yj * a : 0.0;
    const double lo = L - r, hi = Up - r;
    const bool below = z < lo, above = z > hi;
    const double dl = below ? lo : (above ? hi : z);
    if (dout) dout[i] = dl;
    if (xout) xout[i] = r + dl;
    if (mout) mout[i] = below ? 1 : (above ? 2 : 0);
    if (resid) accj += a * dl;
  };
  int64_t covered = 0;
  for (int j = 0; j < m; ++j) {
    const int64_t b = P.row_lo[j], e = P.row_hi[j];
    covered += e - b;
    const double yj = cmd.y[j];
    const double* __restrict__ a = P.grad + (int64_t)j * ld;
    double accj = 0.0;
    const bool need_a = resid || yj != 0.0;
    if (((b | e) & 1) == 0 && al16(rho) && al16(a) && (!dout || al16(dout)) &&
        (!xout || al16(xout)) && !mout) {
      const double2* __restrict__ R2 = reinterpret_cast<const double2*>(rho);
      const double2* __restrict__ A2 = reinterpret_cast<const double2*>(a);
      for (int64_t q = (b >> 1) + c.i0; q < (e >> 1); q += st) {
        const double2 r2 = R2[q];
        const double2 a2 = need_a ? A2[q] : make_double2(0.0, 0.0);
        double d[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const double r = h ? r2.y : r2.x, av = h ? a2.y : a2.x;
          const double z = (yj != 0.0) ? 0.0 + yj * av : 0.0;
          const double lo = L - r, hi = Up - r;
          d[h] = z < lo ? lo : (z > hi ? hi : z);
          if (resid) accj += av * d[h];
        }
        if (dout) reinterpret_cast<double2*>(dout)[q] = make_double2(d[0], d[1]);
        if (xout) reinterpret_cast<double2*>(xout)[q] = make_double2(r2.x + d[0], r2.y + d[1]);
      }
    } else {
      for (int64_t i = b + c.i0; i < e; i += st) one(i, rho[i], need_a ? a[i] : 0.0, yj, accj);
    }
#pragma unroll
    for (int k = 0; k < MAX_M; ++k)
      if (k == j) acc[k] = accj;
  }
  if (covered < n) {   // elements in no set: delta = clip(0, lo, hi)
    const int8_t* __restrict__ owner = P.owner;
    double dummy = 0.0;
    for (int64_t i = c.i0; i < n; i += st)
      if (owner[i] < 0) one(i, rho[i], 0.0, 0.0, dummy);
  }
  if (resid) block_reduce_store<MAX_M>(acc, m, PH_FINAL, 0, c.out, c.smem);
}

__device__ void pass_final(const PassCtx& c) {
  const int m = c.plan->P.m;
  const bool own = c.plan->P.owner != nullptr;
  if (own && c.plan->P.part_ranges) { pass_final_ranges(c); return; }
  if (!own && m == 7) {
    const Problem& P = c.plan->P;
    if (P.pat7 && (P.n & 1) == 0 && (P.ld & 1) == 0 && al16(P.rho) && al16(P.grad) &&
        (!c.cmd->write_delta || al16(P.delta_out)) && (!c.cmd->write_x || al16(P.x_out)) &&
        (!c.cmd->write_mask || (reinterpret_cast<uintptr_t>(P.mask_out) & 1u) == 0))
      pass_final_pat7(c);
    else
      pass_final_m<7, false>(c);
    return;
  }
  if (own) {
    if (m <= 4) pass_final_m<4, true>(c);
    else if (m <= 8) pass_final_m<8, true>(c);
    else pass_final_m<16, true>(c);
  } else {
    if (m <= 1) pass_final_m<1, false>(c);
    else if (m <= 2) pass_final_m<2, false>(c);
    else if (m <= 4) pass_final_m<4, false>(c);
    else if (m <= 8) pass_final_m<8, false>(c);
    else pass_final_m<16, false>(c);
  }
}

__device__ void pass_newton(const PassCtx& c) {
  const int m = c.plan->P.m;
  if (m == 7) {
    const Problem& P = c.plan->P;
    if (!P.structured && (P.n & 1) == 0 && (P.ld & 1) == 0 && al16(P.rho) && al16(P.grad)) {
      if (P.pat7) pass_newton_pat7(c);
      else pass_newton_dense<7>(c);
    }
    else
      pass_newton_m<7>(c);
    return;
  }
  if (m <= 1) pass_newton_m<1>(c);
  else if (m <= 2) pass_newton_m<2>(c);
  else if (m <= 4) pass_newton_m<4>(c);
  else if (m <= 8) pass_newton_m<8>(c);
  else pass_newton_m<16>(c);
}

// ---- PH_EXACT: reference-order sequential sums (strict parity) -------------
//
// A reference sum s = fl(...fl(fl(start + t_0) + t_1)... + t_{L-1}) cannot be
// reassociated, so it runs as a CHAIN: one lane per sum, one dependent fp64
// add per element (~8 cycles, the DADD latency).  The pass interleaves two
// roles per segment of SEG elements of the element sequence:
//   * fill (CTAs 1..nb-1, grid-stride, full bandwidth): every element's terms
//     of every chain, with the reference's expressions, into T[p][NCp]
//     (double-buffered in global memory);
//   * consume (CTA 0): one thread streams the previous segment's T through a
//     shared-memory ring with 1-D TMA bulk copies (cp.async.bulk + mbarrier
//     complete_tx); consumer warps add one staged term per lane per element.
// Every term is a separately rounded IEEE product (__dmul_rn / __dadd_rn),
// so the chain reproduces the reference binary's sum bit for bit.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  unsigned ok = 0;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                 " selp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(smem_u32(b)), "r"(parity) : "memory");
  } while (!ok);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(b)) : "memory");
}

constexpr int EX_CHUNK_BYTES = 16384;

// Element index of position q of the pass's sequence.
__device__ __forceinline__ int64_t ex_elem(const Problem& P, int seq, int64_t q) {
  if (seq < 0) return q;
  if (P.part_ranges) return P.row_lo[seq] + q;
  return (int64_t)P.part_idx[P.part_off[seq] + q];
}
__device__ __forceinline__ int64_t ex_len(const Problem& P, int seq) {
  if (seq < 0) return P.n;
  if (P.part_ranges) return P.row_hi[seq] - P.row_lo[seq];
  return P.part_off[seq + 1] - P.part_off[seq];
}

// Terms of every chain at element i (the reference's expressions).
__device__ __forceinline__ void ex_terms(const Problem& P, const Cmd& cmd, int64_t i,
                                         double* __restrict__ out) {
  const int m = P.m;
  const double* __restrict__ A = P.grad;
  const int64_t ld = P.ld;
  double lo = 0.0, hi = 0.0, delta = 0.0;
  bool freev = false;
  const bool need_rho = cmd.ex_what != EXW_STEP && cmd.ex_what != EXW_GHAT;
  if (need_rho) {
    const double r = P.rho[i];
    lo = __dsub_rn(P.lower, r);            // projection.cpp:32, :207
    hi = __dsub_rn(P.upper, r);
  }
  if (cmd.ex_what == EXW_NEWTON || cmd.ex_what == EXW_RESH) {
    double z = 0.0;                        // projection.cpp:199-205: ascending j from 0.0
    for (int j = 0; j < m; ++j) {
      const double yj = cmd.y[j];
      if (yj == 0.0) continue;
      z = __dadd_rn(z, __dmul_rn(yj, A[(int64_t)j * ld + i]));
    }
    delta = clipd(z, lo, hi);
    freev = !(z < lo || z > hi);           // projection.cpp:369
  }
  double sx = 0.0, sy = 0.0, gg = 0.0, gp = 0.0, gd = 0.0;
  if (cmd.ex_what == EXW_STEP) {
    const double x = P.x[i], xp = P.x_prev[i];
    gg = P.g[i];
    gp = P.g_prev[i];
    sx = __dsub_rn(x, xp);
    sy = __dsub_rn(gg, gp);
  } else if (cmd.ex_what == EXW_GHAT) {
    gd = P.gd_step ? P.gd_step[i] : __dmul_rn(cmd.wa, P.d_out[i]);   // oracle.c: wa * d
  }
  for (int q = 0; q < cmd.ex_n; ++q) {
    const ExChain& e = cmd.ex[q];
    double t;
    switch (e.kind) {
      case CH_RESID: {
        const double a = A[(int64_t)e.j * ld + i];
        t = __dmul_rn(a, clipd(__dmul_rn(e.y, a), lo, hi));
        break;
      }
      case CH_DOTZ:
        t = __dmul_rn(A[(int64_t)e.k * ld + i], delta);
        break;
      case CH_GRAM:
        t = freev ? __dmul_rn(A[(int64_t)e.j * ld + i], A[(int64_t)e.k * ld + i]) : 0.0;
        break;
      case CH_FEAS: {
        const double z = e.j < 0 ? 0.0 : __dadd_rn(0.0, __dmul_rn(e.y, A[(int64_t)e.j * ld + i]));
        t = __dmul_rn(A[(int64_t)e.k * ld + i], clipd(z, lo, hi));
        break;
      }
      case CH_GHAT:
        t = __dmul_rn(gd, A[(int64_t)e.j * ld + i]);
        break;
      default: {   // CH_STEP, oracle.c orc_spectral_step_size / orc_pr_beta
        const int k = e.k;
        t = k == 0 ? __dmul_rn(sx, sx)
          : k == 1 ? __dmul_rn(sx, sy)
          : k == 2 ? __dmul_rn(sy, sy)
          : k == 3 ? __dmul_rn(gg, sy)
                   : __dmul_rn(gp, gp);
        break;
      }
    }
    out[q] = t;
  }
}

__device__ __noinline__ void pass_exact(const PassCtx& c) {
  const Problem& P = c.plan->P;
  const Cmd& cmd = *c.cmd;
  cg::grid_group grid = cg::this_grid();
  const int nc = cmd.ex_n;
  if (nc <= 0) return;                           // (uniform: no barrier skipped)
  const int NCp = (nc + 1) & ~1;                 // 16-byte rows
  const int seq = cmd.ex_seq;
  const int64_t L = ex_len(P, seq);
  const int64_t SEG = P.ex_seg;
  const int S = (int)((L + SEG - 1) / SEG);
  const int nb = gridDim.x;
  // consumer side (CTA 0): ring in dynamic shared memory
  const int NST = P.ex_nst;
  char* ring = reinterpret_cast<char*>(c.ex_smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + (size_t)NST * EX_CHUNK_BYTES);
  uint64_t* empty = full + NST;
  const int ncw = (nc + 31) / 32;                // consumer warps
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int CE = EX_CHUNK_BYTES / (NCp * 8);     // elements per chunk
  double acc = 0.0;
  const int my = warp * 32 + lane;
  if (blockIdx.x == 0) {
    if (warp < ncw && my < nc) acc = cmd.ex[my].start;
    if (threadIdx.x == 0) {
      for (int k = 0; k < NST; ++k) { mbar_init(full + k, 1); mbar_init(empty + k, ncw); }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
  }
  int stage = 0;
  unsigned phase = 0;
  for (int s = 0; s <= S; ++s) {
    if (blockIdx.x != 0 && s < S) {              // fill segment s
      double* T = P.ex_buf + (size_t)(s & 1) * (size_t)SEG * NCp;
      const int64_t q0 = (int64_t)s * SEG;
      const int64_t len = (L - q0 < SEG) ? L - q0 : SEG;
      for (int64_t p = (int64_t)(blockIdx.x - 1) * BLOCK + threadIdx.x; p < len;
           p += (int64_t)(nb - 1) * BLOCK)
        ex_terms(P, cmd, ex_elem(P, seq, q0 + p), T + (size_t)p * NCp);
      asm volatile("fence.proxy.async.global;" ::: "memory");   // generic writes -> TMA reads
    }
    if (blockIdx.x == 0 && s > 0) {              // consume segment s - 1
      const double* T = P.ex_buf + (size_t)((s - 1) & 1) * (size_t)SEG * NCp;
      const int64_t q0 = (int64_t)(s - 1) * SEG;
      const int64_t len = (L - q0 < SEG) ? L - q0 : SEG;
      const int64_t nch = (len + CE - 1) / CE;
      if (warp == ncw) {                         // TMA producer (one lane)
        if (lane == 0) {
          // the segment was written through the generic proxy by other CTAs
          // (ordered by the grid barrier): order it before these async-proxy reads
          asm volatile("fence.proxy.async.global;" ::: "memory");
          int st = stage;
          unsigned ph = phase;
          for (int64_t k = 0; k < nch; ++k) {
            mbar_wait(empty + st, ph ^ 1u);
            const int64_t e0 = k * CE;
            const int ne = (int)((len - e0 < CE) ? len - e0 : CE);
            const unsigned bytes = (unsigned)(ne * NCp * 8);
            mbar_expect_tx(full + st, bytes);
            bulk_g2s(ring + (size_t)st * EX_CHUNK_BYTES, T + (size_t)e0 * NCp, bytes, full + st);
            if (++st == NST) { st = 0; ph ^= 1u; }
          }
        }
      } else if (warp < ncw) {                   // consumers: lane = chain
        int st = stage;
        unsigned ph = phase;
        for (int64_t k = 0; k < nch; ++k) {
          mbar_wait(full + st, ph);
          const int64_t e0 = k * CE;
          const int ne = (int)((len - e0 < CE) ? len - e0 : CE);
          const double* buf = reinterpret_cast<const double*>(ring + (size_t)st * EX_CHUNK_BYTES) +
                              (my < NCp ? my : 0);
          int e = 0;
          for (; e + 8 <= ne; e += 8) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = buf[(size_t)(e + u) * NCp];
#pragma unroll
            for (int u = 0; u < 8; ++u) acc = __dadd_rn(acc, v[u]);
          }
          for (; e < ne; ++e) acc = __dadd_rn(acc, buf[(size_t)e * NCp]);
          __syncwarp();
          if (lane == 0) mbar_arrive(empty + st);
          if (++st == NST) { st = 0; ph ^= 1u; }
        }
      }
      // every role advanced the ring by nch chunks
      const int64_t adv = stage + nch;
      phase ^= (unsigned)((adv / NST) & 1);
      stage = (int)(adv % NST);
    }
    grid.sync();
  }
  if (blockIdx.x == 0) {
    if (warp < ncw && my < nc) c.out[my] = acc;
    // every chunk was consumed (the grid barrier above): retire the barriers,
    // the next chain pass initializes them afresh
    if (threadIdx.x == 0)
      for (int k = 0; k < NST; ++k) {
        asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(full + k)) : "memory");
        asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(empty + k)) : "memory");
      }
    __syncthreads();
  }
}

__device__ void run_pass(const PassCtx& c) {
  switch (c.cmd->phase) {
    case PH_STEP_REDUCE: pass_step_reduce(c); break;
    case PH_PREP: pass_prep(c); break;
    case PH_SWEEP: pass_sweep(c); break;
    case PH_FEAS: pass_feas(c); break;
    case PH_NEWTON: pass_newton(c); break;
    case PH_FINAL: pass_final(c); break;
    case PH_GATHER: pass_gather(c); break;
    case PH_EXACT: pass_exact(c); break;
    default: break;
  }
}

}  // namespace topt_b200
