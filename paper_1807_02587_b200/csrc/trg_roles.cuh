// Roles inside a persistent grid.
//
// The registration EM and the leaf calibration alternate a wide, FP64-heavy
// point pass (every point's tree descent) with a short chain of serial
// latency-bound math (3x3 eigensolves and moment matches, the 6x6 solve).
// Run on the same SMs, that chain always starts with a cold instruction
// cache (the point pass evicted it: a leaf refit measured ~10 us instead of
// ~1.2 us warm).  So the grid is split by SM: the CTAs of the lowest
// `upd_sms` SMs are UPDATERS -- they never run the point pass, keep the
// serial code resident, and synchronise among themselves with a small group
// barrier -- while every other CTA is a WORKER that only runs point passes.
// The two sides hand over with one counter and one flag per step instead of
// two grid-wide barriers:
//   workers:  wait flag >= step  ->  point pass  ->  fence, arrive (+1)
//   updaters: wait arrivals == n_work * (step + 1)  ->  serial math  ->
//             fence, flag = step + 1
// (counter/flag updates are GPU-scope releases, the waits acquire loads,
// which also drop stale L1 lines, as in grid_sync).
#pragma once
#include "trg_solve.cuh"

namespace trg {

struct Roles {
  bool upd;    // this CTA is an updater
  int idx;     // index among its role (CTA order)
  int n_upd, n_work;
};

__device__ __forceinline__ unsigned sm_id() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

// Every CTA registers its SM in smtab[G]; after a grid barrier each CTA
// derives the same role table: updaters are the CTAs on the `upd_sms`
// lowest-numbered SMs present (at least one CTA).  Block-wide; `bar` is
// the grid barrier of the launch.
static __device__ Roles assign_roles(unsigned* smtab, unsigned* bar, int G, int upd_sms) {
  __shared__ unsigned present[8];  // SM bitmap (<= 256 SMs)
  __shared__ int s_cut, s_nu, s_idx;
  const int tid = threadIdx.x;
  if (tid == 0) smtab[blockIdx.x] = sm_id();
  if (tid < 8) present[tid] = 0u;
  grid_sync(bar, G);
  for (int c = tid; c < G; c += blockDim.x) {
    const unsigned s = __ldcg(&smtab[c]) & 255u;
    atomicOr(&present[s >> 5], 1u << (s & 31));
  }
  __syncthreads();
  if (tid == 0) {
    // cut = the smallest SM id that is NOT an updater SM
    int seen = 0, cut = 256;
    for (int s = 0; s < 256 && cut == 256; ++s)
      if ((present[s >> 5] >> (s & 31)) & 1u) {
        if (seen == upd_sms) cut = s;
        ++seen;
      }
    // (fewer SMs than upd_sms: cut stays 256, every CTA is an updater, and
    // the single-SM fallback below applies)
    s_cut = cut;
  }
  __syncthreads();
  const unsigned cut = (unsigned)s_cut;
  int nu = 0, before = 0;
  const unsigned mine = __ldcg(&smtab[blockIdx.x]) & 255u;
  const bool upd = mine < cut;
  for (int c = tid; c < G; c += blockDim.x) {
    const bool u = (__ldcg(&smtab[c]) & 255u) < cut;
    nu += u;
    if (c < (int)blockIdx.x && u == upd) ++before;
  }
  if (tid == 0) {
    s_nu = 0;
    s_idx = 0;
  }
  __syncthreads();
  if (nu) atomicAdd(&s_nu, nu);
  if (before) atomicAdd(&s_idx, before);
  __syncthreads();
  Roles r;
  r.n_upd = s_nu;
  r.n_work = G - s_nu;
  r.upd = upd;
  r.idx = s_idx;
  if (r.n_work == 0) {  // one SM only: CTA 0 updates, the rest work
    r.upd = blockIdx.x == 0;
    r.idx = r.upd ? 0 : (int)blockIdx.x - 1;
    r.n_upd = 1;
    r.n_work = G - 1;
  }
  __syncthreads();
  return r;
}

// Roles of a CTA group by index (one launch running several independent
// groups): the group's CTA 0 updates, the rest work.  Block-wide; the group
// barrier orders what the CTAs wrote before the call.
static __device__ Roles roles_by_index(unsigned* bar, int G, int cta) {
  grid_sync(bar, G);
  Roles r;
  r.upd = cta == 0;
  r.idx = r.upd ? 0 : cta - 1;
  r.n_upd = 1;
  r.n_work = G - 1;
  return r;
}

// Workers: wait until the updaters published step `s` (flag >= s).
__device__ __forceinline__ void wait_flag(const unsigned* flag, unsigned s) {
  __syncthreads();
  if (threadIdx.x == 0 && ld_acquire_u32(flag) < s) {
    unsigned ns = 32, polls = 0;
    const unsigned long long t0 = gtimer();
    while (ld_acquire_u32(flag) < s) {
      __nanosleep(ns);
      ns = ns < 128 ? 2 * ns : 128;
      spin_guard_every(t0, polls);
    }
  }
  __syncthreads();
}

// Updaters: wait until `target` worker arrivals are counted.
__device__ __forceinline__ void wait_count(const unsigned* cnt, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0 && ld_acquire_u32(cnt) < target) {
    const unsigned long long t0 = gtimer();
    unsigned polls = 0;
    while (ld_acquire_u32(cnt) < target) {
      __nanosleep(32);
      spin_guard_every(t0, polls);
    }
  }
  __syncthreads();
}

// Workers: this CTA's point pass is complete (all its threads' writes and
// reductions are ordered before the arrival by the CTA barrier; the release
// publishes them).
__device__ __forceinline__ void arrive_count(unsigned* cnt) {
  __syncthreads();
  if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
}

// Updater 0: publish step s (its CTA's writes ordered before by the caller).
__device__ __forceinline__ void publish_flag(unsigned* flag, unsigned s) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flag), "r"(s) : "memory");
}

}  // namespace trg
