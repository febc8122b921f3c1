// Grid-barrier latency: __threadfence (MEMBAR.SC) vs release/acquire
// (MEMBAR.ALL) arrival + polling.  444 CTAs x 256 threads, 2000 barriers.
#include <cstdio>
#include <cooperative_groups.h>
__device__ __forceinline__ void bar_sc(unsigned* bar, unsigned n) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* vb = bar;
    const unsigned gen = vb[1];
    __threadfence();
    const unsigned arrived = atomicAdd(&bar[0], 1u);
    if (arrived == n - 1) {
      atomicExch(&bar[0], 0u);
      __threadfence();
      atomicAdd(&bar[1], 1u);
    } else {
      unsigned ns = 32;
      while (vb[1] == gen) { __nanosleep(ns); ns = ns < 256 ? 2 * ns : 256; }
    }
    __threadfence();
  }
  __syncthreads();
}
__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ unsigned atom_ar(unsigned* p, unsigned v) {
  unsigned o; asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(o) : "l"(p), "r"(v) : "memory"); return o;
}
__device__ __forceinline__ void red_rel(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
// counting barrier: arrivals accumulate forever; barrier k completes when
// count reaches k * n (no reset, no generation word)
__device__ __forceinline__ void bar_ar(unsigned* bar, unsigned n, unsigned& k, int spin) {
  __syncthreads();
  if (threadIdx.x == 0) {
    ++k;
    const unsigned target = k * n;
    const unsigned old = atom_ar(&bar[2], 1u);
    if (old + 1 != target) {
      unsigned ns = 32;
      while ((int)(ld_acq(&bar[2]) - target) < 0) { if (spin) { __nanosleep(ns); ns = ns < 128 ? 2 * ns : 128; } }
    }
  }
  __syncthreads();
}
__global__ void kb(unsigned* bar, long long* out, int mode, int iters) {
  unsigned k = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (mode == 0) bar_sc(bar, gridDim.x);
    else bar_ar(bar, gridDim.x, k, mode == 1);
  }
  long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = (t1 - t0) / iters;
}
int main() {
  unsigned* bar; long long* out;
  cudaMalloc(&bar, 64); cudaMalloc(&out, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int per = 1; per <= 3; ++per)
    for (int mode = 0; mode < 3; ++mode) {
      cudaMemset(bar, 0, 64);
      int G = sms * per, it = 2000;
      void* args[] = {&bar, &out, &mode, &it};
      cudaLaunchCooperativeKernel((void*)kb, G, 256, args, 0, 0);
      cudaError_t e = cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
      printf("G=%d mode=%d (%s): %lld cycles/barrier (%.2f us) %s\n", G, mode,
             mode == 0 ? "threadfence" : mode == 1 ? "acq/rel + nanosleep" : "acq/rel spin", c, c / 1965.0,
             cudaGetErrorString(e));
    }
  return 0;
}
