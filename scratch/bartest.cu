// Grid-barrier microbenchmark: flat atomic counter vs two-level.
#include <cstdio>
__device__ __forceinline__ void flat_sync(unsigned* bar, unsigned nb) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* vb = bar;
    const unsigned gen = vb[1];
    __threadfence();
    const unsigned arrived = atomicAdd(&bar[0], 1u);
    if (arrived == nb - 1) { atomicExch(&bar[0], 0u); __threadfence(); atomicAdd(&bar[1], 1u); }
    else { while (vb[1] == gen) __nanosleep(20); }
    __threadfence();
  }
  __syncthreads();
}
// two-level: groups of GS CTAs; bar[2+g*32] group counters (separate 128B lines)
template <int GS>
__device__ __forceinline__ void tree_sync(unsigned* bar, unsigned nb) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* vb = bar;
    const unsigned gen = vb[1];
    const unsigned g = blockIdx.x / GS, ng = (nb + GS - 1) / GS;
    const unsigned gsize = min((unsigned)GS, nb - g * GS);
    __threadfence();
    const unsigned a = atomicAdd(&bar[64 + g * 32], 1u);
    if (a == gsize - 1) {
      bar[64 + g * 32] = 0u;
      const unsigned arrived = atomicAdd(&bar[0], 1u);
      if (arrived == ng - 1) { atomicExch(&bar[0], 0u); __threadfence(); atomicAdd(&bar[1], 1u); }
      else { while (vb[1] == gen) __nanosleep(20); }
    } else {
      while (vb[1] == gen) __nanosleep(20);
    }
    __threadfence();
  }
  __syncthreads();
}
__device__ __forceinline__ void nofence_sync(unsigned* bar, unsigned nb) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned gen;
    asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(gen) : "l"(bar + 1));
    unsigned arrived;
    asm volatile("atom.add.release.gpu.u32 %0, [%1], 1;" : "=r"(arrived) : "l"(bar));
    if (arrived == nb - 1) {
      asm volatile("st.relaxed.gpu.u32 [%0], 0;" :: "l"(bar));
      asm volatile("red.release.gpu.add.u32 [%0], 1;" :: "l"(bar + 1));
    } else {
      unsigned g2;
      do { asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(g2) : "l"(bar + 1)); } while (g2 == gen);
    }
  }
  __syncthreads();
}
// counting barrier: arrivals only add (no return value), every CTA polls the
// monotonic counter until it reaches epoch * nb
template <bool SLEEP>
__device__ __forceinline__ void count_sync(unsigned* bar, unsigned nb, unsigned& epoch) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned target = (++epoch) * nb;
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" :: "l"(bar) : "memory");
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
      if (SLEEP && v < target) __nanosleep(32);
    } while (v < target);
  }
  __syncthreads();
}
template <int MODE>
__global__ void k(unsigned* bar, int iters, long long* out) {
  unsigned epoch = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (MODE == 0) flat_sync(bar, gridDim.x);
    else if (MODE == 1) tree_sync<16>(bar, gridDim.x);
    else if (MODE == 2) nofence_sync(bar, gridDim.x);
    else if (MODE == 3) count_sync<false>(bar, gridDim.x, epoch);
    else count_sync<true>(bar, gridDim.x, epoch);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *out = (clock64() - t0) / iters;
}
int main() {
  unsigned* bar; long long* out; cudaMalloc(&bar, 1 << 16); cudaMalloc(&out, 8);
  for (int per : {1, 2, 3, 4}) {
    const int G = 148 * per;
    for (int mode = 0; mode < 5; ++mode) {
      cudaMemset(bar, 0, 1 << 16);
      int it = 2000; void* args[] = {&bar, &it, &out};
      void* fn = mode == 0 ? (void*)k<0> : mode == 1 ? (void*)k<1> : mode == 2 ? (void*)k<2> : mode == 3 ? (void*)k<3> : (void*)k<4>;
      cudaLaunchCooperativeKernel(fn, G, 256, args, 0, 0);
      cudaError_t e = cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
      printf("G=%d mode=%d: %lld cycles/barrier (%.2f us) %s\n", G, mode, c, c / 1950.0, cudaGetErrorString(e));
    }
  }
  return 0;
}
