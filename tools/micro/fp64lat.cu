// FP64 latency / throughput on one SM: dependent DFMA chains (1..8 per
// thread, 1..32 warps), clock64 around 1024 steps.
#include <cstdio>
#include <cuda_runtime.h>
template <int C>
__global__ void k(double* out, long long* cyc, double a, double b) {
  double x[C];
#pragma unroll
  for (int c = 0; c < C; ++c) x[c] = threadIdx.x * 1e-3 + c;
  __syncthreads();
  const long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < 1024; ++i)
#pragma unroll
    for (int c = 0; c < C; ++c) x[c] = fma(x[c], a, b);
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int C>
void run(int warps) {
  double* o; long long* c;
  cudaMalloc(&o, 8 * 1024 * 8); cudaMalloc(&c, 8 * 8);
  k<C><<<1, 32 * warps>>>(o, c, 0.999999, 1e-9);
  k<C><<<1, 32 * warps>>>(o, c, 0.999999, 1e-9);
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  const double per_step = (double)h / 1024.0;
  printf("chains/thread %d warps %2d: %.2f cycles per step (per dependent op); warp-DFMA issued per cycle per SM %.2f\n",
         C, warps, per_step, (double)C * warps / per_step);
  cudaFree(o); cudaFree(c);
}
int main() {
  for (int w : {1, 4, 8, 16, 32}) { run<1>(w); run<4>(w); run<8>(w); }
  return 0;
}
