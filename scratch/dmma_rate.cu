// FP64 tensor-core (DMMA m8n8k4) throughput and dependent latency on this GPU.
#include <cstdio>
template <int CHAINS>
__global__ void k(double* out, int iters) {
  double c[CHAINS][2];
  for (int i = 0; i < CHAINS; ++i) c[i][0] = c[i][1] = 0.0;
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < CHAINS; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};"
                   : "=d"(c[i][0]), "=d"(c[i][1]) : "d"(a), "d"(b), "d"(c[i][0]), "d"(c[i][1]));
  double s = 0;
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1];
  if (s == 1.2345) out[0] = s;
}
int main() {
  double* d; cudaMalloc(&d, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int rep = 0; rep < 2; ++rep) {
    const int it = 4000;
    float ms;
    // latency: 1 warp, 1 chain
    cudaEventRecord(a); k<1><<<1, 32>>>(d, it); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("dependent DMMA latency ~%.0f cycles\n", ms * 1e-3 * 1.965e9 / it);
    // throughput: many warps, 4 chains
    cudaEventRecord(a); k<4><<<sms * 4, 256>>>(d, it); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    const double flops = 2.0 * 8 * 8 * 4 * (double)(sms * 4 * 8) * it * 4;
    printf("DMMA throughput: %.1f TFLOP/s\n", flops / (ms * 1e-3) / 1e12);
  }
}
