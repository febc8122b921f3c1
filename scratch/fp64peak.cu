// FP64 pipe throughput on this device: independent DFMA chains, and the
// exp_fast / rcp_sum building blocks of the E-step.
#include <cstdio>
#include "../paper_1807_02587_b200/csrc/trg_math.cuh"
__global__ void k_fma(double* out, int iters) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  const double b = 1.0000001, c = 1e-9;
  for (int k = 0; k < iters; ++k)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 1.2345) out[0] = s;
}
__global__ void k_exp(double* out, int iters) {
  double a[4];
  for (int i = 0; i < 4; ++i) a[i] = -(threadIdx.x * 1e-3 + i);
  double s = 0;
  for (int k = 0; k < iters; ++k)
#pragma unroll
    for (int i = 0; i < 4; ++i) { s += trg::exp_fast(a[i]); a[i] -= 1e-7; }
  if (s == 1.2345) out[0] = s;
}
__global__ void k_exp_lib(double* out, int iters) {
  double a[4];
  for (int i = 0; i < 4; ++i) a[i] = -(threadIdx.x * 1e-3 + i);
  double s = 0;
  for (int k = 0; k < iters; ++k)
#pragma unroll
    for (int i = 0; i < 4; ++i) { s += exp(a[i]); a[i] -= 1e-7; }
  if (s == 1.2345) out[0] = s;
}
int main() {
  double* d; cudaMalloc(&d, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int blocks = sms * 8, threads = 256;
  for (int rep = 0; rep < 2; ++rep) {
    int it = 20000;
    cudaEventRecord(a); k_fma<<<blocks, threads>>>(d, it); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double fmas = (double)blocks * threads * it * 8;
    printf("DFMA: %.1f TFMA/s = %.1f TFLOP/s; per SM per clk (1.965GHz): %.1f lanes\n", fmas / ms / 1e9, 2 * fmas / ms / 1e9,
           fmas / (ms * 1e-3) / sms / 1.965e9);
    it = 2000;
    cudaEventRecord(a); k_exp<<<blocks, threads>>>(d, it); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    double ev = (double)blocks * threads * it * 4;
    printf("exp_fast: %.1f G/s = %.2f per SM per clk\n", ev / ms / 1e6, ev / (ms * 1e-3) / sms / 1.965e9);
    cudaEventRecord(a); k_exp_lib<<<blocks, threads>>>(d, it); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("libdevice exp: %.1f G/s = %.2f per SM per clk\n", ev / ms / 1e6, ev / (ms * 1e-3) / sms / 1.965e9);
  }
}
