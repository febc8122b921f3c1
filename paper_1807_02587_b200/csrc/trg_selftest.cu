// Diagnostic entry point: runs the device eigen/solve math on caller data so
// tests can check it bit-for-bit against the host (oracle) arithmetic.
#include "trg_internal.cuh"

namespace trg {
__global__ void k_eig_selftest(int n, const double* in, int count, double* evals, double* evecs,
                               int* status3) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  if (n == 6) {
    double a[6][6], ev[6], vec[6][6];
    for (int r = 0; r < 6; ++r)
      for (int c = 0; c < 6; ++c) a[r][c] = in[36 * i + 6 * r + c];
    jacobi_eig<6>(a, ev, vec);
    for (int r = 0; r < 6; ++r) {
      evals[6 * i + r] = ev[r];
      for (int c = 0; c < 6; ++c) evecs[36 * i + 6 * r + c] = vec[r][c];
    }
  } else {
    // n == 3: strict eig_sym3 (geometry.cpp:40-79); n == -3: floored at 1e-4
    // (Jacobi); n == 33 / -33: the same with the closed-form solver
    double m[3][3], lam[3], ax[3][3];
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) m[r][c] = in[9 * i + 3 * r + c];
    status3[i] = n == 3    ? eig_sym3(m, lam, ax)
                 : n == -3 ? eig_sym3_floored(m, 1e-4, lam, ax)
                 : n == 33 ? eig_sym3_cf(m, lam, ax)
                           : eig_sym3_floored_cf(m, 1e-4, lam, ax);
    for (int r = 0; r < 3; ++r) {
      evals[3 * i + r] = lam[r];
      for (int c = 0; c < 3; ++c) evecs[9 * i + 3 * r + c] = ax[r][c];
    }
  }
}
}  // namespace trg

using namespace trg;
extern "C" int trg_debug_eig(trg_ctx* ctx, int n, const double* in, int count, double* evals,
                             double* evecs, int* status3) {
  const int k = n == 6 ? 6 : 3;
  double *din, *dev, *dvec;
  int* dst;
  TRG_CU(cudaSetDevice(ctx->device));
  TRG_CU(cudaMalloc(&din, sizeof(double) * k * k * count));
  TRG_CU(cudaMalloc(&dev, sizeof(double) * k * count));
  TRG_CU(cudaMalloc(&dvec, sizeof(double) * k * k * count));
  TRG_CU(cudaMalloc(&dst, sizeof(int) * count));
  TRG_CU(cudaMemcpy(din, in, sizeof(double) * k * k * count, cudaMemcpyHostToDevice));
  k_eig_selftest<<<(count + 127) / 128, 128, 0, ctx->stream>>>(n, din, count, dev, dvec, dst);
  TRG_CU(cudaStreamSynchronize(ctx->stream));
  TRG_CU(cudaMemcpy(evals, dev, sizeof(double) * k * count, cudaMemcpyDeviceToHost));
  TRG_CU(cudaMemcpy(evecs, dvec, sizeof(double) * k * k * count, cudaMemcpyDeviceToHost));
  if (status3) TRG_CU(cudaMemcpy(status3, dst, sizeof(int) * count, cudaMemcpyDeviceToHost));
  cudaFree(din);
  cudaFree(dev);
  cudaFree(dvec);
  cudaFree(dst);
  return TRG_OK;
}

#include "trg_solve.cuh"
namespace trg {
__global__ void k_solve_selftest(const double* v, int nvp, SolveOut* out) {
  __shared__ SolveOut so;
  const long long t0 = clock64();
  __shared__ Eig6Smem e6;
  __shared__ double vs[kNormalEq];
  if (threadIdx.x < kNormalEq) vs[threadIdx.x] = v[threadIdx.x];
  __syncthreads();
  if (threadIdx.x < 32) warp_solve_normal_eq(vs, nvp, &so, e6);
  __syncthreads();
  if (threadIdx.x == 0) {
    so.crit_after = (double)(clock64() - t0);
    *out = so;
  }
}
}  // namespace trg
extern "C" int trg_debug_solve(trg_ctx* ctx, const double* v27, int nvp, double* out16) {
  double* dv;
  trg::SolveOut* dso;
  TRG_CU(cudaMalloc(&dv, sizeof(double) * 27));
  TRG_CU(cudaMalloc(&dso, sizeof(trg::SolveOut)));
  TRG_CU(cudaMemcpy(dv, v27, sizeof(double) * 27, cudaMemcpyHostToDevice));
  trg::k_solve_selftest<<<1, 64, 0, ctx->stream>>>(dv, nvp, dso);
  trg::SolveOut so;
  TRG_CU(cudaStreamSynchronize(ctx->stream));
  TRG_CU(cudaMemcpy(&so, dso, sizeof so, cudaMemcpyDeviceToHost));
  for (int i = 0; i < 3; ++i) {
    out16[i] = so.omega[i];
    out16[3 + i] = so.trans[i];
  }
  out16[6] = so.cond;
  out16[7] = so.degenerate;
  out16[8] = so.eig_sweeps;
  out16[9] = so.crit_after;  // cycles
  cudaFree(dv);
  cudaFree(dso);
  return TRG_OK;
}
