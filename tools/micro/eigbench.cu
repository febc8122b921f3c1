// eig3_cf vs eig3_cf2 (trg_math.cuh): cycles per call on 16 lanes of one
// warp and accuracy against the oracle's Jacobi (jacobi3) on random SPD,
// rank-deficient, near-degenerate and diagonal matrices.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include "../../paper_1807_02587_b200/csrc/trg_gmm.cuh"
using namespace trg;

__global__ void k(const double* M, int n, double* out, long long* cyc, int which) {
  const int i = blockIdx.x * 16 + (threadIdx.x & 15);
  if (threadIdx.x >= 16 || i >= n) return;
  double m[3][3];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) m[r][c] = M[9 * i + 3 * r + c];
  double ev[3], vec[3][3];
  const long long t0 = clock64();
  if (which == 0) eig3_cf(m, ev, vec);
  else if (which == 1) eig3_cf2(m, ev, vec);
  else { double mm[3][3]; for (int r = 0; r < 3; ++r) for (int c = 0; c < 3; ++c) mm[r][c] = m[r][c]; jacobi3(mm, ev, vec, nullptr); }
  const long long t1 = clock64();
  for (int c = 0; c < 3; ++c) out[12 * i + c] = ev[c];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) out[12 * i + 3 + 3 * r + c] = vec[r][c];
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  const int n = 16 * 512;
  double* h = (double*)malloc(sizeof(double) * 9 * n);
  srand(7);
  auto rnd = [] { return 2.0 * rand() / RAND_MAX - 1.0; };
  for (int i = 0; i < n; ++i) {
    double a[3][3];
    for (int r = 0; r < 3; ++r) for (int c = 0; c < 3; ++c) a[r][c] = rnd();
    double lam[3] = {fabs(rnd()) + 1e-3, fabs(rnd()) + 1e-3, fabs(rnd()) + 1e-3};
    const int kind = i % 5;
    if (kind == 1) { lam[1] = 0; lam[2] = 0; }            // rank 1
    if (kind == 2) { lam[1] = lam[0] * (1 + 1e-9); }      // near-degenerate pair
    if (kind == 3) { lam[0] *= 1e6; }                     // ill-conditioned
    // Q from Gram-Schmidt of a
    double q[3][3];
    for (int c = 0; c < 3; ++c) {
      double v[3] = {a[0][c], a[1][c], a[2][c]};
      for (int p = 0; p < c; ++p) { double d = v[0]*q[0][p]+v[1]*q[1][p]+v[2]*q[2][p]; for (int r = 0; r < 3; ++r) v[r] -= d*q[r][p]; }
      double nn = sqrt(v[0]*v[0]+v[1]*v[1]+v[2]*v[2]); for (int r = 0; r < 3; ++r) q[r][c] = v[r]/nn;
    }
    double sc = pow(10.0, (i % 7) - 3);
    for (int r = 0; r < 3; ++r) for (int c = 0; c < 3; ++c) {
      double s = 0; for (int l = 0; l < 3; ++l) s += q[r][l] * lam[l] * q[c][l];
      h[9 * i + 3 * r + c] = (kind == 4 && r != c) ? 0.0 : s * sc;
    }
    for (int r = 0; r < 3; ++r) for (int c = r + 1; c < 3; ++c) h[9*i+3*c+r] = h[9*i+3*r+c];
  }
  double *dM, *dO[3]; long long* dc;
  cudaMalloc(&dM, sizeof(double) * 9 * n); cudaMemcpy(dM, h, sizeof(double) * 9 * n, cudaMemcpyHostToDevice);
  cudaMalloc(&dc, sizeof(long long) * n / 16);
  double* ho[3];
  for (int w = 0; w < 3; ++w) {
    cudaMalloc(&dO[w], sizeof(double) * 12 * n);
    k<<<n / 16, 32>>>(dM, n, dO[w], dc, w);
    k<<<n / 16, 32>>>(dM, n, dO[w], dc, w);
    long long* hc = (long long*)malloc(sizeof(long long) * n / 16);
    cudaMemcpy(hc, dc, sizeof(long long) * n / 16, cudaMemcpyDeviceToHost);
    long long s = 0; for (int b = 0; b < n / 16; ++b) s += hc[b];
    printf("%s: %.0f cycles per call (16 lanes)\n", w == 0 ? "eig3_cf " : w == 1 ? "eig3_cf2" : "jacobi3 ", (double)s / (n / 16));
    ho[w] = (double*)malloc(sizeof(double) * 12 * n);
    cudaMemcpy(ho[w], dO[w], sizeof(double) * 12 * n, cudaMemcpyDeviceToHost);
  }
  // eigenvalue error vs Jacobi relative to ||A||_max, and reconstruction error
  for (int w = 0; w < 2; ++w) {
    double emax = 0, rmax = 0;
    for (int i = 0; i < n; ++i) {
      double am = 0; for (int q = 0; q < 9; ++q) am = fmax(am, fabs(h[9*i+q]));
      for (int c = 0; c < 3; ++c) emax = fmax(emax, fabs(ho[w][12*i+c] - ho[2][12*i+c]) / am);
      for (int r = 0; r < 3; ++r) for (int c = 0; c < 3; ++c) {
        double s = 0; for (int l = 0; l < 3; ++l) s += ho[w][12*i+3+3*r+l] * ho[w][12*i+l] * ho[w][12*i+3+3*c+l];
        rmax = fmax(rmax, fabs(s - h[9*i+3*r+c]) / am);
      }
    }
    printf("%s: max |dlambda|/|A| vs jacobi %.3g, max reconstruction error/|A| %.3g\n", w == 0 ? "eig3_cf " : "eig3_cf2", emax, rmax);
  }
  return 0;
}
