// Latency of the device 3x3 eigen pieces (one thread, dependent chain).
#include <cstdio>
#include "../paper_1807_02587_b200/csrc/trg_internal.cuh"
#include "../paper_1807_02587_b200/csrc/trg_gmm.cuh"
using namespace trg;
__global__ void kb(DNode* nodes, double* cov, long long* out, int warm, int reps) {
  DNode d = nodes[0];
  double c[9];
  for (int i = 0; i < 9; ++i) c[i] = cov[i];
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    refresh_node(d, c, warm != 0);
    c[1] += d.lam[0] * 1e-30;  // dependency
    c[3] = c[1];
  }
  long long t1 = clock64();
  out[0] = (t1 - t0) / reps;
  nodes[1] = d;
}
__global__ void kjac(DNode* nodes, double* cov, long long* out, int mode, int reps) {
  DNode d = nodes[0];
  double c[9];
  for (int i = 0; i < 9; ++i) c[i] = cov[i];
  long long t0 = clock64();
  double acc = 0;
  for (int r = 0; r < reps; ++r) {
    double a[3][3], ev[3], vec[3][3], lam[3], ax[3][3];
    for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j) a[i][j] = c[3 * i + j];
    if (mode == 0) { jacobi_eig<3>(a, ev, vec, d.axT); acc = ev[0] + vec[1][1]; }
    if (mode == 1) { eig_sym3(a, lam, ax, d.axT); acc = lam[0] + ax[1][1]; }
    if (mode == 2) { jacobi_eig<3>(a, ev, vec, nullptr); acc = ev[0] + vec[1][1]; }
    c[1] += acc * 1e-30;
    c[3] = c[1];
  }
  long long t1 = clock64();
  out[0] = (t1 - t0) / reps;
  nodes[1].lam[0] = c[1];
}
__global__ void kldlt(double* A0, long long* out, int mode, int reps) {
  double A[6][6], b[6], x[6], tr, mind;
  for (int i = 0; i < 6; ++i) { b[i] = A0[36 + i]; for (int j = 0; j < 6; ++j) A[i][j] = A0[6 * i + j]; }
  long long t0 = clock64();
  double acc = 0;
  for (int r = 0; r < reps; ++r) {
    if (mode == 0) { ldlt_solve6_tr(A, b, x, &tr, &mind); acc = x[0] + tr; }
    if (mode == 1) { double w[3] = {x[0] + 1e-3, x[1], x[2]}, R[9]; small_angle_rotation(w, R); acc = R[1]; x[0] = acc * 1e-9; }
    b[0] += acc * 1e-30;
  }
  long long t1 = clock64();
  out[0] = (t1 - t0) / reps;
  A0[50] = acc;
}
__global__ void klog(double* x, long long* out, int reps) {
  double v = x[0];
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) v = log(v) + 3.0;
  long long t1 = clock64();
  out[0] = (t1 - t0) / reps;
  x[1] = v;
}
__global__ void kfma(double* x, long long* out, int reps) {
  double v = x[0];
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) v = fma(v, 0.999, 1e-3);
  long long t1 = clock64();
  out[0] = (t1 - t0) / reps;
  x[1] = v;
}
__global__ void krcp(double* x, long long* out, int reps) {
  double v = x[0];
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) v = __drcp_rn(v) + 0.5;
  long long t1 = clock64();
  out[0] = (t1 - t0) / reps;
  x[1] = v;
}
__global__ void kdiv(double* x, long long* out, int reps) {
  double v = x[0], w = x[2];
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) v = w / v + 0.5;
  long long t1 = clock64();
  out[0] = (t1 - t0) / reps;
  x[1] = v;
}
__global__ void ksqrt(double* x, long long* out, int reps) {
  double v = x[0];
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) v = __dsqrt_rn(v) + 1.5;
  long long t1 = clock64();
  out[0] = (t1 - t0) / reps;
  x[1] = v;
}
int main() {
  // a node with a random rotation basis
  DNode h{};
  double lam[3] = {0.04, 0.01, 0.0004};
  double th = 0.3, ph = 0.7;
  double R[3][3] = {{cos(th), -sin(th), 0}, {sin(th), cos(th), 0}, {0, 0, 1}};
  double S[3][3] = {{1, 0, 0}, {0, cos(ph), -sin(ph)}, {0, sin(ph), cos(ph)}};
  double A[3][3];
  for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j) { A[i][j] = 0; for (int k = 0; k < 3; ++k) A[i][j] += R[i][k] * S[k][j]; }
  double cov[9];
  for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j) { double s = 0; for (int k = 0; k < 3; ++k) s += A[i][k] * lam[k] * A[j][k]; cov[3 * i + j] = s; }
  for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j) h.axT[3 * i + j] = A[j][i];
  cov[1] += 1e-7; cov[3] += 1e-7;
  DNode* dn; double* dc; long long* dout; double* dx;
  cudaMalloc(&dn, 2 * sizeof(DNode)); cudaMalloc(&dc, 72); cudaMalloc(&dout, 8); cudaMalloc(&dx, 24);
  cudaMemcpy(dn, &h, sizeof(DNode), cudaMemcpyHostToDevice);
  cudaMemcpy(dc, cov, 72, cudaMemcpyHostToDevice);
  double x[3] = {1.7, 0, 2.3};
  cudaMemcpy(dx, x, 24, cudaMemcpyHostToDevice);
  long long o;
  for (int warm = 0; warm < 2; ++warm) {
    kb<<<1, 1>>>(dn, dc, dout, warm, 50); cudaMemcpy(&o, dout, 8, cudaMemcpyDeviceToHost);
    printf("refresh_node warm=%d: %lld cycles\n", warm, o);
  }
  for (int m = 0; m < 3; ++m) {
    kjac<<<1, 1>>>(dn, dc, dout, m, 50); cudaMemcpy(&o, dout, 8, cudaMemcpyDeviceToHost);
    printf("mode %d (0 jacobi warm, 1 eig_sym3 warm, 2 jacobi cold): %lld cycles\n", m, o);
  }
  {
    double hA[64];
    for (int i = 0; i < 6; ++i) for (int j = 0; j < 6; ++j) hA[6 * i + j] = (i == j ? 10.0 + i : 0.0) + 1.0 / (1 + i + j);
    for (int i = 0; i < 6; ++i) hA[36 + i] = 1.0 + i;
    double* dA; cudaMalloc(&dA, 64 * 8); cudaMemcpy(dA, hA, 64 * 8, cudaMemcpyHostToDevice);
    for (int m = 0; m < 2; ++m) {
      kldlt<<<1, 1>>>(dA, dout, m, 50); cudaMemcpy(&o, dout, 8, cudaMemcpyDeviceToHost);
      printf("%s: %lld cycles\n", m == 0 ? "ldlt_solve6_tr" : "small_angle_rotation", o);
    }
  }
  klog<<<1, 1>>>(dx, dout, 200); cudaMemcpy(&o, dout, 8, cudaMemcpyDeviceToHost); printf("log: %lld\n", o);
  kfma<<<1, 1>>>(dx, dout, 1000); cudaMemcpy(&o, dout, 8, cudaMemcpyDeviceToHost); printf("dfma: %lld\n", o);
  krcp<<<1, 1>>>(dx, dout, 200); cudaMemcpy(&o, dout, 8, cudaMemcpyDeviceToHost); printf("drcp_rn+add: %lld\n", o);
  kdiv<<<1, 1>>>(dx, dout, 200); cudaMemcpy(&o, dout, 8, cudaMemcpyDeviceToHost); printf("ddiv+add: %lld\n", o);
  ksqrt<<<1, 1>>>(dx, dout, 200); cudaMemcpy(&o, dout, 8, cudaMemcpyDeviceToHost); printf("dsqrt_rn+add: %lld\n", o);
  return 0;
}
