#include <cstdio>
#include <cstdlib>
#include <cmath>
#include "../paper_1807_02587_b200/csrc/trg_math.cuh"
template <int N, int VARIANT>
__host__ __device__ void jac(double a[N][N], double evals[N]) {
  double v[N][N];
  for (int i = 0; i < N; ++i) for (int j = 0; j < N; ++j) v[i][j] = (i == j) ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 64; ++sweep) {
    bool rotated = false;
#pragma unroll 1
    for (int p = 0; p < N - 1; ++p)
#pragma unroll 1
      for (int q = p + 1; q < N; ++q) {
        const double apq = a[p][q];
        if (apq == 0.0) continue;
        const double app = a[p][p], aqq = a[q][q];
        const double g = 100.0 * fabs(apq);
        if (fabs(app) + g == fabs(app) && fabs(aqq) + g == fabs(aqq)) { a[p][q] = 0.0; a[q][p] = 0.0; continue; }
        rotated = true;
        const double h = aqq - app;
        double t;
        if (fabs(h) + g == fabs(h)) t = apq / h;
        else { const double theta = 0.5 * h / apq; t = 1.0 / (fabs(theta) + sqrt(1.0 + theta * theta)); if (theta < 0.0) t = -t; }
        const double c = 1.0 / sqrt(1.0 + t * t), s = t * c, tau = s / (1.0 + c);
        if (VARIANT == 1) {
          double cp[N], cq[N];
          for (int r = 0; r < N; ++r) { cp[r] = a[r][p]; cq[r] = a[r][q]; }
          for (int r = 0; r < N; ++r) {
            if (r == p || r == q) continue;
            const double np = cp[r] - s * (cq[r] + cp[r] * tau), nq = cq[r] + s * (cp[r] - cq[r] * tau);
            a[r][p] = np; a[p][r] = np; a[r][q] = nq; a[q][r] = nq;
          }
        } else {
          for (int r = 0; r < N; ++r) {
            if (r == p || r == q) continue;
            const double arp = a[r][p], arq = a[r][q];
            const double np = arp - s * (arq + arp * tau), nq = arq + s * (arp - arq * tau);
            a[r][p] = np; a[p][r] = np; a[r][q] = nq; a[q][r] = nq;
          }
        }
        a[p][p] = app - t * apq; a[q][q] = aqq + t * apq; a[p][q] = 0.0; a[q][p] = 0.0;
        for (int r = 0; r < N; ++r) { const double vrp = v[r][p], vrq = v[r][q]; v[r][p] = vrp - s * (vrq + vrp * tau); v[r][q] = vrq + s * (vrp - vrq * tau); }
      }
    if (!rotated) break;
  }
  for (int i = 0; i < N; ++i) evals[i] = a[i][i];
}
template <int VAR>
__global__ void k(const double* in, double* out, int cnt) {
  int i = threadIdx.x; if (i >= cnt) return;
  double a[6][6], ev[6];
  for (int r = 0; r < 6; ++r) for (int c = 0; c < 6; ++c) a[r][c] = in[36*i + 6*r + c];
  if (VAR == 9) { double vec[6][6]; trg::jacobi_eig<6>(a, ev, vec); }
  else jac<6, VAR>(a, ev);
  for (int r = 0; r < 6; ++r) out[6*i + r] = ev[r];
}
int main() {
  const int cnt = 8; double h[36*cnt], hev[6*cnt], dev_ev[6*cnt];
  srand(1);
  for (int i = 0; i < cnt; ++i) {
    double b[6][6];
    for (int r=0;r<6;++r) for(int c=0;c<6;++c) b[r][c] = (rand()/(double)RAND_MAX) - 0.5;
    for (int r=0;r<6;++r) for(int c=0;c<6;++c) { double s=0; for(int k2=0;k2<6;++k2) s+=b[r][k2]*b[c][k2]; h[36*i+6*r+c]=s + (r==c ? 0.01*(i+1) : 0); }
  }
  double *din, *dout; cudaMalloc(&din, sizeof h); cudaMalloc(&dout, sizeof dev_ev);
  cudaMemcpy(din, h, sizeof h, cudaMemcpyHostToDevice);
  for (int var : {0, 1, 9}) {
    for (int i = 0; i < cnt; ++i) { double a[6][6], ev[6]; for (int r=0;r<6;++r) for(int c=0;c<6;++c) a[r][c]=h[36*i+6*r+c]; jac<6,0>(a, ev); for (int r=0;r<6;++r) hev[6*i+r]=ev[r]; }
    if (var == 0) k<0><<<1,32>>>(din, dout, cnt); else if (var == 1) k<1><<<1,32>>>(din, dout, cnt); else k<9><<<1,32>>>(din, dout, cnt);
    cudaMemcpy(dev_ev, dout, sizeof dev_ev, cudaMemcpyDeviceToHost);
    // compare sorted eigenvalue sets (jac returns unsorted diag)
    int bad = 0; double worst = 0;
    for (int i = 0; i < cnt; ++i) {
      double x[6], y[6]; for (int r=0;r<6;++r) { x[r]=hev[6*i+r]; y[r]=dev_ev[6*i+r]; }
      for (int p=0;p<6;++p) for(int q=p+1;q<6;++q) { if (x[q]<x[p]) {double t=x[p];x[p]=x[q];x[q]=t;} if (y[q]<y[p]) {double t=y[p];y[p]=y[q];y[q]=t;} }
      for (int r=0;r<6;++r) { double d = fabs(x[r]-y[r]); if (d > 1e-12) ++bad; if (d > worst) worst = d; }
    }
    printf("variant %d: bad %d worst %.3g\n", var, bad, worst);
  }
  return 0;
}
