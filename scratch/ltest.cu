#include <cstdio>
#include <cstdlib>
#include "../paper_1807_02587_b200/csrc/trg_math.cuh"
__global__ void k(const double* in, const double* bb, double* out, int cnt) {
  int i = threadIdx.x; if (i >= cnt) return;
  double a[6][6], b[6], x[6];
  for (int r = 0; r < 6; ++r) { b[r] = bb[6*i+r]; for (int c = 0; c < 6; ++c) a[r][c] = in[36*i + 6*r + c]; }
  trg::ldlt_solve6(a, b, x);
  for (int r = 0; r < 6; ++r) out[6*i + r] = x[r];
}
int main() {
  const int cnt = 8; double h[36*cnt], hb[6*cnt], hx[6*cnt], dx[6*cnt];
  srand(3);
  for (int i = 0; i < cnt; ++i) {
    double m[6][6];
    for (int r=0;r<6;++r) for(int c=0;c<6;++c) m[r][c] = (rand()/(double)RAND_MAX) - 0.5;
    for (int r=0;r<6;++r) { hb[6*i+r] = rand()/(double)RAND_MAX; for(int c=0;c<6;++c) { double s=0; for(int k2=0;k2<6;++k2) s+=m[r][k2]*m[c][k2]; h[36*i+6*r+c]=s + (r==c ? 0.1*(i+1) : 0); } }
    double a[6][6], b[6], x[6];
    for (int r=0;r<6;++r) { b[r]=hb[6*i+r]; for(int c=0;c<6;++c) a[r][c]=h[36*i+6*r+c]; }
    trg::ldlt_solve6(a, b, x);
    for (int r=0;r<6;++r) hx[6*i+r]=x[r];
  }
  double *din, *db, *dout; cudaMalloc(&din, sizeof h); cudaMalloc(&db, sizeof hb); cudaMalloc(&dout, sizeof dx);
  cudaMemcpy(din, h, sizeof h, cudaMemcpyHostToDevice); cudaMemcpy(db, hb, sizeof hb, cudaMemcpyHostToDevice);
  k<<<1, 32>>>(din, db, dout, cnt); cudaMemcpy(dx, dout, sizeof dx, cudaMemcpyDeviceToHost);
  int bad = 0; for (int i=0;i<6*cnt;++i) if (hx[i] != dx[i]) ++bad;
  printf("ldlt mismatches %d / %d  (e.g. host %.6g dev %.6g)\n", bad, 6*cnt, hx[0], dx[0]);
  return 0;
}
