#include <cstdio>
#include <cstdlib>
#include "../paper_1807_02587_b200/csrc/trg_math.cuh"
__global__ void k(const double* in, double* out, int cnt) {
  int i = threadIdx.x; if (i >= cnt) return;
  double a[6][6], ev[6], vec[6][6];
  for (int r = 0; r < 6; ++r) for (int c = 0; c < 6; ++c) a[r][c] = in[36*i + 6*r + c];
  trg::jacobi_eig<6>(a, ev, vec);
  for (int r = 0; r < 6; ++r) out[6*i + r] = ev[r];
}
int main() {
  const int cnt = 8; double h[36*cnt], hev[6*cnt], dev_ev[6*cnt];
  srand(1);
  for (int i = 0; i < cnt; ++i) {
    double b[6][6];
    for (int r=0;r<6;++r) for(int c=0;c<6;++c) b[r][c] = (rand()/(double)RAND_MAX) - 0.5;
    for (int r=0;r<6;++r) for(int c=0;c<6;++c) { double s=0; for(int k2=0;k2<6;++k2) s+=b[r][k2]*b[c][k2]; h[36*i+6*r+c]=s + (r==c ? 0.01*(i+1) : 0); }
    double a[6][6], ev[6], vec[6][6];
    for (int r=0;r<6;++r) for(int c=0;c<6;++c) a[r][c]=h[36*i+6*r+c];
    trg::jacobi_eig<6>(a, ev, vec);
    for (int r=0;r<6;++r) hev[6*i+r]=ev[r];
  }
  double *din, *dout; cudaMalloc(&din, sizeof h); cudaMalloc(&dout, sizeof dev_ev);
  cudaMemcpy(din, h, sizeof h, cudaMemcpyHostToDevice);
  k<<<1, 32>>>(din, dout, cnt); cudaMemcpy(dev_ev, dout, sizeof dev_ev, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i=0;i<6*cnt;++i) if (hev[i] != dev_ev[i]) { ++bad; if (bad < 6) printf("i %d host %.17g dev %.17g\n", i, hev[i], dev_ev[i]); }
  printf("mismatches %d / %d\n", bad, 6*cnt);
  return 0;
}
