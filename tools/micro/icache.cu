// Does a 3x3 eigensolve slow down when its code is not in the SM's
// instruction cache?  Times one SIMT eigensolve (clock64) right after
// executing ~256 KB of unrelated straight-line code.  Not product code.
#include <cstdio>
#include "../../paper_1807_02587_b200/csrc/trg_gmm.cuh"
using namespace trg;

#include "junk.inc"

__global__ void kb(const double* mats, long long* cyc, double* out, int evict) {
  const int lane = threadIdx.x;
  double a[3][3], w[9];
  for (int i = 0; i < 9; ++i) a[i / 3][i % 3] = mats[i] + lane * 1e-3 * (i % 4 == 0);
  for (int i = 0; i < 9; ++i) w[i] = (i % 4) == 0 ? 1.0 : 0.0;
  double ev[3], vec[3][3];
  double x = a[0][0];
  for (int rep = 0; rep < 3; ++rep) {
    if (evict) x = junk_big(x);
    a[1][1] += x * 1e-300;
    __syncwarp();
    const long long t0 = clock64();
    jacobi3_simt(a, ev, vec, w);
    const long long t1 = clock64();
    a[0][0] += ev[0] * 1e-300;
    if (lane == 0) cyc[rep] = t1 - t0;
  }
  out[lane] = ev[0] + vec[0][0] + x;
}

int main() {
  double hm[9] = {2.0, 0.3, 0.1, 0.3, 1.0, 0.05, 0.1, 0.05, 0.2};
  double *dm, *dout; long long* dc;
  cudaMalloc(&dm, sizeof hm); cudaMalloc(&dout, 8 * 32); cudaMalloc(&dc, 8 * 3);
  cudaMemcpy(dm, hm, sizeof hm, cudaMemcpyHostToDevice);
  for (int ev = 0; ev < 2; ++ev)
    for (int r = 0; r < 2; ++r) {
      kb<<<1, 32>>>(dm, dc, dout, ev);
      long long c[3]; cudaMemcpy(c, dc, 24, cudaMemcpyDeviceToHost);
      printf("evict=%d launch %d: eig cycles per rep %lld %lld %lld\n", ev, r, c[0], c[1], c[2]);
    }
  return 0;
}
