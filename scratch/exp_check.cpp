// Host check of exp_nonpos against libm exp (ulp error over [-708, 0]).
#include <cstdio>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include "../paper_1807_02587_b200/csrc/trg_math.cuh"
static double ulps(double a, double b) {
  if (a == b) return 0;
  int64_t ia, ib; memcpy(&ia, &a, 8); memcpy(&ib, &b, 8);
  return (double)std::llabs(ia - ib);
}
int main() {
  std::mt19937_64 g(1);
  double worst = 0, wx = 0;
  for (int i = 0; i < 20000000; ++i) {
    double x = -std::ldexp(std::uniform_real_distribution<double>(0, 1)(g), (int)(g() % 12) - 2);
    if (i % 7 == 0) x = -std::uniform_real_distribution<double>(0, 708)(g);
    if (i % 11 == 0) x = -std::uniform_real_distribution<double>(700, 746)(g);
    if (i % 13 == 0) x = std::uniform_real_distribution<double>(0, 700)(g);
    const double u = ulps(trg::exp_fast(x), std::exp(x));
    if (u > worst) { worst = u; wx = x; }
  }
  printf("max ulp %.0f at x=%.17g; exp(0)=%.17g exp(-708)=%g exp(-709)=%g exp(-745)=%g exp(-746)=%g exp(-inf)=%g\n", worst, wx,
         trg::exp_nonpos(0.0), trg::exp_nonpos(-708.0), trg::exp_nonpos(-709.0), trg::exp_nonpos(-745.0), trg::exp_nonpos(-746.0), trg::exp_nonpos(-INFINITY));
}
