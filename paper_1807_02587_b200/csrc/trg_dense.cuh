// Dense association (responsibilities_dense, association.cpp:54-89): every
// point against every component.  Two passes with a grid barrier between
// them: per-point score sums, then per-component deposits into the
// epoch-stamped partial rows the tree path uses (combine_node follows).
// Shared by the standalone kernel (trg_flat.cu) and k_register<true>.
#pragma once
#include "trg_assoc.cuh"

namespace trg {

// Sum node j's partial rows over CTAs in fixed order (one warp per node).
// Rows are read in batches of 4 per lane with the stamp test as a select,
// so the loads of a batch are all in flight together (a branch per row
// serialises the L2 round trips); skipped rows add exactly 0.
template <int NM>
__device__ __forceinline__ void combine_node(const double* __restrict__ partials,
                                             const uint32_t* __restrict__ stamps, uint32_t epoch,
                                             int G, int j, double out[NM]) {
  const int lane = threadIdx.x & 31;
  double acc[NM];
#pragma unroll
  for (int m = 0; m < NM; ++m) acc[m] = 0.0;
  const size_t base = (size_t)j * G;
  for (int c0 = lane; c0 < G; c0 += 128) {
    uint32_t st[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int c = c0 + 32 * u;
      st[u] = c < G ? __ldcg(stamps + base + c) : 0u;
    }
    double v[4][NM];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int c = c0 + 32 * u;
      const bool ok = c < G && st[u] == epoch;
      const double* row = partials + (base + (ok ? c : 0)) * NM;
#pragma unroll
      for (int m = 0; m < NM; ++m) v[u][m] = ok ? __ldcg(row + m) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int m = 0; m < NM; ++m) acc[m] += v[u][m];
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1)
#pragma unroll
    for (int m = 0; m < NM; ++m) acc[m] += __shfl_xor_sync(0xffffffffu, acc[m], off);
#pragma unroll
  for (int m = 0; m < NM; ++m) out[m] = acc[m];
}


// -------------------------------------------------------- dense association
struct DenseParams {
  const double* pts;
  size_t n;
  const DNode* comps;
  int J;
  double outlier_floor;
  double* psum;  // [N] per-point score sum (0: outlier)
  double* partials;
  uint32_t* stamps;
  uint32_t epoch;
  unsigned long long* counters;  // [0] outliers, [1] density evaluations
  int* status;
};

// Pass 1 (association.cpp:66-80): per point the sum of w_j N(y; j).
static __device__ void dense_pass1(const DenseParams& p, const double* Rt, int G, int cta) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = G * (blockDim.x / 32), gw = cta * (blockDim.x / 32) + warp;
  unsigned long long outl = 0;
  for (size_t i = gw; i < p.n; i += nw) {
    double y0, y1, y2;
    apply_rt(Rt, p.pts[3 * i], p.pts[3 * i + 1], p.pts[3 * i + 2], y0, y1, y2);
    double s = 0.0;
    for (int k = lane; k < p.J; k += 32) s += node_score(p.comps + k, y0, y1, y2, p.status);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const bool out = !(s > p.outlier_floor);
    if (lane == 0) {
      p.psum[i] = out ? 0.0 : s;
      outl += out ? 1 : 0;
    }
  }
  if (lane == 0 && outl) atomicAdd(&p.counters[0], outl);
  if (cta == 0 && threadIdx.x == 0)
    atomicAdd(&p.counters[1], (unsigned long long)p.n * (unsigned long long)p.J);
}

// Pass 2 (association.cpp:81-85): lane per component, warps over point
// chunks; each (component, chunk) deposit lands in its own stamped row.
template <int NM>
__device__ void dense_pass2(const DenseParams& p, const double* Rt, int G, int cta) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = G * (blockDim.x / 32), gw = cta * (blockDim.x / 32) + warp;
  const int nb = (p.J + 31) / 32;
  const int nchunks = max(1, min(min(nw / nb, G), (int)((p.n + 7) / 8)));
  const int cb = gw % nb, chunk = gw / nb;
  if (chunk >= nchunks) return;
  const int k = cb * 32 + lane;
  if (k >= p.J) return;
  const size_t c0 = (p.n * (size_t)chunk) / nchunks, c1 = (p.n * (size_t)(chunk + 1)) / nchunks;
  double v[NM];
#pragma unroll
  for (int q = 0; q < NM; ++q) v[q] = 0.0;
  const DNode* g = p.comps + k;
  for (size_t i = c0; i < c1; ++i) {
    const double s = __ldcg(p.psum + i);
    if (!(s > 0.0)) continue;
    double y0, y1, y2;
    apply_rt(Rt, p.pts[3 * i], p.pts[3 * i + 1], p.pts[3 * i + 2], y0, y1, y2);
    const double sc = node_score(g, y0, y1, y2, p.status);
    if (!(sc > 0.0)) continue;
    const double gam = sc / s;
    double d[NM];
    deposit_values<NM>(gam, y0, y1, y2, d);
#pragma unroll
    for (int q = 0; q < NM; ++q) v[q] += d[q];
  }
  const size_t row = (size_t)k * G + chunk;
  double* o = p.partials + row * NM;
#pragma unroll
  for (int q = 0; q < NM; ++q) o[q] = v[q];
  p.stamps[row] = p.epoch;
}

}  // namespace trg
