// Device building blocks of the adaptive E-step (K7 associate_descend):
// per-point log-time tree descent (association.cpp:91-157, Algorithm 1 of
// the paper) and the deterministic per-CTA reduction of the deposits.
//
// Reduction scheme (no float atomics anywhere): each CTA processes tiles of
// 256 points; per tile the (stop node, deposit) pairs are stably radix-sorted
// by node inside the block, reduced by a segmented scan, and each segment
// tail adds its sum into this CTA's private row of the partial table
// partials[node][cta][NM] (epoch-stamped, so nothing is zeroed between
// calls).  A combine pass then sums each node over CTAs in fixed order.
#pragma once
#include <cub/block/block_radix_sort.cuh>

#include "trg_internal.cuh"

namespace trg {

constexpr int kAssocBlock = 256;

// gmm.cpp:37-51 log_density / density, association.cpp:129 score.
// Evaluation order is the reference's (see oracle/trg_oracle.c log_density).
// Every field is loaded before any test, so one node costs one memory round
// trip (the eight siblings' loads are all in flight together).
__device__ __forceinline__ double node_score(const DNode* __restrict__ g, double y0, double y1,
                                             double y2, int* status) {
  const double w = g->weight;
  const double lam2 = g->lam[2];
  const double q = fast_q(g->mean, g->axT, g->il, y0, y1, y2);
  const double sc = __dmul_rn(w, trg_exp(__fma_rn(-0.5, q, g->log_norm)));
  if (!(w > 0.0)) return 0.0;
  if (!(lam2 > 0.0)) {
    atomicCAS(status, 0, kEDomain);  // log_density: covariance is not PD
    return 0.0;
  }
  return sc;
}

// Score for the descent without an early return, so the <= 8 sibling
// evaluations are straight-line code; `bad` collects the non-PD error.
__device__ __forceinline__ double node_score_nb(const DNode* __restrict__ g, double y0, double y1,
                                                double y2, bool& bad) {
  const double w = g->weight;
  const double lam2 = g->lam[2];
  const double q = fast_q(g->mean, g->axT, g->il, y0, y1, y2);
  const double sc = __dmul_rn(w, trg_exp(__fma_rn(-0.5, q, g->log_norm)));
  const bool live = w > 0.0;
  bad = bad || (live && !(lam2 > 0.0));
  return (live && lam2 > 0.0) ? sc : 0.0;
}

struct Descent {
  int node;       // stop node, -1 = outlier
  double path;    // product of sibling-normalised responsibilities
  uint32_t evals; // density evaluations
};

// association.cpp:117-150 for one transformed point y.
__device__ __forceinline__ Descent descend(const DNode* __restrict__ nodes, const DNode* snodes,
                                           int n_snodes, int root_count, int depth,
                                           double lambda_c, double outlier_floor, double y0,
                                           double y1, double y2, int* status) {
  Descent r{-1, 1.0, 0};
  int node = -1;
#ifdef TRG_DESCENT_PROBE
  long long tp[8];
  int np = 0;
  tp[np++] = clock64();
#endif
  for (int l = 0; l < depth; ++l) {
    const DNode* cur = node < n_snodes ? snodes + node : nodes + node;
    const int first = node < 0 ? 0 : cur->first_child;
    const int count = node < 0 ? root_count : cur->child_count;
    // siblings from the shared-memory stage when the whole run is staged
    const DNode* sib = first + count <= n_snodes ? snodes + first : nodes + first;
    // the <= 8 sibling scores are independent: evaluate them together (ILP),
    // then sum and arg-max in sibling order exactly like the reference
    double sc[8];
    bool bad = false;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const double v = node_score_nb(sib + (k < count ? k : 0), y0, y1, y2, bad);
      sc[k] = k < count ? v : 0.0;
    }
    if (bad) atomicCAS(status, 0, kEDomain);  // log_density: covariance is not PD
    double sum = 0.0, best_s = 0.0;
    int best = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (k >= count) break;
      sum += sc[k];
      if (k == 0 || sc[k] > best_s) {  // strict '>' : lowest index wins ties
        best_s = sc[k];
        best = k;
      }
    }
    r.evals += count;
    if (l == 0 && !(sum > outlier_floor)) {
      r.node = -1;
      return r;
    }
    if (!(sum > 0.0)) break;  // deeper underflow: keep the current node
    node = first + best;
    r.path *= best_s / sum;
    const DNode* nd = sib + best;
    if (nd->child_count == 0) break;
    if (nd->cplx < 0.0) {
      atomicCAS(status, 0, kEDomain);  // node_complexity: no positive trace
      break;
    }
    if (nd->cplx <= lambda_c) break;
#ifdef TRG_DESCENT_PROBE
    tp[np++] = clock64();
#endif
  }
#ifdef TRG_DESCENT_PROBE
  tp[np++] = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0 && lambda_c == 0.0)
    printf("descent cycles: %lld %lld %lld (levels %d)\n", np > 1 ? tp[1] - tp[0] : -1LL,
           np > 2 ? tp[2] - tp[1] : -1LL, np > 3 ? tp[3] - tp[2] : -1LL, np - 1);
#endif
  r.node = node;
  return r;
}

// Upper levels staged per CTA (18 KB): the descent's first L-1 levels then
// read shared memory; the last level reads global memory.
constexpr int kStageNodes = 96;

// Copies nodes [0, S) into the stage (16-byte loads through L2: another CTA
// may have rewritten them since this SM last read them).  Block-wide.
__device__ __forceinline__ void stage_nodes(DNode* snodes, const DNode* __restrict__ nodes, int S) {
  const int4* src = reinterpret_cast<const int4*>(nodes);
  int4* dst = reinterpret_cast<int4*>(snodes);
  const int n16 = S * (int)(sizeof(DNode) / 16);
  for (int i = threadIdx.x; i < n16; i += blockDim.x) dst[i] = __ldcg(src + i);
  __syncthreads();
}

// Deposit vector of one point (association.cpp:20-23): NM = 4 -> (g, g y),
// NM = 10 adds the 6 unique entries of g (y y^T).
template <int NM>
__device__ __forceinline__ void deposit_values(double g, double y0, double y1, double y2,
                                               double v[NM]) {
  v[0] = g;
  v[1] = g * y0;
  v[2] = g * y1;
  v[3] = g * y2;
  if constexpr (NM == 10) {
    v[4] = g * (y0 * y0);
    v[5] = g * (y0 * y1);
    v[6] = g * (y0 * y2);
    v[7] = g * (y1 * y1);
    v[8] = g * (y1 * y2);
    v[9] = g * (y2 * y2);
  }
}

template <int NM>
struct AssocSmem {
  using Sort = cub::BlockRadixSort<unsigned, kAssocBlock, 1, int>;
  typename Sort::TempStorage sort;
  double vals_copy[kAssocBlock][NM];
  unsigned skeys[kAssocBlock];
  double warp_v[kAssocBlock / 32][NM];
  int warp_f[kAssocBlock / 32];
  double carry[kAssocBlock / 32][NM];
  unsigned long long outliers, evals;
};

// Reduces one tile's deposits (key = node or >= J for "none") into the CTA's
// row of the partial table.  Must be called by all threads of the block.
template <int NM>
__device__ void tile_reduce(AssocSmem<NM>& sm, unsigned key, const double v[NM], int J,
                            int key_bits, double* __restrict__ partials,
                            uint32_t* __restrict__ stamps, uint32_t epoch, int G, int cta) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#pragma unroll
  for (int m = 0; m < NM; ++m) sm.vals_copy[tid][m] = v[m];
  unsigned k1[1] = {key};
  int i1[1] = {tid};
  __syncthreads();
  typename AssocSmem<NM>::Sort(sm.sort).Sort(k1, i1, 0, key_bits);
  sm.skeys[tid] = k1[0];
  __syncthreads();
  const unsigned k = k1[0];
  double x[NM];
#pragma unroll
  for (int m = 0; m < NM; ++m) x[m] = sm.vals_copy[i1[0]][m];
  const bool head = (tid == 0) || sm.skeys[tid - 1] != k;
  const bool tail = (tid == kAssocBlock - 1) || sm.skeys[tid + 1] != k;
  // warp-level inclusive segmented scan: (v, f) op: f_r ? v_r : v_l + v_r
  int f = head ? 1 : 0;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    double o[NM];
#pragma unroll
    for (int m = 0; m < NM; ++m) o[m] = __shfl_up_sync(0xffffffffu, x[m], off);
    const int of = __shfl_up_sync(0xffffffffu, f, off);
    if (lane >= off) {
      if (!f) {
#pragma unroll
        for (int m = 0; m < NM; ++m) x[m] = o[m] + x[m];
      }
      f |= of;
    }
  }
  if (lane == 31) {
#pragma unroll
    for (int m = 0; m < NM; ++m) sm.warp_v[warp][m] = x[m];
    sm.warp_f[warp] = f;
  }
  __syncthreads();
  if (tid == 0) {
    // carry into warp w = inclusive value at the last item of warp w-1
#pragma unroll
    for (int m = 0; m < NM; ++m) sm.carry[0][m] = 0.0;
    for (int w = 1; w < kAssocBlock / 32; ++w)
#pragma unroll
      for (int m = 0; m < NM; ++m)
        sm.carry[w][m] = sm.warp_f[w - 1] ? sm.warp_v[w - 1][m]
                                          : sm.carry[w - 1][m] + sm.warp_v[w - 1][m];
  }
  __syncthreads();
  if (!f && warp > 0) {
#pragma unroll
    for (int m = 0; m < NM; ++m) x[m] = sm.carry[warp][m] + x[m];
  }
  if (tail && k < (unsigned)J) {
    const size_t row = (size_t)k * G + cta;
    double* p = partials + row * NM;
    if (stamps[row] == epoch) {
#pragma unroll
      for (int m = 0; m < NM; ++m) p[m] = p[m] + x[m];
    } else {
#pragma unroll
      for (int m = 0; m < NM; ++m) p[m] = x[m];
      stamps[row] = epoch;
    }
  }
  __syncthreads();
}

__device__ __forceinline__ int key_bits_for(int J) { return 32 - __clz((unsigned)J); }

// Transform y = R p + t (geometry.hpp:31) in the reference's order.
__device__ __forceinline__ void apply_rt(const double* Rt, double p0, double p1, double p2,
                                         double& y0, double& y1, double& y2) {
  if (Rt == nullptr) {
    y0 = p0;
    y1 = p1;
    y2 = p2;
    return;
  }
  double s = Rt[0] * p0;
  s += Rt[1] * p1;
  s += Rt[2] * p2;
  y0 = s + Rt[9];
  s = Rt[3] * p0;
  s += Rt[4] * p1;
  s += Rt[5] * p2;
  y1 = s + Rt[10];
  s = Rt[6] * p0;
  s += Rt[7] * p1;
  s += Rt[8] * p2;
  y2 = s + Rt[11];
}

// Association pass of one CTA over tiles cta, cta+G, ... (persistent).
template <int NM>
__device__ void assoc_pass(AssocSmem<NM>& sm, const AssocParams& p, const double* Rt_smem, int G,
                           int cta, int tile_G = -1, int tile_cta = -1) {
  // tiles are dealt over tile_G CTAs (default: all G); partial rows stay
  // indexed by the CTA's own id among G
  const int tG = tile_G < 0 ? G : tile_G, tc = tile_G < 0 ? cta : tile_cta;
  const int tid = threadIdx.x;
  const int J = p.n_nodes;
  const int kb = key_bits_for(J);
  if (tid == 0) {
    sm.outliers = 0;
    sm.evals = 0;
  }
  __syncthreads();
  unsigned long long my_out = 0, my_ev = 0;
  // tiles of ts <= 256 points: when the cloud is small for the grid, spread
  // it evenly over all CTAs (every SM gets the same share of descents)
  const size_t per_cta = (p.n + tG - 1) / tG;
  const int ts = per_cta < (size_t)kAssocBlock ? (per_cta > 0 ? (int)per_cta : 1) : kAssocBlock;
  const size_t ntiles = (p.n + ts - 1) / ts;
  for (size_t tile = tc; tile < ntiles; tile += tG) {
    const size_t i = tile * ts + tid;
    unsigned key = (unsigned)J;
    double v[NM];
#pragma unroll
    for (int m = 0; m < NM; ++m) v[m] = 0.0;
    if (tid < ts && i < p.n) {
      double y0, y1, y2;
      apply_rt(Rt_smem, p.pts[3 * i], p.pts[3 * i + 1], p.pts[3 * i + 2], y0, y1, y2);
      Descent d;
      if (p.dbg_mode == 2) {
        d.node = (int)(i % (size_t)J);
        d.path = 0.5;
        d.evals = 1;
      } else {
        d = descend(p.nodes, p.snodes, p.n_snodes, p.root_count, p.depth, p.lambda_c,
                    p.outlier_floor, y0, y1, y2, p.status);
      }
      my_ev += d.evals;
      if (d.node < 0) {
        ++my_out;
      } else {
        key = (unsigned)d.node;
        deposit_values<NM>(d.path, y0, y1, y2, v);
      }
      if (p.point_node) {
        p.point_node[i] = d.node;
        p.point_w[i] = d.node < 0 ? 0.0 : d.path;
      }
    }
    // reconverge before the block-wide sort (CUB's warp-level steps assume
    // converged warps; the descent above diverges per point)
    __syncwarp();
    if (p.dbg_mode != 1) tile_reduce<NM>(sm, key, v, J, kb, p.partials, p.stamps, p.epoch, G, cta);
    else if (key < (unsigned)J) p.partials[key] += v[0] * 0.0;
  }
  // integer counters: warp shuffle sums, then one add per warp (no 64-bit
  // shared-memory CAS loops)
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    my_out += __shfl_xor_sync(0xffffffffu, my_out, off);
    my_ev += __shfl_xor_sync(0xffffffffu, my_ev, off);
  }
  if ((tid & 31) == 0 && (my_out | my_ev)) {
    atomicAdd(&p.counters[0], my_out);
    atomicAdd(&p.counters[1], my_ev);
  }
}

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

}  // namespace trg
