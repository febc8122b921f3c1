// Device building blocks of the adaptive E-step (K7 associate_descend):
// per-point log-time tree descent (association.cpp:91-157, Algorithm 1 of
// the paper) and the deposit of the per-point sufficient statistics.
//
// Reduction scheme (no float atomics anywhere): points are processed in
// fixed 32-point windows, one warp each; a window's runs of equal stop nodes
// are summed by a segmented warp scan and each run adds its sums to the
// node's exact fixed-point accumulator (trg_fx.cuh).  Integer addition is
// associative, so the totals are bit-identical for any grid, SM budget or
// CTA schedule -- the reference's thread-count invariance
// (parallel.hpp:30-33) -- and nothing reads per-CTA partial rows.
#pragma once
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
  const double q = fast_q(g->mean, g->prec, y0, y1, y2);
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
__device__ __forceinline__ double node_score_nb(const DNode* __restrict__ g, double w, double y0,
                                                double y1, double y2, bool& bad) {
  const double lam2 = g->lam[2];
  const double q = fast_q(g->mean, g->prec, y0, y1, y2);
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
      const int kk = k < count ? k : 0;
      const double v = node_score_nb(sib + kk, sib[kk].weight, y0, y1, y2, bad);
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
  v[1] = __dmul_rn(g, y0);
  v[2] = __dmul_rn(g, y1);
  v[3] = __dmul_rn(g, y2);
  if constexpr (NM == 10) {
    v[4] = __dmul_rn(g, __dmul_rn(y0, y0));
    v[5] = __dmul_rn(g, __dmul_rn(y0, y1));
    v[6] = __dmul_rn(g, __dmul_rn(y0, y2));
    v[7] = __dmul_rn(g, __dmul_rn(y1, y1));
    v[8] = __dmul_rn(g, __dmul_rn(y1, y2));
    v[9] = __dmul_rn(g, __dmul_rn(y2, y2));
  }
}

__device__ __forceinline__ int key_bits_for(int J) { return 32 - __clz((unsigned)J); }

// Transform y = R p + t (geometry.hpp:31) in the reference's order, with
// explicit round-to-nearest operations: the result is the reference's bit
// for bit whatever the including file's -fmad setting (the fused EM and
// calibration kernels contract elsewhere; the descent must not).
__device__ __forceinline__ void apply_rt(const double* Rt, double p0, double p1, double p2,
                                         double& y0, double& y1, double& y2) {
  if (Rt == nullptr) {
    y0 = p0;
    y1 = p1;
    y2 = p2;
    return;
  }
  double s = __dmul_rn(Rt[0], p0);
  s = __dadd_rn(s, __dmul_rn(Rt[1], p1));
  s = __dadd_rn(s, __dmul_rn(Rt[2], p2));
  y0 = __dadd_rn(s, Rt[9]);
  s = __dmul_rn(Rt[3], p0);
  s = __dadd_rn(s, __dmul_rn(Rt[4], p1));
  s = __dadd_rn(s, __dmul_rn(Rt[5], p2));
  y1 = __dadd_rn(s, Rt[10]);
  s = __dmul_rn(Rt[6], p0);
  s = __dadd_rn(s, __dmul_rn(Rt[7], p1));
  s = __dadd_rn(s, __dmul_rn(Rt[8], p2));
  y2 = __dadd_rn(s, Rt[11]);
}

// Scales of the association's accumulators (trg_fx.cuh): deposits are
// g (<= 1), g y and g y y^T with |y| = |R p + t| <= sqrt(3) max|p| + max|t|.
__device__ __forceinline__ void assoc_scales(const double* pmax, const double* Rt, FxScale sc[3]) {
  double y = 1.7320508075688774 * __ldcg(pmax);
  if (Rt) y += fmax(fabs(Rt[9]), fmax(fabs(Rt[10]), fabs(Rt[11])));
  y *= 1.0000001;
  sc[0] = fx_scale(1.0);
  sc[1] = fx_scale(y);
  sc[2] = fx_scale(y * y);
}

// Association pass of one warp over the fixed 32-point windows w = gwarp,
// gwarp + nwarps, ... (association.cpp:91-157): per point the descent, then
// the window's deposits go to the exact accumulators p.acc[J][NM][3]
// (warp_run_deposit).  The totals do not depend on the grid.
template <int NM>
__device__ void assoc_fx_pass(const AssocParams& p, const double* Rt_smem, const FxScale* sc,
                              int nwarps, int gwarp) {
  constexpr int kOrd[10] = {0, 1, 1, 1, 2, 2, 2, 2, 2, 2};
  const int lane = threadIdx.x & 31;
  unsigned long long my_out = 0, my_ev = 0;
  const size_t nwin = (p.n + 31) / 32;
  for (size_t w = gwarp; w < nwin; w += nwarps) {
    const size_t i = w * 32 + lane;
    int key = -1;
    double v[NM];
#pragma unroll
    for (int m = 0; m < NM; ++m) v[m] = 0.0;
    if (i < p.n) {
      double y0, y1, y2;
      apply_rt(Rt_smem, p.pts[3 * i], p.pts[3 * i + 1], p.pts[3 * i + 2], y0, y1, y2);
      const Descent d = descend(p.nodes, p.snodes, p.n_snodes, p.root_count, p.depth, p.lambda_c,
                                p.outlier_floor, y0, y1, y2, p.status);
      my_ev += d.evals;
      if (d.node < 0) {
        ++my_out;
      } else {
        key = d.node;
        deposit_values<NM>(d.path, y0, y1, y2, v);
      }
      if (p.point_node) {
        p.point_node[i] = d.node;
        p.point_w[i] = d.node < 0 ? 0.0 : d.path;
      }
    }
    __syncwarp();
#ifdef TRG_ASSOC_PROBE
    if (lane == 0 && (gwarp % 32) == 0 && p.tl) tl_mark_any(p.tl, 5101);
#endif
    warp_run_deposit<NM>(key, v, p.acc, p.acc_stride, sc, kOrd);
#ifdef TRG_ASSOC_PROBE
    if (lane == 0 && (gwarp % 32) == 0 && p.tl) tl_mark_any(p.tl, 5102);
#endif
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    my_out += __shfl_xor_sync(0xffffffffu, my_out, off);
    my_ev += __shfl_xor_sync(0xffffffffu, my_ev, off);
  }
  if (lane == 0 && (my_out | my_ev)) {
    atomicAdd(&p.counters[0], my_out);
    atomicAdd(&p.counters[1], my_ev);
  }
}

// ------------------------------------------------------------ FP32 fast path
// (trg_reg_config.fast_scoring) The EM's descent with FP32
// scores: per node a 64-byte record (mean kept FP64 so the point-minus-mean
// difference is exact to FP64 rounding, precision matrix and log(w) +
// log_norm in FP32), the argmax and normaliser in the log domain (the
// maximum's sibling has score ratio 1, the path weight is 1 / sum of
// exp(ls_k - max)), the reference's underflow rules as log-thresholds.
struct __align__(16) FNode {
  double mean[3];
  float prec[6];   // fast_q's packed precision matrix
  float lwn;       // log(weight) + log_norm; -inf when weight == 0 (or not PD)
  float cplx;      // node complexity (-1: no positive trace)
  int first_child;
  short child_count;
  short bad;       // weight > 0 but the covariance is not PD (log_density throws)
};
static_assert(sizeof(FNode) == 64, "FNode layout");

__device__ __forceinline__ void fnode_from(const DNode& d, FNode& f) {
  for (int i = 0; i < 3; ++i) f.mean[i] = d.mean[i];
  for (int i = 0; i < 6; ++i) f.prec[i] = (float)d.prec[i];
  const bool live = d.weight > 0.0, pd = d.lam[2] > 0.0;
  f.lwn = (live && pd) ? (float)(log(d.weight) + d.log_norm) : -INFINITY;
  f.cplx = (float)d.cplx;
  f.first_child = d.first_child;
  f.child_count = (short)d.child_count;
  f.bad = (live && !pd) ? 1 : 0;
}

__device__ __forceinline__ Descent descend_f32(const FNode* __restrict__ nodes, const FNode* snodes,
                                               int n_snodes, int root_count, int depth,
                                               float lambda_c, double y0, double y1, double y2,
                                               int* status) {
  Descent r{-1, 1.0, 0};
  int node = -1;
  for (int l = 0; l < depth; ++l) {
    const FNode* cur = node < n_snodes ? snodes + node : nodes + node;
    const int first = node < 0 ? 0 : cur->first_child;
    const int count = node < 0 ? root_count : cur->child_count;
    const FNode* sib = first + count <= n_snodes ? snodes + first : nodes + first;
    float ls[8];
    bool bad = false;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const FNode& g = sib[k < count ? k : 0];
      const float d0 = (float)(y0 - g.mean[0]), d1 = (float)(y1 - g.mean[1]), d2 = (float)(y2 - g.mean[2]);
      const float u0 = fmaf(g.prec[2], d2, fmaf(g.prec[1], d1, g.prec[0] * d0));
      const float u1 = fmaf(g.prec[4], d2, g.prec[3] * d1);
      const float q = fmaf(d0, u0, fmaf(d1, u1, g.prec[5] * d2 * d2));
      bad = bad || (k < count && g.bad);
      ls[k] = k < count ? fmaf(-0.5f, q, g.lwn) : -INFINITY;
    }
    if (bad) atomicCAS(status, 0, kEDomain);  // log_density: covariance is not PD
    float m = ls[0];
    int best = 0;
#pragma unroll
    for (int k = 1; k < 8; ++k)
      if (ls[k] > m) {  // strict '>' : lowest index wins ties
        m = ls[k];
        best = k;
      }
    float s = 0.0f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += __expf(ls[k] - m);
    r.evals += count;
    const float logsum = m + __logf(s);  // NaN when every score is -inf
    if (l == 0 && !(logsum > -690.7755f)) {  // sum <= 1e-300: outlier
      r.node = -1;
      return r;
    }
    if (!(logsum > -744.44f)) break;  // the FP64 sum would underflow to 0: keep the current node
    node = first + best;
    r.path *= (double)(1.0f / s);
    const FNode* nd = sib + best;
    if (nd->child_count == 0) break;
    if (nd->cplx < 0.0f) {
      atomicCAS(status, 0, kEDomain);  // node_complexity: no positive trace
      break;
    }
    if (nd->cplx <= lambda_c) break;
  }
  r.node = node;
  return r;
}

// assoc_fx_pass with the FP32 descent (same windows, deposits and counters).
template <int NM>
__device__ void assoc_fx_pass_f32(const AssocParams& p, const FNode* fnodes, const FNode* fstage,
                                  const double* Rt_smem, const FxScale* sc, int nwarps, int gwarp) {
  constexpr int kOrd[10] = {0, 1, 1, 1, 2, 2, 2, 2, 2, 2};
  const int lane = threadIdx.x & 31;
  unsigned long long my_out = 0, my_ev = 0;
  const size_t nwin = (p.n + 31) / 32;
  const float lc = (float)p.lambda_c;
  for (size_t w = gwarp; w < nwin; w += nwarps) {
    const size_t i = w * 32 + lane;
    int key = -1;
    double v[NM];
#pragma unroll
    for (int m = 0; m < NM; ++m) v[m] = 0.0;
    if (i < p.n) {
      double y0, y1, y2;
      apply_rt(Rt_smem, p.pts[3 * i], p.pts[3 * i + 1], p.pts[3 * i + 2], y0, y1, y2);
      const Descent d = descend_f32(fnodes, fstage, p.n_snodes, p.root_count, p.depth, lc, y0, y1,
                                    y2, p.status);
      my_ev += d.evals;
      if (d.node < 0) {
        ++my_out;
      } else {
        key = d.node;
        deposit_values<NM>(d.path, y0, y1, y2, v);
      }
    }
    __syncwarp();
    warp_run_deposit<NM>(key, v, p.acc, p.acc_stride, sc, kOrd);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    my_out += __shfl_xor_sync(0xffffffffu, my_out, off);
    my_ev += __shfl_xor_sync(0xffffffffu, my_ev, off);
  }
  if (lane == 0 && (my_out | my_ev)) {
    atomicAdd(&p.counters[0], my_out);
    atomicAdd(&p.counters[1], my_ev);
  }
}

// Stages nodes [0, S) into shared memory with one bulk copy (TMA engine),
// completing on `bar` (phase bit `phase`, flipped on return).  Block-wide;
// the nodes may have been rewritten by other CTAs before the caller's last
// grid barrier.
// In two halves, so that a caller can overlap the copy with other loads.
__device__ __forceinline__ void stage_nodes_issue(DNode* snodes, const DNode* nodes, int S,
                                                  uint64_t* bar) {
  if (S <= 0) return;
  __syncthreads();  // every reader of the previous stage is done
  if (threadIdx.x == 0) {
    fence_proxy_async_shared();
    fence_proxy_async_global();
    bulk_g2s_issue(snodes, nodes, (unsigned)(S * sizeof(DNode)), bar);
  }
}
__device__ __forceinline__ void stage_nodes_wait(int S, uint64_t* bar, unsigned& phase) {
  if (S <= 0) return;
  if (threadIdx.x == 0) mbar_wait(bar, phase);
  __syncthreads();
  phase ^= 1u;
}
__device__ __forceinline__ void stage_nodes_bulk(DNode* snodes, const DNode* nodes, int S,
                                                 uint64_t* bar, unsigned& phase) {
  stage_nodes_issue(snodes, nodes, S, bar);
  stage_nodes_wait(S, bar, phase);
}

// Node j's NM values from the planar accumulators.
template <int NM>
__device__ __forceinline__ void fx_row(const long long* acc, size_t stride, int j, const FxScale* sc,
                                       double out[NM]) {
  constexpr int kOrd[10] = {0, 1, 1, 1, 2, 2, 2, 2, 2, 2};
#pragma unroll
  for (int m = 0; m < NM; ++m) out[m] = fx_load(acc, stride, j, m, sc[kOrd[m]].down);
}

}  // namespace trg
