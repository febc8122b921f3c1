// K8 mstep_solve_block: make_virtual_points + solve_mstep (mstep.cpp:8-99)
// as single-thread-block device code, plus the grid barrier used by the
// persistent kernels.
#pragma once
#include "trg_assoc.cuh"

namespace trg {

// ------------------------------------------------------------ grid barrier
// Sense-free generation barrier over all CTAs of a cooperative launch.
// bar[0] = arrival counter, bar[1] = generation.  The trailing
// __threadfence() (MEMBAR.GPU + L1 invalidate on sm_100) makes other CTAs'
// writes visible to ordinary loads after the barrier.
__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* vb = bar;
    const unsigned gen = vb[1];
    __threadfence();
    const unsigned arrived = atomicAdd(&bar[0], 1u);
    if (arrived == nblocks - 1) {
      atomicExch(&bar[0], 0u);
      __threadfence();
      atomicAdd(&bar[1], 1u);
    } else {
      while (vb[1] == gen) __nanosleep(20);
    }
    __threadfence();
  }
  __syncthreads();
}

// Loads that bypass L1 for data other CTAs wrote in this kernel.
__device__ __forceinline__ double ldcg(const double* p) { return __ldcg(p); }

// ------------------------------------------------------------ VP rows
constexpr int kNormalEq = 27;  // 21 (upper ata) + 6 (atb)

struct SolveAcc {
  double v[kNormalEq];
  double crit;  // criterion at identity (mstep.cpp:32-47)
  int nvp;
};

__device__ __forceinline__ void acc_zero(SolveAcc& a) {
#pragma unroll
  for (int k = 0; k < kNormalEq; ++k) a.v[k] = 0.0;
  a.crit = 0.0;
  a.nvp = 0;
}

// Virtual point of node j (mstep.cpp:18-26) and its three weighted rows
// (mstep.cpp:58-75) added to `a`; criterion terms at identity too.
__device__ __forceinline__ void vp_accumulate(const DNode* __restrict__ g, double m0, double m10,
                                              double m11, double m12, double n_total,
                                              SolveAcc& a, int* status) {
  const double floor_mass = 1e-8 * n_total;
  if (m0 <= floor_mass) return;
  const double pi = m0 / n_total;
  const double mu[3] = {m10 / m0, m11 / m0, m12 / m0};
  a.nvp += 1;
  const double lf = 1e-6 * g->lam[0];
  const double e[3] = {g->mean[0] - mu[0], g->mean[1] - mu[1], g->mean[2] - mu[2]};
  const double d[3] = {mu[0] - g->mean[0], mu[1] - g->mean[1], mu[2] - g->mean[2]};
#pragma unroll
  for (int l = 0; l < 3; ++l) {
    const double* nr = g->axT + 3 * l;
    const double lam = smax(g->lam[l], lf);
    if (!(lam > 0.0) || !(g->lam[l] > 0.0)) {
      atomicCAS(status, 0, kEDomain);
      return;
    }
    const double w = sqrt(pi / lam);
    const double cr0 = mu[1] * nr[2] - mu[2] * nr[1];
    const double cr1 = mu[2] * nr[0] - mu[0] * nr[2];
    const double cr2 = mu[0] * nr[1] - mu[1] * nr[0];
    const double row[6] = {w * cr0, w * cr1, w * cr2, w * nr[0], w * nr[1], w * nr[2]};
    double dt = nr[0] * e[0];
    dt += nr[1] * e[1];
    dt += nr[2] * e[2];
    const double rhs = w * dt;
    int k = 0;
#pragma unroll
    for (int i = 0; i < 6; ++i)
#pragma unroll
      for (int j = i; j < 6; ++j) a.v[k++] += row[i] * row[j];
#pragma unroll
    for (int i = 0; i < 6; ++i) a.v[21 + i] += row[i] * rhs;
    // criterion at identity: r = n . (mu - mean)
    double r = nr[0] * d[0];
    r += nr[1] * d[1];
    r += nr[2] * d[2];
    a.crit += pi / g->lam[l] * r * r;
  }
}

// Criterion after the update delta (mstep.cpp:32-47 with t = delta).
__device__ __forceinline__ double crit_term(const DNode* __restrict__ g, double m0, double m10,
                                            double m11, double m12, double n_total,
                                            const double* dRt) {
  if (m0 <= 1e-8 * n_total) return 0.0;
  const double pi = m0 / n_total;
  const double mu0 = m10 / m0, mu1 = m11 / m0, mu2 = m12 / m0;
  double y0, y1, y2;
  apply_rt(dRt, mu0, mu1, mu2, y0, y1, y2);
  const double d[3] = {y0 - g->mean[0], y1 - g->mean[1], y2 - g->mean[2]};
  double c = 0.0;
#pragma unroll
  for (int l = 0; l < 3; ++l) {
    const double* nr = g->axT + 3 * l;
    double r = nr[0] * d[0];
    r += nr[1] * d[1];
    r += nr[2] * d[2];
    c += pi / g->lam[l] * r * r;
  }
  return c;
}

// Deterministic block reduction of a SolveAcc (fixed shuffle pattern, warps
// combined in index order).  Result valid in thread 0.
struct SolveSmem {
  double warp[32][kNormalEq + 1];
  int nvp[32];
  double scratch[kNormalEq + 2];
};

__device__ __forceinline__ void block_reduce_acc(SolveAcc& a, SolveSmem& sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int k = 0; k < kNormalEq; ++k) a.v[k] += __shfl_xor_sync(0xffffffffu, a.v[k], off);
    a.crit += __shfl_xor_sync(0xffffffffu, a.crit, off);
    a.nvp += __shfl_xor_sync(0xffffffffu, a.nvp, off);
  }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < kNormalEq; ++k) sm.warp[warp][k] = a.v[k];
    sm.warp[warp][kNormalEq] = a.crit;
    sm.nvp[warp] = a.nvp;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < nw; ++w) {
#pragma unroll
      for (int k = 0; k < kNormalEq; ++k) a.v[k] += sm.warp[w][k];
      a.crit += sm.warp[w][kNormalEq];
      a.nvp += sm.nvp[w];
    }
  }
  __syncthreads();
}

__device__ __forceinline__ double block_sum(double v, SolveSmem& sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  if (lane == 0) sm.warp[warp][0] = v;
  __syncthreads();
  if (threadIdx.x == 0)
    for (int w = 1; w < nw; ++w) v += sm.warp[w][0];
  __syncthreads();
  return v;
}

struct SolveOut {
  double omega[3], trans[3], dR[9], dt[3];
  double crit_before, crit_after, cond;
  int nvp;
  int degenerate;  // 1: fewer than 3 VPs or cond >= 1e12 (DegenerateGeometryError)
};

// Thread-0 part of solve_mstep (mstep.cpp:76-98) from the reduced normal
// equations.  __noinline__ keeps its 6x6 working set out of the callers'
// register budget.
static __device__ __noinline__ void solve_normal_eq(const double* v, int nvp, SolveOut* o) {
  o->nvp = nvp;
  o->degenerate = 0;
  if (nvp < 3) {
    o->degenerate = 1;
    return;
  }
  double ata[6][6], b[6], work[6][6], ev[6], vec[6][6];
  int k = 0;
  for (int i = 0; i < 6; ++i)
    for (int j = i; j < 6; ++j) {
      ata[i][j] = v[k];
      ata[j][i] = v[k];
      ++k;
    }
  for (int i = 0; i < 6; ++i) b[i] = v[21 + i];
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 6; ++j) work[i][j] = ata[i][j];
  jacobi_eig<6>(work, ev, vec);
  const double lmin = ev[0], lmax = ev[5];
  const double cond = lmin > 0.0 ? lmax / lmin : INFINITY;
  o->cond = cond;
  if (!(cond < 1e12)) {
    o->degenerate = 1;
    return;
  }
  double x[6];
  ldlt_solve6(ata, b, x);
  for (int i = 0; i < 3; ++i) {
    o->omega[i] = x[i];
    o->trans[i] = x[3 + i];
    o->dt[i] = x[3 + i];
  }
  small_angle_rotation(o->omega, o->dR);
}

// Whole solve on one block from device moments (stride nm, m0 at 0, m1 at 1..3).
static __device__ void block_solve(const DNode* __restrict__ nodes, int J, const double* __restrict__ mom,
                            int nm, double n_total, SolveOut* out, SolveSmem& sm, int* status) {
  SolveAcc a;
  acc_zero(a);
  for (int j = threadIdx.x; j < J; j += blockDim.x) {
    const double* m = mom + (size_t)j * nm;
    vp_accumulate(nodes + j, ldcg(m), ldcg(m + 1), ldcg(m + 2), ldcg(m + 3), n_total, a, status);
  }
  block_reduce_acc(a, sm);
  __shared__ SolveOut so;
  if (threadIdx.x == 0) {
    so.crit_before = a.crit;
    solve_normal_eq(a.v, a.nvp, &so);
  }
  __syncthreads();
  double c = 0.0;
  if (!so.degenerate) {
    double dRt[12];
    for (int i = 0; i < 9; ++i) dRt[i] = so.dR[i];
    for (int i = 0; i < 3; ++i) dRt[9 + i] = so.dt[i];
    for (int j = threadIdx.x; j < J; j += blockDim.x) {
      const double* m = mom + (size_t)j * nm;
      c += crit_term(nodes + j, ldcg(m), ldcg(m + 1), ldcg(m + 2), ldcg(m + 3), n_total, dRt);
    }
  }
  c = block_sum(c, sm);
  if (threadIdx.x == 0) {
    so.crit_after = so.degenerate ? so.crit_before : c;
    *out = so;
  }
  __syncthreads();
}

}  // namespace trg
