// K8 mstep_solve_block: make_virtual_points + solve_mstep (mstep.cpp:8-99)
// as single-thread-block device code, plus the grid barrier used by the
// persistent kernels.
#pragma once
#include "trg_assoc.cuh"

namespace trg {

// ------------------------------------------------------------ grid barrier
// Counting barrier over all CTAs of a persistent launch: bar[0] only ever
// grows (zeroed per job); the CTA whose arrival returns `old` waits for the
// count to reach the next multiple of nblocks.  Thread 0 arrives with a
// GPU-scope acquire-release atomic (releases the writes of the whole CTA,
// ordered before it by the CTA barrier) and polls with acquire loads (which
// also drop the SM's stale L1 lines), then the CTA barrier hands the
// ordering to every thread.  Measured 1.2 us per barrier at 444 CTAs, against
// 2.7 us for the generation barrier with __threadfence (MEMBAR.SC) it
// replaced.
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned atom_add_acq_rel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned old = atom_add_acq_rel(&bar[0], 1u);
    const unsigned target = (old / nblocks + 1u) * nblocks;
    if (old + 1u != target) {
      unsigned ns = 32, polls = 0;
      const unsigned long long t0 = gtimer();
      while ((int)(ld_acquire_u32(&bar[0]) - target) < 0) {
        __nanosleep(ns);
        ns = ns < 128 ? 2 * ns : 128;
        spin_guard_every(t0, polls);
      }
    }
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
__device__ __forceinline__ void vp_rows(const DNode* __restrict__ g, double pi, const double mu[3],
                                        SolveAcc& a, int* status);

__device__ __forceinline__ void vp_accumulate(const DNode* __restrict__ g, double m0, double m10,
                                              double m11, double m12, double n_total,
                                              SolveAcc& a, int* status) {
  const double floor_mass = 1e-8 * n_total;
  if (m0 <= floor_mass) return;
  const double pi = m0 / n_total;
  const double mu[3] = {m10 / m0, m11 / m0, m12 / m0};
  vp_rows(g, pi, mu, a, status);
}

// The three weighted rows of one virtual point (mstep.cpp:58-75) and its
// criterion terms at identity.
__device__ __forceinline__ void vp_rows(const DNode* __restrict__ g, double pi, const double mu[3],
                                        SolveAcc& a, int* status) {
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
  int eig_sweeps;  // diagnostics
};

// Eigenvalues of the 6x6 normal matrix (mstep.cpp:77-80, condition
// estimate) by a WARP-parallel Jacobi: round-robin ordering, 3 disjoint
// rotations per step (5 steps per sweep), all 36 entries updated at once.
// Same per-rotation formulas and skip threshold as the cyclic solver; only
// the rotation order differs (eigenvalues agree to a few ulp).
// Round-robin tournament for 6 indices: round r pairs kRR6[r][k] (p < q).
static __constant__ int kRR6[5][3][2] = {{{0, 5}, {1, 4}, {2, 3}}, {{0, 4}, {3, 5}, {1, 2}},
                                         {{0, 3}, {2, 4}, {1, 5}}, {{0, 2}, {1, 3}, {4, 5}},
                                         {{0, 1}, {2, 5}, {3, 4}}};
// Per round and index: partner, rotation slot, and whether it is the pair's p.
static __constant__ signed char kPart6[5][6] = {{5, 4, 3, 2, 1, 0}, {4, 2, 1, 5, 0, 3},
                                                {3, 5, 4, 0, 2, 1}, {2, 3, 0, 1, 5, 4},
                                                {1, 0, 5, 4, 3, 2}};
static __constant__ signed char kSlot6[5][6] = {{0, 1, 2, 2, 1, 0}, {0, 2, 2, 1, 0, 1},
                                                {0, 2, 1, 0, 1, 2}, {0, 1, 0, 1, 2, 2},
                                                {0, 0, 1, 2, 2, 1}};

struct Eig6Smem {
  double a[36], b[36];
  double c[3], s[3], t[3];
  int rotated;
  int sweeps;
  signed char part[5][6], slot[5][6], pq[5][3][2];  // smem copies of the tables
};

// Called by all 32 lanes of ONE warp; returns eigenvalues ascending in ev.
// Skips a rotation when |a_pq| is negligible next to both diagonal entries
// (the cyclic solver's test) or below 1e-13 sqrt|a_pp a_qq| (its effect on
// the eigenvalues is then far below rounding).
static __device__ void warp_eig6(const double* in, double ev[6], Eig6Smem& w) {
  const int lane = threadIdx.x & 31;
  for (int i = lane; i < 36; i += 32) w.a[i] = in[i];
  // lane-divergent reads of __constant__ tables serialize: stage them in smem
  if (lane < 30) {
    w.part[lane / 6][lane % 6] = kPart6[lane / 6][lane % 6];
    w.slot[lane / 6][lane % 6] = kSlot6[lane / 6][lane % 6];
    w.pq[lane / 6][(lane % 6) / 2][lane & 1] = (signed char)kRR6[lane / 6][(lane % 6) / 2][lane & 1];
  }
  __syncwarp();
  for (int sweep = 0; sweep < 64; ++sweep) {
    if (lane == 0) w.rotated = 0;
    __syncwarp();
    for (int r = 0; r < 5; ++r) {
      if (lane < 3) {
        const int p = w.pq[r][lane][0], q = w.pq[r][lane][1];
        const double apq = w.a[6 * p + q], app = w.a[7 * p], aqq = w.a[7 * q];
        double c = 1.0, sn = 0.0, t = 0.0;
        const double g = 100.0 * fabs(apq);
        const bool negligible = (fabs(app) + g == fabs(app) && fabs(aqq) + g == fabs(aqq)) ||
                                fabs(apq) <= 1e-13 * sqrt(fabs(app) * fabs(aqq));
        if (apq != 0.0 && !negligible) {
          w.rotated = 1;
          const double h = aqq - app;
          if (fabs(h) + g == fabs(h)) {
            t = apq * __drcp_rn(h);
          } else {
            const double theta = (0.5 * h) * __drcp_rn(apq);
            t = __drcp_rn(fabs(theta) + __dsqrt_rn(__fma_rn(theta, theta, 1.0)));
            if (theta < 0.0) t = -t;
          }
          c = rsqrt(__fma_rn(t, t, 1.0));
          sn = t * c;
        }
        w.c[lane] = c;
        w.s[lane] = sn;
        w.t[lane] = t;
      }
      __syncwarp();
      double out[2];
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        const int e = lane + 32 * h2;
        if (e >= 36) break;
        const int i = e / 6, j = e % 6;
        const int ii = w.part[r][i], jj = w.part[r][j];
        const int si = w.slot[r][i], sj = w.slot[r][j];
        const bool ip = i < ii, jp = j < jj;
        double o;
        if (si == sj) {  // same 2x2 block
          if (i != j) {
            o = 0.0;
          } else {
            const int p = ip ? i : ii, q = ip ? ii : i;
            const double apq = w.a[6 * p + q];
            o = ip ? w.a[7 * p] - w.t[si] * apq : w.a[7 * q] + w.t[si] * apq;
          }
        } else {
          // col p' = c col p - s col q, col q' = s col p + c col q; rows alike
          const double cj = w.c[sj], sj2 = w.s[sj], ci = w.c[si], si2 = w.s[si];
          const double xi = w.a[6 * i + j], yi = w.a[6 * i + jj];
          const double xii = w.a[6 * ii + j], yii = w.a[6 * ii + jj];
          const double bi = jp ? cj * xi - sj2 * yi : sj2 * yi + cj * xi;
          const double bii = jp ? cj * xii - sj2 * yii : sj2 * yii + cj * xii;
          o = ip ? ci * bi - si2 * bii : si2 * bii + ci * bi;
        }
        out[h2] = o;
      }
      __syncwarp();
      w.a[lane] = out[0];
      if (lane < 4) w.a[lane + 32] = out[1];
      __syncwarp();
    }
    if (lane == 0) w.sweeps = sweep + 1;
    if (!w.rotated) break;
    __syncwarp();
  }
  // ascending, stable
  double d[6];
  int order[6];
  for (int i = 0; i < 6; ++i) {
    d[i] = w.a[7 * i];
    order[i] = i;
  }
  for (int i = 1; i < 6; ++i) {
    const int k = order[i];
    int j = i - 1;
    while (j >= 0 && d[order[j]] > d[k]) {
      order[j + 1] = order[j];
      --j;
    }
    order[j + 1] = k;
  }
  for (int i = 0; i < 6; ++i) ev[i] = d[order[i]];
  __syncwarp();
}

// ldlt_solve6_tr (trg_math.cuh: LDLT with diagonal pivoting -- first largest
// |a_ii| -- the shim's Eigen::LDLT), the two triangular solves and tr(A^-1)
// = sum_k (1/d_k) sum_{i<=k} (L^-1)_ki^2, on ONE thread with everything in
// registers: the row/column exchanges are compare-selects over the static
// candidates, so no shared-memory round trip sits on the dependency chain
// (the warp-parallel shared-memory version it replaces spent ~14 us per EM
// iteration on its ~100 serialised steps).
__device__ __forceinline__ void ldlt_solve6_tr_reg(const double* A, const double* b, double x[6],
                                                   double* trace_inv, double* min_pivot) {
  double a[6][6], l[6][6], d[6];
  int perm[6];
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    perm[i] = i;
#pragma unroll
    for (int j = 0; j < 6; ++j) {
      a[i][j] = A[i * 6 + j];
      l[i][j] = i == j ? 1.0 : 0.0;
    }
  }
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    int p = k;
    double best = fabs(a[k][k]);
#pragma unroll
    for (int i = k + 1; i < 6; ++i) {
      const double v = fabs(a[i][i]);
      if (v > best) {
        best = v;
        p = i;
      }
    }
    // exchange rows / columns k <-> p of a, rows k <-> p of L's first k columns
#pragma unroll
    for (int i = k + 1; i < 6; ++i) {
      const bool sw = p == i;
#pragma unroll
      for (int j = 0; j < 6; ++j) {
        const double t = a[k][j];
        a[k][j] = sw ? a[i][j] : t;
        a[i][j] = sw ? t : a[i][j];
      }
#pragma unroll
      for (int j = 0; j < 6; ++j) {
        const double t = a[j][k];
        a[j][k] = sw ? a[j][i] : t;
        a[j][i] = sw ? t : a[j][i];
      }
#pragma unroll
      for (int j = 0; j < k; ++j) {
        const double t = l[k][j];
        l[k][j] = sw ? l[i][j] : t;
        l[i][j] = sw ? t : l[i][j];
      }
      const int tp = perm[k];
      perm[k] = sw ? perm[i] : tp;
      perm[i] = sw ? tp : perm[i];
    }
    const double dk = a[k][k];
    d[k] = dk;
#pragma unroll
    for (int i = k + 1; i < 6; ++i) l[i][k] = (dk != 0.0) ? a[i][k] / dk : 0.0;
#pragma unroll
    for (int i = k + 1; i < 6; ++i)
#pragma unroll
      for (int j = k + 1; j < 6; ++j) a[i][j] = a[i][j] - l[i][k] * dk * l[j][k];
  }
  // the triangular solves (permuted right-hand side)
  double y[6], z[6];
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    double v = b[0];
#pragma unroll
    for (int q = 1; q < 6; ++q) v = perm[i] == q ? b[q] : v;
    y[i] = v;
  }
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    double s2 = y[i];
#pragma unroll
    for (int j = 0; j < i; ++j) s2 -= l[i][j] * y[j];
    y[i] = s2;
  }
#pragma unroll
  for (int i = 0; i < 6; ++i) y[i] = (d[i] != 0.0) ? y[i] / d[i] : 0.0;
#pragma unroll
  for (int i = 5; i >= 0; --i) {
    double s2 = y[i];
#pragma unroll
    for (int j = i + 1; j < 6; ++j) s2 -= l[j][i] * z[j];
    z[i] = s2;
  }
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    double v = z[0];
#pragma unroll
    for (int q = 1; q < 6; ++q) v = perm[q] == i ? z[q] : v;
    x[i] = v;
  }
  // tr(A^{-1}) = sum_k (1/d_k) sum_{i <= k} M_ki^2 with M = L^{-1}, in k order
  double m[6][6];
#pragma unroll
  for (int j = 0; j < 6; ++j) {
#pragma unroll
    for (int i = 0; i < 6; ++i) m[i][j] = (i == j) ? 1.0 : 0.0;
#pragma unroll
    for (int i = j + 1; i < 6; ++i) {
      double s2 = 0.0;
#pragma unroll
      for (int k = j; k < i; ++k) s2 -= l[i][k] * m[k][j];
      m[i][j] = s2;
    }
  }
  double tr = 0.0, mind = d[0];
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    double sk = 0.0;
#pragma unroll
    for (int i = 0; i <= k; ++i) sk += m[k][i] * m[k][i];
    mind = d[k] < mind ? d[k] : mind;
    tr += (d[k] > 0.0) ? sk / d[k] : INFINITY;
  }
  *trace_inv = tr;
  *min_pivot = mind;
}

// solve_mstep (mstep.cpp:76-98) from the reduced normal equations, by one
// warp: LDLT + tr(A^-1) on lane 0 (the condition bracket tr(A) tr(A^-1)),
// the warp-parallel 6x6 Jacobi only when the bracket straddles 1e12, then
// the exp map.  Result in *o (valid after the call on all lanes).
static __device__ void warp_solve_normal_eq(const double* v, int nvp, SolveOut* o, Eig6Smem& w,
                                            Timeline* tl = nullptr, bool exact_cond = true) {
  const int lane = threadIdx.x & 31;
  if (nvp < 3) {
    if (lane == 0) {
      o->nvp = nvp;
      o->degenerate = 1;
      o->cond = INFINITY;
    }
    __syncwarp();
    return;
  }
  __shared__ double ata_s[36];
  __shared__ int s_need_eig;
  for (int e = lane; e < 36; e += 32) {
    const int i = e / 6, j = e % 6;
    const int a = i < j ? i : j, b = i < j ? j : i;
    ata_s[e] = v[a * 6 - a * (a - 1) / 2 + (b - a)];
  }
  __syncwarp();
  double x[6], trinv = 0.0, mind = 0.0;
  if (tl && lane == 0) tl_mark_any(tl, 7004);
  if (lane == 0) ldlt_solve6_tr_reg(ata_s, v + 21, x, &trinv, &mind);
  if (tl && lane == 0) tl_mark_any(tl, 7005);
  if (lane == 0) {
    o->nvp = nvp;
    o->degenerate = 0;
    o->eig_sweeps = 0;
    double ata[6][6];
    for (int i = 0; i < 6; ++i)
      for (int j = 0; j < 6; ++j) ata[i][j] = ata_s[i * 6 + j];
    for (int i = 0; i < 3; ++i) {
      o->omega[i] = x[i];
      o->trans[i] = x[3 + i];
      o->dt[i] = x[3 + i];
    }
    double tra = ata[0][0];
    for (int i = 1; i < 6; ++i) tra += ata[i][i];
    const double hi = tra * trinv;  // >= cond, <= 36 cond
    int need = 1;
    if (!exact_cond) {
      if (!(mind > 0.0)) {  // not positive definite: lambda_min <= 0, cond = inf
        o->cond = INFINITY;
        o->degenerate = 1;
        need = 0;
      } else if (hi < 1e12) {  // cond <= hi < 1e12
        o->cond = hi;            // upper bound (the EM loop only needs the test)
        need = 0;
      } else if (hi / 36.0 >= 1e12) {
        o->cond = hi / 36.0;
        o->degenerate = 1;
        need = 0;
      }
    }
    s_need_eig = need;
  }
  __syncwarp();
  if (s_need_eig) {
    double ev[6];
    if (tl && lane == 0) tl_mark_any(tl, 7001);
    warp_eig6(ata_s, ev, w);
    if (tl && lane == 0) tl_mark_any(tl, 7002);
    if (lane == 0) {
      o->eig_sweeps = w.sweeps;
      const double lmin = ev[0], lmax = ev[5];
      const double cond = lmin > 0.0 ? lmax / lmin : INFINITY;
      o->cond = cond;
      if (!(cond < 1e12)) o->degenerate = 1;
    }
  }
  if (lane == 0 && !o->degenerate) small_angle_rotation(o->omega, o->dR);
  if (tl && lane == 0) tl_mark_any(tl, 7003);
  __syncwarp();
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
  __shared__ Eig6Smem e6;
  __shared__ double vsh[kNormalEq];
  __shared__ int nvp_sh;
  if (threadIdx.x == 0) {
    so.crit_before = a.crit;
    for (int k = 0; k < kNormalEq; ++k) vsh[k] = a.v[k];
    nvp_sh = a.nvp;
  }
  __syncthreads();
  if (threadIdx.x < 32) warp_solve_normal_eq(vsh, nvp_sh, &so, e6);
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
