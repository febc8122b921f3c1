// Registration EM resident on the GPU (registration.cpp:47-82, 140-209):
// one persistent cooperative kernel runs every iteration -- E-step
// (K7 descent + deterministic per-CTA reduction), node combine + virtual
// point rows, single-block 6-DoF solve (K8), T <- delta o T, convergence and
// degenerate-streak control -- with grid barriers between phases, so the
// host never sees an iteration boundary.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <cstdio>
#include <memory>
#include <string>
#include <vector>

#include "trg_dense.cuh"
#include "trg_roles.cuh"

namespace trg {

struct EmState {
  double Rt[12];        // running transform (R row-major, t)
  double trans_limit;   // translation_tol * diag
  int done, converged, iterations, fails;
};

struct EmParams {
  AssocParams a;
  double* moments;  // [J][4] (dense path)
  double* cta_acc;  // [G][kNormalEq + 2] (dense path)
  long long* acc;   // tree path: [2][12][acc_stride] exact planar accumulators (trg_fx.cuh)
  unsigned* sync;   // [16]: grid barrier, flag, arrivals (zeroed per launch)
  unsigned* smtab;  // [G] SM id per CTA (roles)
  unsigned* bar;
  EmState* st;
  double* crit_before;
  double* crit_after;
  unsigned long long* evals;
  int max_iters;
  double rot_tol;
  uint32_t epoch0;
  Timeline* tl;
  // Point-sharded mode: seg = it >= 0 finishes iteration it-1
  // from the all-reduced moments in xmom ([J][4] + evals, outliers) and runs
  // the E-step of iteration it up to the local per-node combine, then exits.
  int seg;
  double* xmom;
  double n_total;  // total source points over all shards (mass floor)
  double* psum;    // dense (flat mixture) E-step: per-point score sums
  // Queued behind an asynchronous build (register_clouds): the tree's size
  // comes from the build's published meta (nothing to do unless meta->ok).
  const TreeMeta* meta;
  // FP32 fast path (trg_reg_config.fast_scoring): the tree as FNode records,
  // converted by the launch's own CTAs before its first grid barrier
  FNode* fnodes;
  int fast;
};

constexpr int kAccStride = kNormalEq + 2;

// Per-node (m0, m1) of iteration `it`: the exchanged doubles (sharded) or
// the iteration's exact accumulators.
__device__ __forceinline__ void em_node_moments(const EmParams& p, bool sharded, const long long* acc,
                                                const FxScale* sc, int j, double m[4]) {
  if (sharded) {
#pragma unroll
    for (int k = 0; k < 4; ++k) m[k] = ldcg(p.xmom + (size_t)j * 4 + k);
  } else {
    fx_row<4>(acc, p.a.acc_stride, j, sc, m);
  }
}

// One EM iteration (tree model) = E-step: every CTA's warps descend their
// fixed 32-point windows and add each window's runs to the iteration's exact
// per-node accumulators | ONE grid barrier | EVERY CTA reads all J nodes'
// moments, forms the virtual-point rows (27-term normal equations) in the
// same thread mapping, reduces them in a fixed order and solves (identical
// bits everywhere), so T <- delta o T and the stop decision need no second
// barrier.  The accumulators rotate over three buffers: iteration it writes
// acc[it % 3], and after its barrier every CTA zeroes its slice of
// acc[(it + 2) % 3] (last read before that barrier, next written after the
// following one).
// DENSE: the flat-mixture variant (registration.cpp:191-202): the E-step is
// responsibilities_dense over the J components (per-component rows + a
// per-node combine on ceil(J/8) CTAs, then a second barrier).
template <bool DENSE>
__global__ void __launch_bounds__(kAssocBlock, 2) k_register(EmParams p) {
  __shared__ SolveSmem ss;
  __shared__ Eig6Smem e6;
  __shared__ SolveOut so;
  __shared__ double rt[12];
  __shared__ double red[kAccStride];
  __shared__ FxScale sc[3], sc_prev[3];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ int s_done, s_fails, s_conv, s_iters;
  const int G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  constexpr int WPB = kAssocBlock / 32;
  int J = p.a.n_nodes, root_count = p.a.root_count, n_snodes = p.a.n_snodes;
  if (p.meta) {
    if (!__ldcg(&p.meta->ok)) return;  // the build failed or overflowed: the host retries / reports
    J = __ldcg(&p.meta->J);
    root_count = __ldcg(&p.meta->root_count);
    n_snodes = min(__ldcg(&p.meta->n_upper), kStageNodes);
  }
  const int P2 = min(G, (J + WPB - 1) / WPB);  // DENSE: producer CTAs of the per-node rows
  const bool sharded = p.seg >= 0;
  const double n_total = sharded ? p.n_total : (double)p.a.n;
  const size_t accJ = p.a.acc_stride * 4 * 3;  // limbs per accumulator buffer
  if (tid < 12) rt[tid] = ldcg(&p.st->Rt[tid]);
  if (tid == 0) {
    s_done = sharded ? *(volatile int*)&p.st->done : 0;
    s_fails = sharded ? *(volatile int*)&p.st->fails : 0;
    s_conv = sharded ? *(volatile int*)&p.st->converged : 0;
    s_iters = sharded ? *(volatile int*)&p.st->iterations : 0;
    mbar_init(&mbar, 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (s_done) return;
  const double trans_limit = ldcg(&p.st->trans_limit);
  // the model is fixed during the EM: stage its upper levels once (bulk copy)
  extern __shared__ __align__(128) unsigned char k_reg_stage[];
  DNode* reg_stage = reinterpret_cast<DNode*>(k_reg_stage);
  unsigned mphase = 0;
  if (!DENSE) stage_nodes_bulk(reg_stage, p.a.nodes, n_snodes, &mbar, mphase);
  // criterion after the update of iteration k (trace only), CTA 0.  Single
  // GPU (defer): CTA 0 takes no E-step windows and computes it for iteration
  // it-1 while the other CTAs run iteration it's E-step (the moments of it-1
  // and its solve are still in place then), so the trace leaves the
  // iteration's critical path; the last iteration's is computed after the loop.
  const bool defer = !sharded && !DENSE && G > 1;
  auto crit_trace = [&](int k, const FxScale* s) {
    unsigned long long* counters = p.a.counters + 2 * (k & 1);
    double c = 0.0;
    if (!so.degenerate) {
      double dRt[12];
      for (int i = 0; i < 9; ++i) dRt[i] = so.dR[i];
      for (int i = 0; i < 3; ++i) dRt[9 + i] = so.dt[i];
      const long long* acc = p.acc + (size_t)(k % 3) * accJ;
      for (int j = tid; j < J; j += blockDim.x) {
        double m[4];
        if (DENSE) {
          for (int q = 0; q < 4; ++q) m[q] = ldcg(p.moments + (size_t)j * 4 + q);
        } else {
          em_node_moments(p, sharded, acc, s, j, m);
        }
        c += crit_term(p.a.nodes + j, m[0], m[1], m[2], m[3], n_total, dRt);
      }
    }
    c = block_sum(c, ss);
    if (tid == 0) {
      p.evals[k] = sharded ? (unsigned long long)ldcg(p.xmom + (size_t)J * 4)
                           : atomicExch(&counters[1], 0ull);
      p.crit_before[k] = so.crit_before;
      p.crit_after[k] = so.degenerate ? so.crit_before : c;
    }
  };
  for (int it = 0; it < p.max_iters; ++it) {
    const bool run_e = !sharded || p.seg == it;      // E-step of iteration it
    const bool run_m = !sharded || p.seg == it + 1;  // solve of iteration it
    if (!run_e && !run_m) continue;
    AssocParams a = p.a;
    a.n_nodes = J;
    a.root_count = root_count;
    a.n_snodes = n_snodes;
    a.epoch = p.epoch0 + (uint32_t)it;
    a.snodes = reg_stage;
    a.acc = p.acc + (size_t)(it % 3) * accJ;
    // per-iteration counters alternate between two slots: CTA 0 reads and
    // clears slot it&1 while faster CTAs may already count iteration it+1's
    // evaluations (slot (it+1)&1); nobody reaches it+2 before that
    a.counters = p.a.counters + 2 * (it & 1);
    if (tid < 3) sc_prev[tid] = sc[tid];
    __syncthreads();
    if (tid == 0) assoc_scales(p.a.pmax, rt, sc);
    __syncthreads();
    if (run_e) {
      // ---- E-step
      tl_mark(p.tl, 2000 + it * 10);
      if constexpr (DENSE) {
        DenseParams d{};
        d.pts = a.pts;
        d.n = a.n;
        d.comps = a.nodes;
        d.J = J;
        d.outlier_floor = a.outlier_floor;
        d.psum = p.psum;
        d.partials = a.partials;
        d.stamps = a.stamps;
        d.epoch = a.epoch;
        d.counters = a.counters;
        d.status = a.status;
        dense_pass1(d, rt, G, cta);
        grid_sync(p.bar, G);
        dense_pass2<4>(d, rt, G, cta);
      } else if (defer && cta == 0) {
        if (it > 0) crit_trace(it - 1, sc_prev);
      } else {
        const int ctas = defer ? G - 1 : G, c = defer ? cta - 1 : cta;
        assoc_fx_pass<4>(a, rt, sc, ctas * WPB, warp * ctas + c);
      }
      grid_sync(p.bar, G);
      tl_mark(p.tl, 2000 + it * 10 + 1);
      if (sharded) {
        // this shard's per-node moments + counters, for the all-reduce
        // (the accumulator rows are zeroed for the next segment)
        for (int j = cta * WPB + warp; j < J; j += G * WPB) {
          double m[4];
          if constexpr (DENSE) {
            combine_node<4>(a.partials, a.stamps, a.epoch, G, j, m);
          } else {
            fx_row<4>(a.acc, a.acc_stride, j, sc, m);
          }
          __syncwarp();
          if (!DENSE)
            if (lane < 12) a.acc[(size_t)lane * a.acc_stride + j] = 0;
          if (lane == 0)
#pragma unroll
            for (int k = 0; k < 4; ++k) p.xmom[(size_t)j * 4 + k] = m[k];
        }
        if (cta == 0 && tid == 0) {
          p.xmom[(size_t)J * 4] = (double)atomicExch(&a.counters[1], 0ull);
          p.xmom[(size_t)J * 4 + 1] = (double)atomicExch(&a.counters[0], 0ull);
        }
        return;
      }
    }
    // ---- normal equations of iteration it
    if constexpr (DENSE) {
      if (cta < P2) {
        SolveAcc acc;
        acc_zero(acc);
        for (int j = cta * WPB + warp; j < J; j += P2 * WPB) {
          double m[4];
          if (sharded) {
#pragma unroll
            for (int k = 0; k < 4; ++k) m[k] = ldcg(p.xmom + (size_t)j * 4 + k);
          } else {
            combine_node<4>(a.partials, a.stamps, a.epoch, G, j, m);
          }
          if (lane == 0) {
#pragma unroll
            for (int k = 0; k < 4; ++k) p.moments[(size_t)j * 4 + k] = m[k];
            vp_accumulate(a.nodes + j, m[0], m[1], m[2], m[3], n_total, acc, a.status);
          }
        }
        block_reduce_acc(acc, ss);
        if (tid == 0) {
          double* o = p.cta_acc + (size_t)cta * kAccStride;
#pragma unroll
          for (int k = 0; k < kNormalEq; ++k) o[k] = acc.v[k];
          o[kNormalEq] = acc.crit;
          o[kNormalEq + 1] = (double)acc.nvp;
        }
      }
      grid_sync(p.bar, G);
      tl_mark(p.tl, 2000 + it * 10 + 2);
      {
        const int v = tid >> 3, sub = tid & 7;
        double s = 0.0;
        if (v < kAccStride)
          for (int c = sub; c < P2; c += 8) s += ldcg(p.cta_acc + (size_t)c * kAccStride + v);
        s += __shfl_xor_sync(0xffffffffu, s, 1);
        s += __shfl_xor_sync(0xffffffffu, s, 2);
        s += __shfl_xor_sync(0xffffffffu, s, 4);
        if (v < kAccStride && sub == 0) red[v] = s;
      }
    } else {
      if (!sharded) {
        // zero this CTA's slice of the buffer iteration it+2 writes
        long long* z = p.acc + (size_t)((it + 2) % 3) * accJ;
        for (size_t q = (size_t)cta * blockDim.x + tid; q < accJ; q += (size_t)G * blockDim.x) z[q] = 0;
      }
      // every CTA: all nodes' rows, fixed thread mapping and reduction order
      SolveAcc acc;
      acc_zero(acc);
      for (int j = tid; j < J; j += blockDim.x) {
        double m[4];
        em_node_moments(p, sharded, a.acc, sc, j, m);
        vp_accumulate(a.nodes + j, m[0], m[1], m[2], m[3], n_total, acc, a.status);
      }
      block_reduce_acc(acc, ss);
      if (tid == 0) {
#pragma unroll
        for (int k = 0; k < kNormalEq; ++k) red[k] = acc.v[k];
        red[kNormalEq] = acc.crit;
        red[kNormalEq + 1] = (double)acc.nvp;
      }
    }
    __syncthreads();
    if (tid == 0) so.crit_before = red[kNormalEq];
    __syncthreads();
    if (tid < 32) warp_solve_normal_eq(red, (int)red[kNormalEq + 1], &so, e6, nullptr, false);
    __syncthreads();
    tl_mark(p.tl, 2000 + it * 10 + 3);
    if (cta == 0 && !defer) crit_trace(it, sc);
    if (tid == 0) {
      s_iters = it + 1;
      if (!so.degenerate) {
        // T = delta * T (geometry.hpp:42-47)
        double nR[9], nt[3];
        for (int i = 0; i < 3; ++i)
          for (int jj = 0; jj < 3; ++jj) {
            double q = so.dR[3 * i] * rt[jj];
            q += so.dR[3 * i + 1] * rt[3 + jj];
            q += so.dR[3 * i + 2] * rt[6 + jj];
            nR[3 * i + jj] = q;
          }
        for (int i = 0; i < 3; ++i) {
          double q = so.dR[3 * i] * rt[9];
          q += so.dR[3 * i + 1] * rt[10];
          q += so.dR[3 * i + 2] * rt[11];
          nt[i] = q + so.dt[i];
        }
        for (int k = 0; k < 9; ++k) rt[k] = nR[k];
        for (int k = 0; k < 3; ++k) rt[9 + k] = nt[k];
        s_fails = 0;
        // rotation_angle (geometry.cpp:17-20) and |t| (registration.cpp:68-69)
        double cth = ((so.dR[0] + so.dR[4]) + so.dR[8] - 1.0) * 0.5;
        cth = cth < -1.0 ? -1.0 : (cth > 1.0 ? 1.0 : cth);
        double tn = so.trans[0] * so.trans[0];
        tn += so.trans[1] * so.trans[1];
        tn += so.trans[2] * so.trans[2];
        if (acos(cth) < p.rot_tol && sqrt(tn) < trans_limit) {
          s_conv = 1;
          s_done = 1;
        }
      } else if (++s_fails >= 3) {
        s_done = 1;
      }
    }
    __syncthreads();
    if (sharded) {
      // the running state crosses the launch boundary through EmState
      if (cta == 0 && tid == 0) {
        EmState* st = p.st;
        for (int k = 0; k < 12; ++k) st->Rt[k] = rt[k];
        st->iterations = s_iters;
        st->converged = s_conv;
        st->fails = s_fails;
        st->done = s_done || it + 1 >= p.max_iters;
      }
      if (s_done) return;
      continue;  // on to the E-step of iteration it+1 (run_e of the next pass)
    }
    if (s_done) break;
  }
  if (defer && cta == 0) crit_trace(s_iters - 1, sc);
  if (!sharded && cta == 0 && tid == 0) {
    EmState* st = p.st;
    for (int k = 0; k < 12; ++k) st->Rt[k] = rt[k];
    st->iterations = s_iters;
    st->converged = s_conv;
    st->fails = s_fails;
    st->done = 1;
  }
}

// ---------------------------------------------------------------- tree EM
constexpr int kEmBlock = 320;  // 10 warps: 2 CTAs x 147 worker SMs >= 2,400 windows (C2)
// Registration EM with a tree model (registration.cpp:47-82) as ONE
// persistent launch with roles (trg_roles.cuh): WORKER CTAs run each
// iteration's E-step -- the descent of their fixed 32-point windows and the
// exact per-node deposits into acc[it % 2] -- and arrive on a counter; ONE
// SOLVER CTA (on an updater SM, its instruction cache holding the solver)
// waits for the arrivals, forms the virtual-point rows of all J nodes
// (make_virtual_points + the 27-term normal equations, mstep.cpp:8-75),
// solves (mstep.cpp:76-98), applies T <- delta o T and the stop tests
// (registration.cpp:66-78), zeroes acc[(it + 1) % 2], publishes the new
// state with a flag, and only then computes the criterion-after trace of
// the iteration (diagnostics, off the critical path).  No grid barrier per
// iteration.
// Sharded (p.seg >= 0): segment s finishes iteration s-1 from the
// all-reduced moments in xmom, publishes iteration s, waits for the local
// E-step and exports this shard's per-node moments for the all-reduce.
__device__ __forceinline__ void em_apply_update(const SolveOut& so, double* rt, const EmParams& p,
                                                double trans_limit, int& s_fails, int& s_conv,
                                                int& s_done) {
  if (!so.degenerate) {
    // T = delta * T (geometry.hpp:42-47)
    double nR[9], nt[3];
    for (int i = 0; i < 3; ++i)
      for (int jj = 0; jj < 3; ++jj) {
        double q = so.dR[3 * i] * rt[jj];
        q += so.dR[3 * i + 1] * rt[3 + jj];
        q += so.dR[3 * i + 2] * rt[6 + jj];
        nR[3 * i + jj] = q;
      }
    for (int i = 0; i < 3; ++i) {
      double q = so.dR[3 * i] * rt[9];
      q += so.dR[3 * i + 1] * rt[10];
      q += so.dR[3 * i + 2] * rt[11];
      nt[i] = q + so.dt[i];
    }
    for (int k = 0; k < 9; ++k) rt[k] = nR[k];
    for (int k = 0; k < 3; ++k) rt[9 + k] = nt[k];
    s_fails = 0;
    // rotation_angle (geometry.cpp:17-20) and |t| (registration.cpp:68-69)
    double cth = ((so.dR[0] + so.dR[4]) + so.dR[8] - 1.0) * 0.5;
    cth = cth < -1.0 ? -1.0 : (cth > 1.0 ? 1.0 : cth);
    double tn = so.trans[0] * so.trans[0];
    tn += so.trans[1] * so.trans[1];
    tn += so.trans[2] * so.trans[2];
    if (acos(cth) < p.rot_tol && sqrt(tn) < trans_limit) {
      s_conv = 1;
      s_done = 1;
    }
  } else if (++s_fails >= 3) {
    s_done = 1;
  }
}

#ifndef TRG_KEM_MINB
#define TRG_KEM_MINB 2
#endif
// The EM of one registration on a group of G CTAs (this CTA: `cta`).
// by_sm: the solver is the CTA on the group's lowest SM, whose other CTAs
// idle (a single registration on the whole grid: that SM keeps the serial
// code resident); otherwise the group's CTA 0 (batches).
__device__ __forceinline__ void em_tree_run(const EmParams& p, int G, int cta, bool by_sm) {
  __shared__ SolveSmem ss;
  __shared__ Eig6Smem e6;
  __shared__ SolveOut so;
  __shared__ double rt[12];
  __shared__ double red[kAccStride];
  __shared__ FxScale sc[3];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ int s_done, s_fails, s_conv, s_iters;
  extern __shared__ __align__(128) unsigned char k_em_stage[];
  const int tid = threadIdx.x, warp = tid >> 5;
  constexpr int WPB = kEmBlock / 32;
  int J = p.a.n_nodes, root_count = p.a.root_count, n_snodes = p.a.n_snodes;
  if (p.meta) {
    if (!__ldcg(&p.meta->ok)) return;  // the build failed or overflowed: the host retries / reports
    J = __ldcg(&p.meta->J);
    root_count = __ldcg(&p.meta->root_count);
    n_snodes = min(__ldcg(&p.meta->n_upper), kStageNodes);
  }
  const bool sharded = p.seg >= 0;
  const int it0 = sharded ? p.seg : 0;
  const double n_total = sharded ? p.n_total : (double)p.a.n;
  const size_t S = p.a.acc_stride;
  unsigned* flag = p.sync + 2;
  unsigned* arrived = p.sync + 3;
  if (p.fast)  // the FP32 records, ordered before use by assign_roles' grid barrier
    for (int j = cta * blockDim.x + tid; j < J; j += G * blockDim.x) {
      FNode f;
      fnode_from(p.a.nodes[j], f);
      p.fnodes[j] = f;
    }
  const Roles r = by_sm ? assign_roles(p.smtab, p.sync, G, 1) : roles_by_index(p.sync, G, cta);
  if (r.upd && r.idx != 0) return;  // the solver's SM stays free of E-step work
  EmState* st = p.st;
  if (!r.upd) {
    // ------------------------------------------------ workers: E-steps
    if (tid == 0) {
      mbar_init(&mbar, 1);
      mbar_fence_init();
    }
    __syncthreads();
    DNode* stage = reinterpret_cast<DNode*>(k_em_stage);
    FNode* fstage = reinterpret_cast<FNode*>(k_em_stage);
    unsigned mphase = 0;
    if (p.fast) {  // the model is fixed: its upper levels staged once
      if (n_snodes > 0) {
        if (tid == 0) {
          fence_proxy_async_global();
          bulk_g2s_issue(fstage, p.fnodes, (unsigned)(n_snodes * sizeof(FNode)), &mbar);
          mbar_wait(&mbar, mphase);
        }
        __syncthreads();
        mphase ^= 1u;
      }
    } else {
      stage_nodes_bulk(stage, p.a.nodes, n_snodes, &mbar, mphase);
    }
    AssocParams a = p.a;
    a.n_nodes = J;
    a.root_count = root_count;
    a.n_snodes = n_snodes;
    a.snodes = stage;
    for (int k = 0;; ++k) {
      const int it = it0 + k;
      wait_flag(flag, (unsigned)k + 1);
      if (tid == 0) s_done = __ldcg(&st->done);
      if (tid < 12) rt[tid] = __ldcg(&st->Rt[tid]);
      __syncthreads();
      if (s_done || it >= p.max_iters) return;
      if (tid == 0) assoc_scales(p.a.pmax, rt, sc);
      __syncthreads();
      a.acc = p.acc + (size_t)(it & 1) * S * 12;
      a.counters = p.a.counters + 2 * (it & 1);
      if (p.fast)
        assoc_fx_pass_f32<4>(a, p.fnodes, fstage, rt, sc, r.n_work * WPB, warp * r.n_work + r.idx);
      else
        // warp-major window order: every worker CTA gets windows, spread over
        // the SMs (CTA-major left the last CTAs idle when windows < warps)
        assoc_fx_pass<4>(a, rt, sc, r.n_work * WPB, warp * r.n_work + r.idx);
      arrive_count(arrived);
      if (sharded) return;  // one E-step per segment
    }
  }
  // -------------------------------------------------- the solver CTA
  if (tid == 0) {
    s_done = __ldcg(&st->done);
    s_fails = __ldcg(&st->fails);
    s_conv = __ldcg(&st->converged);
    s_iters = __ldcg(&st->iterations);
  }
  if (tid < 12) rt[tid] = __ldcg(&st->Rt[tid]);
  __syncthreads();
  const double trans_limit = __ldcg(&st->trans_limit);
  // moments of iteration `it` (exchanged doubles when sharded)
  auto node_m = [&](int it, int j, double m[4]) {
    if (sharded) {
#pragma unroll
      for (int q = 0; q < 4; ++q) m[q] = __ldcg(p.xmom + (size_t)j * 4 + q);
    } else {
      fx_row<4>(p.acc + (size_t)(it & 1) * S * 12, S, j, sc, m);
    }
  };
  // criterion after the update of iteration it (trace only)
  auto crit_trace = [&](int it) {
    double c = 0.0;
    if (!so.degenerate) {
      double dRt[12];
      for (int i = 0; i < 9; ++i) dRt[i] = so.dR[i];
      for (int i = 0; i < 3; ++i) dRt[9 + i] = so.dt[i];
      for (int j = tid; j < J; j += blockDim.x) {
        double m[4];
        node_m(it, j, m);
        c += crit_term(p.a.nodes + j, m[0], m[1], m[2], m[3], n_total, dRt);
      }
    }
    c = block_sum(c, ss);
    if (tid == 0) {
      p.evals[it] = sharded ? (unsigned long long)__ldcg(p.xmom + (size_t)J * 4)
                            : atomicExch(&p.a.counters[2 * (it & 1) + 1], 0ull);
      p.crit_before[it] = so.crit_before;
      p.crit_after[it] = so.degenerate ? so.crit_before : c;
    }
  };
  // solve of iteration it from its moments; state update
  auto solve = [&](int it) {
    SolveAcc acc;
    acc_zero(acc);
    for (int j = tid; j < J; j += blockDim.x) {
      double m[4];
      node_m(it, j, m);
      vp_accumulate(p.a.nodes + j, m[0], m[1], m[2], m[3], n_total, acc, p.a.status);
    }
#ifdef TRG_EM_PROBE
    if (tid == 0) tl_mark_any(p.tl, 7100);
#endif
    block_reduce_acc(acc, ss);
    if (tid == 0) {
#pragma unroll
      for (int k = 0; k < kNormalEq; ++k) red[k] = acc.v[k];
      red[kNormalEq] = acc.crit;
      red[kNormalEq + 1] = (double)acc.nvp;
      so.crit_before = acc.crit;
    }
    __syncthreads();
#ifdef TRG_EM_PROBE
    if (tid == 0) tl_mark_any(p.tl, 7101);
#endif
#ifdef TRG_EM_PROBE
    if (tid < 32) warp_solve_normal_eq(red, (int)red[kNormalEq + 1], &so, e6, p.tl, false);
#else
    if (tid < 32) warp_solve_normal_eq(red, (int)red[kNormalEq + 1], &so, e6, nullptr, false);
#endif
    __syncthreads();
#ifdef TRG_EM_PROBE
    if (tid == 0) tl_mark_any(p.tl, 7102);
#endif
    if (tid == 0) {
      s_iters = it + 1;
      em_apply_update(so, rt, p, trans_limit, s_fails, s_conv, s_done);
      if (it + 1 >= p.max_iters) s_done = 1;
    }
    __syncthreads();
  };
  auto publish_state = [&](unsigned f) {
    if (tid == 0) {
      for (int k = 0; k < 12; ++k) st->Rt[k] = rt[k];
      st->iterations = s_iters;
      st->converged = s_conv;
      st->fails = s_fails;
      st->done = s_done;
      publish_flag(flag, f);
    }
  };
  if (sharded && it0 > 0 && !s_done) {
    // finish iteration it0-1 from the all-reduced moments
    solve(it0 - 1);
    publish_state(1u);
    crit_trace(it0 - 1);
  } else {
    if (tid == 0 && it0 >= p.max_iters) s_done = 1;
    __syncthreads();
    publish_state(1u);
  }
  if (s_done) return;
  for (int k = 0;; ++k) {
    const int it = it0 + k;
    if (tid == 0) assoc_scales(p.a.pmax, rt, sc);  // the scales the workers used
    wait_count(arrived, (unsigned)r.n_work * (unsigned)(k + 1));
    if (tid == 0) tl_mark_any(p.tl, 2000 + it * 10 + 1);
    if (sharded) {
      // this shard's per-node moments + counters, for the all-reduce (the
      // accumulator rows are zeroed for the next segment)
      long long* acc = p.acc + (size_t)(it & 1) * S * 12;
      for (int j = tid; j < J; j += blockDim.x) {
        double m[4];
        fx_row<4>(acc, S, j, sc, m);
        for (int q = 0; q < 12; ++q) acc[(size_t)q * S + j] = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) p.xmom[(size_t)j * 4 + q] = m[q];
      }
      if (tid == 0) {
        p.xmom[(size_t)J * 4] = (double)atomicExch(&p.a.counters[2 * (it & 1) + 1], 0ull);
        p.xmom[(size_t)J * 4 + 1] = (double)atomicExch(&p.a.counters[2 * (it & 1)], 0ull);
      }
      return;
    }
    solve(it);
    {  // the buffer iteration it+1 writes (last read by iteration it-1)
      long long* z = p.acc + (size_t)((it + 1) & 1) * S * 12;
      for (size_t q = tid; q < S * 12; q += blockDim.x) z[q] = 0;
    }
    __syncthreads();
    publish_state((unsigned)k + 2);
    if (tid == 0) tl_mark_any(p.tl, 2000 + it * 10 + 3);
    crit_trace(it);
    if (s_done) break;
  }
}

// Registrations per launch: k_em_tree takes a batch of independent EM runs,
// run i on CTAs [i * group, (i + 1) * group) (trg_register_batch); a single
// registration is a batch of one on the whole grid with SM-placed roles.
// One kernel for both (see k_build: per-kernel FP64 contraction).
constexpr int kMaxEmBatch = kBatchInflightMax;
struct EmBatch {
  int group, n, by_sm;
  EmParams p[kMaxEmBatch];
};
static_assert(sizeof(EmBatch) <= 32000, "kernel parameter space");

__global__ void __launch_bounds__(kEmBlock, TRG_KEM_MINB) k_em_tree(const __grid_constant__ EmBatch b) {
  const int i = blockIdx.x / b.group;
  if (i < b.n) em_tree_run(b.p[i], b.group, blockIdx.x - i * b.group, b.by_sm != 0);
}

// registration.cpp:140-151 tree_extent_estimate (single block; min/max are
// exact, so the result is bit-identical to the reference).
__global__ void k_extent(const DNode* __restrict__ nodes, int J, EmState* st, double diag,
                         double tol, const TreeMeta* meta, const double* diag_dev) {
  __shared__ double lo[3][256], hi[3][256];
  if (meta) {
    if (!__ldcg(&meta->ok)) return;
    J = __ldcg(&meta->J);
  }
  if (diag_dev) diag = __ldcg(diag_dev);
  double l[3] = {INFINITY, INFINITY, INFINITY}, h[3] = {-INFINITY, -INFINITY, -INFINITY};
  if (!(diag > 0.0)) {
    for (int j = threadIdx.x; j < J; j += blockDim.x) {
      const DNode& g = nodes[j];
      if (g.child_count != 0) continue;
      const double r = 3.0 * sqrt(smax(g.lam[0], 0.0));
      for (int k = 0; k < 3; ++k) {
        l[k] = smin(l[k], g.mean[k] - r);
        h[k] = smax(h[k], g.mean[k] + r);
      }
    }
  }
  for (int k = 0; k < 3; ++k) {
    lo[k][threadIdx.x] = l[k];
    hi[k][threadIdx.x] = h[k];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double d = diag;
    if (!(diag > 0.0)) {
      for (int t = 1; t < blockDim.x; ++t)
        for (int k = 0; k < 3; ++k) {
          l[k] = smin(l[k], lo[k][t]);
          h[k] = smax(h[k], hi[k][t]);
        }
      double s = (h[0] - l[0]) * (h[0] - l[0]);
      s += (h[1] - l[1]) * (h[1] - l[1]);
      s += (h[2] - l[2]) * (h[2] - l[2]);
      d = sqrt(s);
    }
    st->trans_limit = tol * d;
  }
}

__global__ void k_check_finite(const double* __restrict__ p, size_t n3, int* status) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n3;
       i += (size_t)gridDim.x * blockDim.x)
    if (!isfinite(p[i])) atomicCAS(status, 0, kEInval);
}

__global__ void k_solve(const DNode* __restrict__ nodes, int J, const double* __restrict__ mom,
                        double n_total, SolveOut* out, int* status) {
  __shared__ SolveSmem ss;
  block_solve(nodes, J, mom, 4, n_total, out, ss, status);
}

// solve_mstep on explicit virtual points (mstep.hpp:21-32): n VPs with their
// components' (mean, lambdas, axes) as packed DNodes.
__global__ void k_solve_vps(const DNode* __restrict__ comps, const double* __restrict__ pimu,
                            int n, SolveOut* out, int* status) {
  __shared__ SolveSmem ss;
  __shared__ SolveOut so;
  __shared__ Eig6Smem e6;
  __shared__ double vsh[kNormalEq];
  __shared__ int nvp_sh;
  SolveAcc a;
  acc_zero(a);
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const double mu[3] = {pimu[4 * j + 1], pimu[4 * j + 2], pimu[4 * j + 3]};
    vp_rows(comps + j, pimu[4 * j], mu, a, status);
  }
  block_reduce_acc(a, ss);
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
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      // criterion term with pi, mu given: reuse crit_term via m0 = pi, N = 1
      const double pi = pimu[4 * j];
      c += crit_term(comps + j, pi, pi * pimu[4 * j + 1], pi * pimu[4 * j + 2],
                     pi * pimu[4 * j + 3], 1.0, dRt);
    }
  }
  c = block_sum(c, ss);
  if (threadIdx.x == 0) {
    so.crit_after = so.degenerate ? so.crit_before : c;
    *out = so;
  }
}

// make_virtual_points (mstep.cpp:8-30): order-preserving filter m0 > 1e-8 N.
__global__ void k_make_vps(const double* __restrict__ mom, int J, double n_total, int* idx,
                           double* pimu, int* count) {
  __shared__ int wsum[33];
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int per = (J + nt - 1) / nt;
  const int b = min(J, tid * per), e = min(J, b + per);
  const double floor_mass = 1e-8 * n_total;
  int my = 0;
  for (int j = b; j < e; ++j) my += (mom[4 * j] <= floor_mass) ? 0 : 1;
  int x = my;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  if (tid == 0) {
    int run = 0;
    for (int w = 0; w < nt / 32; ++w) {
      const int v = wsum[w];
      wsum[w] = run;
      run += v;
    }
    *count = run;
  }
  __syncthreads();
  int pos = wsum[warp] + x - my;
  for (int j = b; j < e; ++j) {
    const double m0 = mom[4 * j];
    if (m0 <= floor_mass) continue;
    idx[pos] = j;
    pimu[4 * pos] = m0 / n_total;
    pimu[4 * pos + 1] = mom[4 * j + 1] / m0;
    pimu[4 * pos + 2] = mom[4 * j + 2] / m0;
    pimu[4 * pos + 3] = mom[4 * j + 3] / m0;
    ++pos;
  }
}

}  // namespace trg

using namespace trg;

namespace trg {
int stage_points_public(trg_ctx* ctx, const double* xyz, size_t n, int on_device, int slot,
                        const double** dev);
}

namespace {

struct EmJob {
  const void* kernel = nullptr;
  int block = 0;
  size_t smem = 0;
  EmParams p;
  int G = 0, J = 0, K = 0;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  int* status = nullptr;  // the status word this run reports through
};

// Parameters, workspace and initial state of one EM run (sharded: seg mode
// with the exchange buffer xmom and the global point count).
// meta / diag_dev (asynchronous register_clouds): the tree is still being
// built; its size and the target diagonal are read on the device, workspace
// is sized for the tree's capacity, and errors go to ctx->status2 so the
// build's collect does not see them.  Nothing here synchronises the stream.
int em_prepare(trg_ctx* ctx, const trg_tree_dev* tree, const double* src_dev, size_t n,
               const trg_reg_config* cfg, double target_diag, bool sharded, double n_total,
               EmJob* job, bool dense = false, const TreeMeta* meta = nullptr,
               const double* diag_dev = nullptr) {
  const int J = meta ? tree->capacity : tree->n_nodes;
  int* status = meta ? ctx->status2 : ctx->status;
  job->status = status;
  job->kernel = dense ? (const void*)k_register<true> : (const void*)k_em_tree;
  job->block = dense ? kAssocBlock : kEmBlock;
  job->smem = dense ? 0 : sizeof(DNode) * kStageNodes;
  TRG_CU(set_dynamic_smem(job->kernel, std::max<size_t>(job->smem, 1)));
  // dense: 2 CTAs per SM (of the 3 that fit).  tree: enough worker warps
  // for one 32-point window each (a second window per warp doubles the
  // E-step's latency), at most 2 CTAs per SM, plus the solver's SM
  int per_sm = n >= 40000 ? 2 : 1;
  if (!dense) {
    const size_t windows = (n + 31) / 32;
    const size_t wpc = kEmBlock / 32;
    per_sm = (int)std::min<size_t>(2, std::max<size_t>(1, (windows + wpc * (ctx->sms - 1) - 1) /
                                                              (wpc * std::max(1, ctx->sms - 1))));
  }
  const int G = std::min(persistent_grid(ctx, job->kernel, job->block, job->smem),
                         ctx->sms * std::max(1, per_sm));
  EmParams p{};
  p.a.nodes = tree->nodes;
  p.a.n_nodes = J;
  p.a.root_count = tree->root_count;
  p.a.n_snodes = dense ? 0 : std::min(tree->n_upper, kStageNodes);
  p.a.depth = tree->max_level;
  p.a.lambda_c = cfg->variant_kind == TRG_VARIANT_TREE ? 0.0 : cfg->lambda_c;
  p.a.outlier_floor = 1e-300;
  p.a.pts = src_dev;
  p.a.n = n;
  p.a.status = status;
  p.meta = meta;
  void *part = nullptr, *stamps = nullptr, *mom, *cnt, *em, *tr, *xm, *accv = nullptr;
  if (dense) {
    TRG_TRY(ws_get(ctx, kSlotPartials, sizeof(double) * 4 * (size_t)J * G, &part));
    TRG_TRY(ws_get(ctx, kSlotStamps, sizeof(uint32_t) * (size_t)J * G, &stamps));
  } else {
    TRG_TRY(ws_get(ctx, kSlotPartials, sizeof(long long) * 2 * 12 * (size_t)J, &accv));
  }
  TRG_TRY(ws_get(ctx, kSlotMoments, sizeof(double) * 4 * (size_t)J, &mom));
  TRG_TRY(ws_get(ctx, kSlotCounters, 64 + 8, &cnt));
  const size_t em_bytes = 256 + sizeof(EmState) + sizeof(double) * kAccStride * G + 4 * (size_t)G + 64;
  TRG_TRY(ws_get(ctx, kSlotEm, em_bytes, &em));
  const int K = cfg->max_em_iterations;
  TRG_TRY(ws_get(ctx, kSlotEmTrace, (sizeof(double) * 2 + 8) * (size_t)K, &tr));
  TRG_TRY(ws_get(ctx, kSlotBuild10, sizeof(double) * (4 * (size_t)J + 2), &xm));
  p.a.partials = static_cast<double*>(part);
  p.a.stamps = static_cast<uint32_t*>(stamps);
  p.a.counters = static_cast<unsigned long long*>(cnt);
  p.a.pmax = reinterpret_cast<const double*>(static_cast<char*>(cnt) + 64);
  p.acc = static_cast<long long*>(accv);
  p.a.acc_stride = (size_t)J;
  p.moments = static_cast<double*>(mom);
  p.bar = static_cast<unsigned*>(em);
  p.st = reinterpret_cast<EmState*>(static_cast<char*>(em) + 64);
  p.cta_acc = reinterpret_cast<double*>(static_cast<char*>(em) + 256);
  p.sync = p.bar;  // [0..1] grid barrier, [2] flag, [3] arrivals
  p.smtab = reinterpret_cast<unsigned*>(p.cta_acc + (size_t)kAccStride * G);
  p.crit_before = static_cast<double*>(tr);
  p.crit_after = p.crit_before + K;
  p.evals = reinterpret_cast<unsigned long long*>(p.crit_after + K);
  p.max_iters = K;
  p.rot_tol = cfg->rotation_tol;
  p.tl = ctx->dev_timeline;
  p.seg = sharded ? 0 : -1;
  p.xmom = static_cast<double*>(xm);
  if (dense) {
    void* ps = nullptr;
    TRG_TRY(ws_get(ctx, kSlotDense, sizeof(double) * std::max<size_t>(n, 1), &ps));
    p.psum = static_cast<double*>(ps);
  }
  p.n_total = sharded ? n_total : (double)n;
  p.fast = (!dense && cfg->fast_scoring) ? 1 : 0;
  if (p.fast) {
    void* fb = nullptr;
    TRG_TRY(ws_get(ctx, kSlotBuild9, sizeof(FNode) * (size_t)std::max(J, 1), &fb));
    p.fnodes = static_cast<FNode*>(fb);
  }
  TRG_TRY(timeline_reset(ctx));
  p.epoch0 = ctx->epoch + 1;
  ctx->epoch += (uint32_t)K + 1;
  // initial state through a dedicated pinned buffer: an asynchronous copy,
  // no staging sync (the previous run's copy completed at its collect)
  void* hst = nullptr;
  TRG_TRY(host_ws_get(ctx, kSlotHostEmInit, sizeof(EmState), &hst));
  EmState& st = *static_cast<EmState*>(hst);
  st = EmState{};
  for (int k = 0; k < 9; ++k) st.Rt[k] = cfg->initial_R[k];
  for (int k = 0; k < 3; ++k) st.Rt[9 + k] = cfg->initial_t[k];
  TRG_CU(cudaMemsetAsync(em, 0, 64, ctx->stream));
  TRG_CU(cudaMemsetAsync(cnt, 0, 64 + 8, ctx->stream));
  if (accv)
    TRG_CU(cudaMemsetAsync(accv, 0, sizeof(long long) * 2 * 12 * (size_t)J, ctx->stream));
  TRG_CU(trg_memcpy(ctx, p.st, &st, sizeof st, cudaMemcpyHostToDevice));
  // non-finite check + max |coordinate| (the accumulators' scale)
  TRG_TRY(launch_absmax(ctx, src_dev, n, reinterpret_cast<unsigned long long*>(static_cast<char*>(cnt) + 64),
                        status));
  // the E-steps read a spatially sorted copy (trg_sort.cu)
  if (!dense) TRG_TRY(morton_sorted_copy(ctx, src_dev, n, p.a.pmax, kSlotBuild4, kSlotBuild5, &p.a.pts));
  k_extent<<<1, 256, 0, ctx->stream>>>(tree->nodes, J, p.st, target_diag, cfg->translation_tol,
                                       meta, diag_dev);
  ctx->launches += 1;
  job->p = p;
  job->G = G;
  job->J = J;
  job->K = K;
  TRG_CU(cudaEventCreate(&job->e0));
  TRG_CU(cudaEventCreate(&job->e1));
  TRG_CU(cudaEventRecord(job->e0, ctx->stream));
  return TRG_OK;
}

int em_launch(trg_ctx* ctx, EmJob* job, int seg) {
  if (job->p.seg >= 0) job->p.seg = seg;
  // per-launch handover words (grid barrier, flag, arrivals)
  TRG_CU(cudaMemsetAsync(job->p.sync, 0, 64, ctx->stream));
  void* args[] = {&job->p};
  std::unique_ptr<EmBatch> b;
  if (job->kernel == (const void*)k_em_tree) {  // a batch of one, SM-placed roles
    b.reset(new EmBatch);
    b->group = job->G;
    b->n = 1;
    b->by_sm = 1;
    b->p[0] = job->p;
    args[0] = b.get();
  }
  TRG_CU(launch_persistent(ctx, job->kernel, job->G, job->block, args, job->smem));
  ctx->launches += 1;
  return TRG_OK;
}

int em_collect(trg_ctx* ctx, EmJob* job, trg_reg_result* out) {
  EmParams& p = job->p;
  const int K = job->K;
  TRG_CU(cudaEventRecord(job->e1, ctx->stream));
  // state, traces and status word in one round trip (pinned, one synchronisation)
  int* dev_status = job->status ? job->status : ctx->status;
  const size_t tb = sizeof(double) * K;
  void* hc = nullptr;
  TRG_TRY(host_ws_get(ctx, kSlotHostCollect, sizeof(EmState) + 3 * tb + 16, &hc));
  char* h = static_cast<char*>(hc);
  TRG_CU(cudaMemcpyAsync(h, p.st, sizeof(EmState), cudaMemcpyDeviceToHost, ctx->stream));
  TRG_CU(cudaMemcpyAsync(h + sizeof(EmState), p.crit_before, tb, cudaMemcpyDeviceToHost, ctx->stream));
  TRG_CU(cudaMemcpyAsync(h + sizeof(EmState) + tb, p.crit_after, tb, cudaMemcpyDeviceToHost, ctx->stream));
  TRG_CU(cudaMemcpyAsync(h + sizeof(EmState) + 2 * tb, p.evals, tb, cudaMemcpyDeviceToHost, ctx->stream));
  TRG_CU(cudaMemcpyAsync(h + sizeof(EmState) + 3 * tb, dev_status, sizeof(int), cudaMemcpyDeviceToHost,
                         ctx->stream));
  TRG_CU(cudaStreamSynchronize(ctx->stream));
  ctx->bytes_d2h += sizeof(EmState) + 3 * tb + sizeof(int);
  EmState st;
  std::memcpy(&st, h, sizeof st);
  std::vector<double> cb(K), ca(K);
  std::vector<unsigned long long> ev(K);
  std::memcpy(cb.data(), h + sizeof(EmState), tb);
  std::memcpy(ca.data(), h + sizeof(EmState) + tb, tb);
  std::memcpy(ev.data(), h + sizeof(EmState) + 2 * tb, tb);
  int hst = 0;
  std::memcpy(&hst, h + sizeof(EmState) + 3 * tb, sizeof(int));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, job->e0, job->e1);
  cudaEventDestroy(job->e0);
  cudaEventDestroy(job->e1);
  TRG_TRY(status_result(ctx, hst, dev_status, "register_with_tree"));
  TRG_TRY(timeline_fetch(ctx));
  for (int k = 0; k < 9; ++k) out->R[k] = st.Rt[k];
  for (int k = 0; k < 3; ++k) out->t[k] = st.Rt[9 + k];
  out->iterations = st.iterations;
  out->converged = st.converged;
  out->em_seconds = ms * 1e-3;
  out->model_components = (size_t)job->J;
  const int m = std::min(st.iterations, out->trace_capacity);
  for (int i = 0; i < m; ++i) {
    if (out->criterion_trace) out->criterion_trace[i] = cb[i];
    if (out->criterion_after_trace) out->criterion_after_trace[i] = ca[i];
    if (out->eval_counts) out->eval_counts[i] = ev[i];
  }
  return TRG_OK;
}

int run_em(trg_ctx* ctx, const trg_tree_dev* tree, const double* src_dev, size_t n,
           const trg_reg_config* cfg, double target_diag, trg_reg_result* out, bool dense = false) {
  EmJob job;
  TRG_TRY(em_prepare(ctx, tree, src_dev, n, cfg, target_diag, false, 0.0, &job, dense));
  TRG_TRY(em_launch(ctx, &job, -1));
  return em_collect(ctx, &job, out);
}

// Bounding-box diagonal of a cloud (cloud_io.cpp:21-33): per-block min/max,
// the last block folds them.  min/max are exact, so the result is
// bit-identical to the reference for any reduction order.
__global__ void k_bbox(const double* __restrict__ p, size_t n, double* part, unsigned* cnt,
                       double* out) {
  __shared__ double wl[8][3], wh[8][3];  // per-warp partials (256 threads)
  __shared__ bool last;
  double l[3] = {p[0], p[1], p[2]}, h[3] = {p[0], p[1], p[2]};
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    for (int k = 0; k < 3; ++k) {
      const double v = p[3 * i + k];
      l[k] = (v < l[k]) ? v : l[k];
      h[k] = (h[k] < v) ? v : h[k];
    }
  // min / max are exact in any order: shuffles within the warp, then the
  // eight warps' partials
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
    for (int k = 0; k < 3; ++k) {
      l[k] = smin(l[k], __shfl_xor_sync(0xffffffffu, l[k], o));
      h[k] = smax(h[k], __shfl_xor_sync(0xffffffffu, h[k], o));
    }
  if ((threadIdx.x & 31) == 0)
    for (int k = 0; k < 3; ++k) {
      wl[threadIdx.x >> 5][k] = l[k];
      wh[threadIdx.x >> 5][k] = h[k];
    }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      for (int k = 0; k < 3; ++k) {
        l[k] = smin(l[k], wl[w][k]);
        h[k] = smax(h[k], wh[w][k]);
      }
    for (int k = 0; k < 3; ++k) {
      part[6 * blockIdx.x + k] = l[k];
      part[6 * blockIdx.x + 3 + k] = h[k];
    }
    __threadfence();
    last = atomicAdd(cnt, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x < 32) {
    // the partials over the lanes of one warp (min / max are exact in any
    // order), then a shuffle reduction
    __threadfence();
    for (int b = threadIdx.x; b < (int)gridDim.x; b += 32)
      for (int k = 0; k < 3; ++k) {
        l[k] = smin(l[k], __ldcg(&part[6 * b + k]));
        h[k] = smax(h[k], __ldcg(&part[6 * b + 3 + k]));
      }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
      for (int k = 0; k < 3; ++k) {
        l[k] = smin(l[k], __shfl_xor_sync(0xffffffffu, l[k], o));
        h[k] = smax(h[k], __shfl_xor_sync(0xffffffffu, h[k], o));
      }
  }
  if (last && threadIdx.x == 0) {
    double s = (h[0] - l[0]) * (h[0] - l[0]);
    s += (h[1] - l[1]) * (h[1] - l[1]);
    s += (h[2] - l[2]) * (h[2] - l[2]);
    *out = sqrt(s);
    for (int k = 0; k < 3; ++k) {
      out[2 + k] = l[k];
      out[5 + k] = h[k];
    }
    *cnt = 0u;
  }
}

// bbox of a device cloud, left on the device: od[0] = diagonal, od[2..4] =
// min, od[5..7] = max (stream-ordered, no synchronisation)
int bbox_launch(trg_ctx* ctx, const double* dev, size_t n, double** od_out) {
  void* o = nullptr;
  const int nb = 64;
  TRG_TRY(ws_get(ctx, kSlotBuild11, 64 + sizeof(double) * 6 * nb, &o));
  double* od = static_cast<double*>(o);
  TRG_CU(cudaMemsetAsync(static_cast<char*>(o) + 8, 0, 8, ctx->stream));
  k_bbox<<<nb, 256, 0, ctx->stream>>>(dev, n, od + 8, reinterpret_cast<unsigned*>(od + 1),
                                      od);
  ctx->launches += 1;
  *od_out = od;
  return TRG_OK;
}

// bbox of a device cloud: out[0] = diagonal, out[2..4] = min, out[5..7] = max
int target_bbox(trg_ctx* ctx, const double* dev, size_t n, double out8[8]) {
  double* od = nullptr;
  TRG_TRY(bbox_launch(ctx, dev, n, &od));
  TRG_CU(trg_memcpy(ctx, out8, od, sizeof(double) * 8, cudaMemcpyDeviceToHost));
  TRG_CU(cudaStreamSynchronize(ctx->stream));
  return TRG_OK;
}

double target_bbox_diagonal(trg_ctx* ctx, const double* dev, size_t n) {
  double o[8];
  if (target_bbox(ctx, dev, n, o) != TRG_OK) return 0.0;
  return o[0];
}

}  // namespace

namespace trg {
// Non-finite coordinates -> TRG_EINVAL with `msg` (validate_cloud).
int check_finite_dev(trg_ctx* ctx, const double* dev, size_t n, const char* msg) {
  if (n == 0) return TRG_OK;
  k_check_finite<<<64, 256, 0, ctx->stream>>>(dev, 3 * n, ctx->status);
  ctx->launches += 1;
  const int rc = check_status(ctx, "check_finite");
  if (rc == TRG_EINVAL) set_error(msg);
  return rc;
}

// registration.cpp:174-209 / registration.hpp:29-32 argument checks
int validate_reg_config(const trg_reg_config* cfg) {
  if (!cfg) {
    set_error("register: config is null");
    return TRG_EINVAL;
  }
  if (!(cfg->rotation_tol > 0.0) || !(cfg->translation_tol > 0.0)) {
    set_error("register: tolerances must be positive");
    return TRG_EINVAL;
  }
  if (cfg->max_em_iterations < 1) {
    set_error("register: max_em_iterations must be >= 1");
    return TRG_EINVAL;
  }
  if (cfg->variant_param < 1 && cfg->variant_kind != TRG_VARIANT_ICP) {
    set_error("register: variant parameter must be >= 1");
    return TRG_EINVAL;
  }
  if (cfg->variant_kind != TRG_VARIANT_ADAPTIVE && cfg->variant_kind != TRG_VARIANT_TREE &&
      cfg->variant_kind != TRG_VARIANT_FLAT && cfg->variant_kind != TRG_VARIANT_ICP) {
    set_error("register: unknown variant");
    return TRG_EINVAL;
  }
  {  // initial_transform.is_valid(1e-9) (geometry.cpp:22-38)
    const double* R = cfg->initial_R;
    double o = 0.0;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        double s = R[i] * R[j];
        s += R[3 + i] * R[3 + j];
        s += R[6 + i] * R[6 + j];
        const double d = s - (i == j ? 1.0 : 0.0);
        o += d * d;
      }
    const double det = R[0] * (R[4] * R[8] - R[7] * R[5]) - R[3] * (R[1] * R[8] - R[7] * R[2]) +
                       R[6] * (R[1] * R[5] - R[4] * R[2]);
    bool fin = true;
    for (int k = 0; k < 9; ++k) fin = fin && std::isfinite(R[k]);
    for (int k = 0; k < 3; ++k) fin = fin && std::isfinite(cfg->initial_t[k]);
    if (!fin || !(std::sqrt(o) <= 1e-9) || !(std::fabs(det - 1.0) <= 1e-9)) {
      set_error("register: invalid initial transform");
      return TRG_EINVAL;
    }
  }
  return TRG_OK;
}
}  // namespace trg

extern "C" {

int trg_solve_mstep(trg_ctx* ctx, const trg_tree_dev* tree, const double* m0, const double* m1,
                    uint64_t total_points, trg_mstep_solution* out) {
  trg::NvtxRange nvtx_range_("trg_solve_mstep");
  if (!tree || tree->n_nodes == 0) {
    set_error("make_virtual_points: moment/component count mismatch");
    return TRG_EINVAL;
  }
  if (total_points == 0) {
    set_error("make_virtual_points: no points were associated");
    return TRG_EINVAL;
  }
  TRG_CU(cudaSetDevice(ctx->device));
  const int J = tree->n_nodes;
  std::vector<double> h((size_t)J * 4);
  for (int j = 0; j < J; ++j) {
    h[4 * j] = m0[j];
    for (int k = 0; k < 3; ++k) h[4 * j + 1 + k] = m1[3 * j + k];
  }
  void *mom, *so;
  TRG_TRY(ws_get(ctx, kSlotMoments, sizeof(double) * 4 * (size_t)J, &mom));
  TRG_TRY(ws_get(ctx, kSlotSolve, sizeof(SolveOut), &so));
  TRG_CU(trg_memcpy(ctx, mom, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice));
  k_solve<<<1, 256, 0, ctx->stream>>>(tree->nodes, J, static_cast<double*>(mom),
                                      (double)total_points, static_cast<SolveOut*>(so),
                                      ctx->status);
  ctx->launches += 1;
  SolveOut o;
  TRG_CU(trg_memcpy(ctx, &o, so, sizeof o, cudaMemcpyDeviceToHost));
  TRG_TRY(check_status(ctx, "solve_mstep"));
  out->n_virtual_points = o.nvp;
  out->condition_estimate = o.cond;
  if (o.degenerate) {
    set_error(o.nvp < 3 ? "solve_mstep: fewer than 3 contributing components"
                        : "solve_mstep: normal equations condition estimate exceeds limit");
    return TRG_EDEGENERATE;
  }
  for (int k = 0; k < 3; ++k) {
    out->omega[k] = o.omega[k];
    out->translation[k] = o.trans[k];
    out->delta_t[k] = o.dt[k];
  }
  for (int k = 0; k < 9; ++k) out->delta_R[k] = o.dR[k];
  out->criterion_before = o.crit_before;
  out->criterion_after = o.crit_after;
  return TRG_OK;
}

int trg_make_virtual_points(trg_ctx* ctx, int n_components, const double* m0, const double* m1,
                            uint64_t total_points, int* index, double* pi_star, double* mu_star,
                            int* n_out) {
  trg::NvtxRange nvtx_range_("trg_make_virtual_points");
  if (total_points == 0) {
    set_error("make_virtual_points: no points were associated");
    return TRG_EINVAL;
  }
  if (n_components <= 0) {
    *n_out = 0;
    return TRG_OK;
  }
  TRG_CU(cudaSetDevice(ctx->device));
  const int J = n_components;
  std::vector<double> h((size_t)J * 4);
  for (int j = 0; j < J; ++j) {
    h[4 * j] = m0[j];
    for (int k = 0; k < 3; ++k) h[4 * j + 1 + k] = m1[3 * j + k];
  }
  void* buf = nullptr;
  const size_t bytes = sizeof(double) * 8 * (size_t)J + sizeof(int) * ((size_t)J + 1);
  TRG_TRY(ws_get(ctx, kSlotSolve, bytes + 64, &buf));
  double* dmom = static_cast<double*>(buf);
  double* dpimu = dmom + 4 * J;
  int* didx = reinterpret_cast<int*>(dpimu + 4 * J);
  int* dcnt = didx + J;
  TRG_CU(trg_memcpy(ctx, dmom, h.data(), sizeof(double) * 4 * J, cudaMemcpyHostToDevice));
  k_make_vps<<<1, 256, 0, ctx->stream>>>(dmom, J, (double)total_points, didx, dpimu, dcnt);
  ctx->launches += 1;
  int cnt = 0;
  TRG_CU(trg_memcpy(ctx, &cnt, dcnt, sizeof(int), cudaMemcpyDeviceToHost));
  TRG_CU(cudaStreamSynchronize(ctx->stream));
  std::vector<double> pm((size_t)cnt * 4);
  std::vector<int> ix(cnt);
  if (cnt > 0) {
    TRG_CU(trg_memcpy(ctx, pm.data(), dpimu, sizeof(double) * 4 * cnt, cudaMemcpyDeviceToHost));
    TRG_CU(trg_memcpy(ctx, ix.data(), didx, sizeof(int) * cnt, cudaMemcpyDeviceToHost));
  }
  TRG_TRY(check_status(ctx, "make_virtual_points"));
  for (int v = 0; v < cnt; ++v) {
    index[v] = ix[v];
    pi_star[v] = pm[4 * v];
    for (int k = 0; k < 3; ++k) mu_star[3 * v + k] = pm[4 * v + 1 + k];
  }
  *n_out = cnt;
  return TRG_OK;
}

int trg_solve_mstep_vps(trg_ctx* ctx, int n_vps, const double* pi_star, const double* mu_star,
                        const double* comp_mean, const double* comp_lambdas,
                        const double* comp_axes, trg_mstep_solution* out) {
  trg::NvtxRange nvtx_range_("trg_solve_mstep_vps");
  if (n_vps < 0) {
    set_error("solve_mstep: bad virtual point count");
    return TRG_EINVAL;
  }
  TRG_CU(cudaSetDevice(ctx->device));
  const int n = n_vps;
  std::vector<DNode> comps(std::max(1, n));
  std::vector<double> pimu((size_t)std::max(1, n) * 4);
  for (int v = 0; v < n; ++v) {
    DNode& d = comps[v];
    for (int r = 0; r < 3; ++r) {
      d.mean[r] = comp_mean[3 * v + r];
      d.lam[r] = comp_lambdas[3 * v + r];
      d.il[r] = 1.0 / d.lam[r];
      for (int k = 0; k < 3; ++k) d.axT[3 * r + k] = comp_axes[9 * v + 3 * k + r];
    }
    set_prec(d.axT, d.il, d.prec);
    pimu[4 * v] = pi_star[v];
    for (int k = 0; k < 3; ++k) pimu[4 * v + 1 + k] = mu_star[3 * v + k];
  }
  void* buf = nullptr;
  const size_t cb = sizeof(DNode) * comps.size(), pb = sizeof(double) * pimu.size();
  TRG_TRY(ws_get(ctx, kSlotSolve, cb + pb + sizeof(SolveOut) + 256, &buf));
  char* B = static_cast<char*>(buf);
  DNode* dc = reinterpret_cast<DNode*>(B);
  double* dp = reinterpret_cast<double*>(B + cb);
  SolveOut* dso = reinterpret_cast<SolveOut*>(B + ((cb + pb + 15) & ~size_t(15)));
  TRG_CU(trg_memcpy(ctx, dc, comps.data(), cb, cudaMemcpyHostToDevice));
  TRG_CU(trg_memcpy(ctx, dp, pimu.data(), pb, cudaMemcpyHostToDevice));
  k_solve_vps<<<1, 256, 0, ctx->stream>>>(dc, dp, n, dso, ctx->status);
  ctx->launches += 1;
  SolveOut o;
  TRG_CU(trg_memcpy(ctx, &o, dso, sizeof o, cudaMemcpyDeviceToHost));
  TRG_TRY(check_status(ctx, "solve_mstep"));
  out->n_virtual_points = o.nvp;
  out->condition_estimate = o.cond;
  if (o.degenerate) {
    set_error(o.nvp < 3 ? "solve_mstep: fewer than 3 contributing components"
                        : "solve_mstep: normal equations condition estimate exceeds limit");
    return TRG_EDEGENERATE;
  }
  for (int k = 0; k < 3; ++k) {
    out->omega[k] = o.omega[k];
    out->translation[k] = o.trans[k];
    out->delta_t[k] = o.dt[k];
  }
  for (int k = 0; k < 9; ++k) out->delta_R[k] = o.dR[k];
  out->criterion_before = o.crit_before;
  out->criterion_after = o.crit_after;
  return TRG_OK;
}

int trg_register_with_tree(trg_ctx* ctx, const trg_tree_dev* tree, const double* xyz, size_t n,
                           int xyz_on_device, const trg_reg_config* cfg, double target_diag,
                           trg_reg_result* out) {
  trg::NvtxRange nvtx_range_("trg_register_with_tree");
  if (n == 0 || !xyz) {
    set_error("register: bad source cloud");
    return TRG_EINVAL;
  }
  if (!tree || tree->n_nodes == 0) {
    set_error("association: empty model");
    return TRG_EINVAL;
  }
  if (cfg->max_em_iterations < 1) {
    set_error("register: max_em_iterations must be >= 1");
    return TRG_EINVAL;
  }
  TRG_CU(cudaSetDevice(ctx->device));
  const double* dev = nullptr;
  TRG_TRY(stage_points_public(ctx, xyz, n, xyz_on_device, kSlotPoints2, &dev));
  const int rc = run_em(ctx, tree, dev, n, cfg, target_diag, out);
  if (rc == TRG_EINVAL) set_error("register: bad source cloud");
  return rc;
}

// register_clouds for the tree variants with one host synchronisation: the
// target's bbox, the build and the EM are queued back to back on the stream
// (the EM reads the tree's size and the diagonal on the device), then the
// build and the EM are collected.  An entry-buffer overflow (the EM saw
// meta->ok == 0 and did nothing) re-queues both with the grown allocation.
static int register_tree_async(trg_ctx* ctx, const double* tgt, size_t n_target,
                               const double* src, size_t n_source, bool src_deferred,
                               const trg_reg_config* cfg, trg_reg_result* out) {
  trg_model_config mc = cfg->model_config;
  mc.max_level = cfg->variant_param;
  double* od = nullptr;
  TRG_TRY(bbox_launch(ctx, tgt, n_target, &od));
  AsyncBuild* ab = nullptr;
  int rc = TRG_OK;
  for (int attempt = 0; attempt < 4; ++attempt) {
    cudaEvent_t e0, e1;
    TRG_CU(cudaEventCreate(&e0));
    TRG_CU(cudaEventCreate(&e1));
    TRG_CU(cudaEventRecord(e0, ctx->stream));
    trg_tree_dev* tree = nullptr;
    const TreeMeta* meta = nullptr;
    ctx->build_into_scratch = true;
    rc = build_async_start(ctx, tgt, n_target, &mc, &ab, &tree, &meta);
    ctx->build_into_scratch = false;
    if (rc == TRG_OK) rc = cudaEventRecord(e1, ctx->stream) == cudaSuccess ? TRG_OK : TRG_ECUDA;
    if (rc == TRG_OK && src_deferred) rc = stage_wait(ctx);
    EmJob job;
    if (rc == TRG_OK) rc = em_prepare(ctx, tree, src, n_source, cfg, 0.0, false, 0.0, &job, false, meta, od);
    if (rc == TRG_OK) rc = em_launch(ctx, &job, -1);
    if (rc != TRG_OK) {
      if (job.e0) cudaEventDestroy(job.e0);
      if (job.e1) cudaEventDestroy(job.e1);
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
      cudaStreamSynchronize(ctx->stream);  // nothing queued may outlive the call
      break;
    }
    trg_tree_dev* built = nullptr;
    bool retry = false;
    rc = build_async_finish(ctx, ab, &built, &retry);  // synchronises the stream
    if (rc == TRG_OK && retry) {
      cudaEventDestroy(job.e0);
      cudaEventDestroy(job.e1);
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
      continue;
    }
    if (rc != TRG_OK) {  // the EM's events / status word are dropped with it
      cudaEventDestroy(job.e0);
      cudaEventDestroy(job.e1);
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
      cudaMemsetAsync(ctx->status2, 0, sizeof(int), ctx->stream);
      break;
    }
    job.J = built->n_nodes;
    rc = em_collect(ctx, &job, out);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (rc == TRG_OK) out->model_build_seconds = ms * 1e-3;
    build_async_free(ab);
    return rc;
  }
  build_async_free(ab);
  if (src_deferred) cudaStreamSynchronize(ctx->side);  // no copy may outlive a failed call
  if (rc == TRG_OK) {
    set_error("build_tree: entry buffer growth did not converge");
    rc = TRG_ERUNTIME;
  }
  return rc;
}

// registration.cpp:174-209 register_clouds (adaptive:L / tree:L):
// validate, build the tree on the target, then the EM loop.
int trg_register_clouds(trg_ctx* ctx, const double* target, size_t n_target,
                        const double* source, size_t n_source, int on_device,
                        const trg_reg_config* cfg, trg_reg_result* out) {
  trg::NvtxRange nvtx_range_("trg_register_clouds");
  if (n_target == 0 || n_source == 0 || !target || !source) {
    set_error("register: empty cloud");
    return TRG_EINVAL;
  }
  TRG_TRY(validate_reg_config(cfg));
  TRG_CU(cudaSetDevice(ctx->device));
  const double* src = nullptr;
  const double* tgt = nullptr;
  if (cfg->variant_kind == TRG_VARIANT_ADAPTIVE || cfg->variant_kind == TRG_VARIANT_TREE) {
    // target first; a pinned source streams in on the side stream under the
    // build (the EM waits for it)
    bool deferred = false;
    TRG_TRY(stage_points_public(ctx, target, n_target, on_device, kSlotPoints, &tgt));
    TRG_TRY(stage_points_side(ctx, source, n_source, on_device, kSlotPoints2, &src, &deferred));
    return register_tree_async(ctx, tgt, n_target, src, n_source, deferred, cfg, out);
  }
  TRG_TRY(stage_points_public(ctx, source, n_source, on_device, kSlotPoints2, &src));
  TRG_TRY(stage_points_public(ctx, target, n_target, on_device, kSlotPoints, &tgt));
  if (cfg->variant_kind == TRG_VARIANT_ICP) {  // registration.cpp:205-206
    TRG_TRY(check_finite_dev(ctx, tgt, n_target, "register: non-finite coordinates"));
    TRG_TRY(check_finite_dev(ctx, src, n_source, "register: non-finite coordinates"));
    return register_icp_dev(ctx, tgt, n_target, src, n_source, cfg,
                            target_bbox_diagonal(ctx, tgt, n_target), out);
  }
  cudaEvent_t e0, e1;
  TRG_CU(cudaEventCreate(&e0));
  TRG_CU(cudaEventCreate(&e1));
  TRG_CU(cudaEventRecord(e0, ctx->stream));
  const bool flat = cfg->variant_kind == TRG_VARIANT_FLAT;
  trg_model_config mc = cfg->model_config;
  if (!flat) mc.max_level = cfg->variant_param;
  trg_tree_dev* tree = nullptr;
  ctx->build_into_scratch = true;
  int rc;
  if (flat) {  // registration.cpp:191-202: build_flat_gmm + dense E-step
    rc = check_finite_dev(ctx, tgt, n_target, "point cloud has non-finite coordinates");
    if (rc == TRG_OK) rc = flat_build(ctx, tgt, n_target, (size_t)cfg->variant_param, &mc, &tree, nullptr);
  } else {
    rc = trg_build_tree(ctx, tgt, n_target, 1, &mc, &tree, nullptr);
  }
  ctx->build_into_scratch = false;
  if (rc != TRG_OK) return rc;
  TRG_CU(cudaEventRecord(e1, ctx->stream));
  const double diag = target_bbox_diagonal(ctx, tgt, n_target);
  rc = run_em(ctx, tree, src, n_source, cfg, diag, out, flat);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  out->model_build_seconds = ms * 1e-3;
  trg_tree_free(ctx, tree);
  if (rc == TRG_EINVAL) set_error("register: non-finite coordinates");
  return rc;
}

}  // extern "C"

// ------------------------------------------------------------ sharded EM
extern "C" int trg_register_clouds_sharded(trg_comm* comm, const double* const* target,
                                           const size_t* n_target, const double* const* source,
                                           const size_t* n_source, int on_device,
                                           const trg_reg_config* cfg, trg_reg_result* out) {
  trg::NvtxRange nvtx_range_("trg_register_clouds_sharded");
  if (!comm || !target || !source || !n_target || !n_source || !out) {
    set_error("register_sharded: bad argument");
    return TRG_EINVAL;
  }
  TRG_TRY(validate_reg_config(cfg));
  if (cfg->variant_kind == TRG_VARIANT_FLAT || cfg->variant_kind == TRG_VARIANT_ICP) {
    set_error("register_sharded: the sharded path implements adaptive:L and tree:L");
    return TRG_EINVAL;
  }
  const int S = comm->local;
  trg_ctx* ctx = comm->ctx;
  TRG_CU(cudaSetDevice(ctx->device));
  // global point counts
  std::vector<double> cnt((size_t)S * 2);
  for (int i = 0; i < S; ++i) {
    cnt[(size_t)i * 2] = (double)n_target[i];
    cnt[(size_t)i * 2 + 1] = (double)n_source[i];
  }
  TRG_TRY(comm_host_reduce(comm, cnt.data(), 2, 0));
  if (!(cnt[0] > 0.0) || !(cnt[1] > 0.0)) {
    set_error("register: empty cloud");
    return TRG_EINVAL;
  }
  const double n_total = cnt[1];
  std::vector<const double*> tdev(S), sdev(S);
  for (int i = 0; i < S; ++i) {
    TRG_TRY(stage_points_public(comm->shard_ctx[i], source[i], n_source[i], on_device,
                                kSlotPoints2, &sdev[i]));
    TRG_TRY(stage_points_public(comm->shard_ctx[i], target[i], n_target[i], on_device, kSlotPoints,
                                &tdev[i]));
  }
  cudaEvent_t e0, e1;
  TRG_CU(cudaEventCreate(&e0));
  TRG_CU(cudaEventCreate(&e1));
  TRG_CU(cudaEventRecord(e0, ctx->stream));
  // ---- sharded build (trees owned by the shard contexts)
  trg_model_config mc = cfg->model_config;
  mc.max_level = cfg->variant_param;
  TRG_TRY(check_model_config(&mc));
  std::vector<trg_tree_dev*> trees(S, nullptr);
  for (int i = 0; i < S; ++i) comm->shard_ctx[i]->build_into_scratch = true;
  int rc = build_sharded_dev(comm, tdev.data(), n_target, &mc, trees.data(), nullptr);
  for (int i = 0; i < S; ++i) comm->shard_ctx[i]->build_into_scratch = false;
  if (rc != TRG_OK) return rc;
  TRG_CU(cudaEventRecord(e1, ctx->stream));
  // ---- global bounding-box diagonal of the target (cloud_io.cpp:21-33)
  std::vector<double> lo((size_t)S * 3, INFINITY), hi((size_t)S * 3, -INFINITY);
  for (int i = 0; i < S; ++i) {
    if (n_target[i] == 0) continue;
    double o[8];
    TRG_TRY(target_bbox(comm->shard_ctx[i], tdev[i], n_target[i], o));
    for (int k = 0; k < 3; ++k) {
      lo[(size_t)i * 3 + k] = o[2 + k];
      hi[(size_t)i * 3 + k] = o[5 + k];
    }
  }
  TRG_TRY(comm_host_reduce(comm, lo.data(), 3, 2));
  TRG_TRY(comm_host_reduce(comm, hi.data(), 3, 1));
  double dd = (hi[0] - lo[0]) * (hi[0] - lo[0]);
  dd += (hi[1] - lo[1]) * (hi[1] - lo[1]);
  dd += (hi[2] - lo[2]) * (hi[2] - lo[2]);
  const double diag = std::sqrt(dd);
  // ---- sharded EM: per iteration the per-node (m0, m1) + counters are
  // all-reduced; every shard solves and updates T identically
  std::vector<EmJob> job(S);
  for (int i = 0; i < S; ++i)
    TRG_TRY(em_prepare(comm->shard_ctx[i], trees[i], sdev[i], n_source[i], cfg, diag, true,
                       n_total, &job[i]));
  std::vector<double*> xm(S);
  for (int i = 0; i < S; ++i) xm[i] = job[i].p.xmom;
  const int K = cfg->max_em_iterations;
  const size_t nx = 4 * (size_t)job[0].J + 2;
  for (int it = 0; it <= K; ++it) {
    for (int i = 0; i < S; ++i) TRG_TRY(em_launch(comm->shard_ctx[i], &job[i], it));
    if (it < K) TRG_TRY(comm_allreduce_sum(comm, xm.data(), nx));
  }
  rc = em_collect(comm->shard_ctx[0], &job[0], out);
  for (int i = 1; i < S; ++i) {
    trg_reg_result tmp{};
    const int r2 = em_collect(comm->shard_ctx[i], &job[i], &tmp);
    if (rc == TRG_OK) rc = r2;
  }
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  out->model_build_seconds = ms * 1e-3;
  return rc;
}

// ------------------------------------------------------------ batched pairs
// trg_register_batch for the tree variants (BASELINE config C5): the pairs
// run in waves of up to kBatchInflightMax.  Each pair of a wave has a worker context
// (own stream, workspace, scratch tree, status words) that stages its
// clouds, its target's bbox and its build state; the wave's builds are then
// ONE k_build_batch + ONE k_calibrate_batch launch and its EMs ONE
// k_em_tree launch on the batch context's stream, every pair on its own
// CTA group of the co-resident (cooperative) grid with group barriers.  The
// results are bit-identical to trg_register_clouds (group size does not
// enter any result: tests/test_grid_invariance_gpu.py).
namespace trg {

namespace batch_detail {

int em_batch_launch(trg_ctx* ctx, EmJob* const* js, int m) {
  std::unique_ptr<EmBatch> b(new EmBatch);
  b->n = m;
  b->by_sm = 0;
  for (int k = 0; k < m; ++k) b->p[k] = js[k]->p;
  const size_t smem = sizeof(DNode) * kStageNodes;
  TRG_CU(set_dynamic_smem((const void*)k_em_tree, smem));
  b->group = persistent_grid(ctx, (const void*)k_em_tree, kEmBlock, smem) / m;
  if (b->group < 2) {
    set_error("register_batch: too many pairs in flight for the device");
    return TRG_EINVAL;
  }
  void* args[] = {b.get()};
  TRG_CU(launch_persistent(ctx, (const void*)k_em_tree, b->group * m, kEmBlock, args, smem));
  ctx->launches += 1;
  return TRG_OK;
}

struct BatchSlot {
  AsyncBuild* ab = nullptr;
  trg_tree_dev* tree = nullptr;
  const TreeMeta* meta = nullptr;
  double* od = nullptr;
  const double* tgt = nullptr;
  const double* src = nullptr;
  EmJob job;
  cudaEvent_t b0 = nullptr, b1 = nullptr;  // build span (shared by the wave)
};

void slot_release(BatchSlot& s) {
  if (s.job.e0) cudaEventDestroy(s.job.e0);
  if (s.job.e1) cudaEventDestroy(s.job.e1);
  if (s.b0) cudaEventDestroy(s.b0);
  if (s.b1) cudaEventDestroy(s.b1);
  s.job.e0 = s.job.e1 = s.b0 = s.b1 = nullptr;
  if (s.ab) build_async_free(s.ab);
  s.ab = nullptr;
}

// One wave: pairs [base, base + m) on workers 0..m-1.
int batch_wave(trg_ctx* ctx, int base, int m, const double* const* targets,
               const size_t* n_targets, const double* const* sources, const size_t* n_sources,
               int on_device, const trg_reg_config* cfg, trg_reg_result* out,
               std::vector<BatchSlot>& sl, std::vector<cudaEvent_t>& ev, cudaEvent_t ev_main) {
  trg_model_config mc = cfg->model_config;
  mc.max_level = cfg->variant_param;
  std::vector<AsyncBuild*> abs(m);
  std::vector<EmJob*> jobs(m);
  // 1. per pair: clouds, target bbox, build state (worker streams)
  for (int k = 0; k < m; ++k) {
    trg_ctx* w = ctx->workers[k];
    const int i = base + k;
    BatchSlot& s = sl[k];
    if (n_targets[i] == 0 || n_sources[i] == 0 || !targets[i] || !sources[i]) {
      set_error("register: empty cloud");
      return TRG_EINVAL;
    }
    TRG_TRY(stage_points_public(w, targets[i], n_targets[i], on_device, kSlotPoints, &s.tgt));
    TRG_TRY(stage_points_public(w, sources[i], n_sources[i], on_device, kSlotPoints2, &s.src));
    TRG_TRY(bbox_launch(w, s.tgt, n_targets[i], &s.od));
    TRG_CU(cudaEventCreate(&s.b0));
    TRG_CU(cudaEventCreate(&s.b1));
    TRG_CU(cudaEventRecord(s.b0, w->stream));
    w->build_into_scratch = true;
    const int rc = build_async_start(w, s.tgt, n_targets[i], &mc, &s.ab, &s.tree, &s.meta, false);
    w->build_into_scratch = false;
    TRG_TRY(rc);
    abs[k] = s.ab;
    TRG_CU(cudaEventRecord(ev[k], w->stream));
    TRG_CU(cudaStreamWaitEvent(ctx->stream, ev[k], 0));
  }
  // 2. the wave's builds: one k_build_batch + one k_calibrate_batch
  TRG_TRY(build_batch_launch(ctx, abs.data(), m));
  TRG_CU(cudaEventRecord(ev_main, ctx->stream));
  // 3. EM state behind the builds (worker streams)
  for (int k = 0; k < m; ++k) {
    trg_ctx* w = ctx->workers[k];
    BatchSlot& s = sl[k];
    TRG_CU(cudaStreamWaitEvent(w->stream, ev_main, 0));
    TRG_CU(cudaEventRecord(s.b1, w->stream));
    TRG_TRY(em_prepare(w, s.tree, s.src, n_sources[base + k], cfg, 0.0, false, 0.0, &s.job, false,
                       s.meta, s.od));
    TRG_CU(cudaMemsetAsync(s.job.p.sync, 0, 64, w->stream));  // the launch's handover words
    jobs[k] = &s.job;
    TRG_CU(cudaEventRecord(ev[k], w->stream));
    TRG_CU(cudaStreamWaitEvent(ctx->stream, ev[k], 0));
  }
  // 4. the wave's EMs: one k_em_tree
  TRG_TRY(em_batch_launch(ctx, jobs.data(), m));
  TRG_CU(cudaEventRecord(ev_main, ctx->stream));
  // 5. collect (an entry-buffer overflow re-runs that pair alone, with the
  // grown allocation its worker now holds)
  int rc_all = TRG_OK;
  for (int k = 0; k < m; ++k) {
    trg_ctx* w = ctx->workers[k];
    BatchSlot& s = sl[k];
    const int i = base + k;
    TRG_CU(cudaStreamWaitEvent(w->stream, ev_main, 0));
    trg_tree_dev* built = nullptr;
    bool retry = false;
    int rc = build_async_finish(w, s.ab, &built, &retry);  // synchronises the worker stream
    if (rc == TRG_OK && retry) {
      cudaMemsetAsync(w->status2, 0, sizeof(int), w->stream);
      rc = trg_register_clouds(w, targets[i], n_targets[i], sources[i], n_sources[i], on_device,
                               cfg, &out[i]);
    } else if (rc == TRG_OK) {
      s.job.J = built->n_nodes;
      rc = em_collect(w, &s.job, &out[i]);
      s.job.e0 = s.job.e1 = nullptr;  // destroyed by em_collect
      float ms = 0.f;
      cudaEventElapsedTime(&ms, s.b0, s.b1);
      if (rc == TRG_OK) out[i].model_build_seconds = ms * 1e-3;
    } else {
      cudaMemsetAsync(w->status2, 0, sizeof(int), w->stream);
      if (rc == TRG_EINVAL && trg_last_error()[0] == 'b')
        set_error("point cloud has non-finite coordinates or no mass");
    }
    if (rc != TRG_OK && rc_all == TRG_OK) {
      rc_all = rc;
      set_error("register_batch: pair " + std::to_string(i) + ": " + trg_last_error());
    }
  }
  return rc_all;
}

}  // namespace batch_detail

using namespace batch_detail;

int register_batch_fused(trg_ctx* ctx, int n_pairs, const double* const* targets,
                         const size_t* n_targets, const double* const* sources,
                         const size_t* n_sources, int on_device, const trg_reg_config* cfg,
                         int inflight, trg_reg_result* out) {
  TRG_TRY(validate_reg_config(cfg));
  for (int i = 0; i < n_pairs; ++i)  // argument errors before any work
    if (n_targets[i] == 0 || n_sources[i] == 0 || !targets[i] || !sources[i]) {
      set_error("register_batch: pair " + std::to_string(i) + ": register: empty cloud");
      return TRG_EINVAL;
    }
  inflight = std::min({inflight, n_pairs, kBatchInflightMax, kMaxEmBatch});
  while ((int)ctx->workers.size() < inflight) {
    trg_ctx* w = nullptr;
    TRG_TRY(trg_ctx_create(ctx->device, &w));
    ctx->workers.push_back(w);
  }
  // full-device workers: their workspaces are sized for a whole-grid run
  for (int k = 0; k < inflight; ++k) TRG_TRY(trg_ctx_set_sm_budget(ctx->workers[k], ctx->device_sms));
  // inputs the caller produced on its own stream must be complete
  TRG_CU(cudaStreamSynchronize(ctx->stream));
  std::vector<uint64_t> l0(inflight), h0(inflight), d0(inflight);
  for (int k = 0; k < inflight; ++k) {
    l0[k] = ctx->workers[k]->launches;
    h0[k] = ctx->workers[k]->bytes_h2d;
    d0[k] = ctx->workers[k]->bytes_d2h;
  }
  std::vector<cudaEvent_t> ev(inflight, nullptr);
  cudaEvent_t ev_main = nullptr;
  int rc = TRG_OK;
  for (int k = 0; k < inflight && rc == TRG_OK; ++k)
    if (cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming) != cudaSuccess) rc = TRG_ECUDA;
  if (rc == TRG_OK && cudaEventCreateWithFlags(&ev_main, cudaEventDisableTiming) != cudaSuccess)
    rc = TRG_ECUDA;
  // every wave runs (the other pairs' results are filled when one fails);
  // the call returns the status of the lowest-index failing pair
  std::string first_msg;
  for (int base = 0; base < n_pairs && rc != TRG_ECUDA; base += inflight) {
    const int m = std::min(inflight, n_pairs - base);
    std::vector<BatchSlot> sl(m);
    const int rw = batch_wave(ctx, base, m, targets, n_targets, sources, n_sources, on_device, cfg,
                              out, sl, ev, ev_main);
    if (rw != TRG_OK) {  // nothing queued may outlive the call
      cudaStreamSynchronize(ctx->stream);
      for (int k = 0; k < m; ++k) cudaStreamSynchronize(ctx->workers[k]->stream);
      if (rc == TRG_OK) {
        rc = rw;
        first_msg = trg_last_error();
      }
    }
    for (auto& s : sl) slot_release(s);
  }
  if (rc != TRG_OK && !first_msg.empty()) set_error(first_msg);
  for (auto e : ev)
    if (e) cudaEventDestroy(e);
  if (ev_main) cudaEventDestroy(ev_main);
  for (int k = 0; k < inflight; ++k) {
    ctx->launches += ctx->workers[k]->launches - l0[k];
    ctx->bytes_h2d += ctx->workers[k]->bytes_h2d - h0[k];
    ctx->bytes_d2h += ctx->workers[k]->bytes_d2h - d0[k];
  }
  return rc;
}

}  // namespace trg
