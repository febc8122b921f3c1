// Tree construction (build_tree, gmm.cpp:584-657) as ONE persistent
// cooperative kernel: every expansion round processes all frontier nodes of
// a level at once over a level-wide, node-sorted entry buffer (K1..K6 of
// SURVEY.md §2b), then leaf calibration (gmm.cpp:523-580) reuses the K7
// association code.  No float atomics: per-tile partials are combined in
// tile order by the last-arriving CTA of each node ("last arriver").
//
// Round r expands K_r nodes (r = 0: the virtual root over all N points).
// Phase schedule of a round (I = em_iterations_per_node, default 8):
//   p = 0          list_moments pass 1 (+ heaviest entry = FPS seed 0)
//   p = 1          list_moments pass 2; corner seeds + corner init; FPS round 1
//   p = 2..7       FPS rounds 2..7 (farthest_point_seeds, gmm.cpp:267-303)
//   corner fit     EM iterations at p = 2..I+1, final pass at p = I+2
//   FPS fit        init after p = 7, EM at p = 8..I+7, final pass at p = I+8
//   p = I+9        candidate choice + survivors done; partition count pass
//   p = I+10       layout: create tree nodes, next round's segments (CTA 0)
//   p = I+11       partition write pass (skipped in the last round)
#include <cub/block/block_scan.cuh>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <vector>

#include "trg_gmm.cuh"

namespace trg {

constexpr int kTile = 256;     // entries per tile (tiles never span nodes)
constexpr int kRec = 210;      // doubles per tile partial record
constexpr int kOffEm = 0;      // EM moments: cand c at c*81: comp*10 + {m0,m1[3],m2[6]}, ll at 80
constexpr int kOffFin = 162;   // final pass: cand c at 162 + 9c: ll, child_mass[8]
constexpr int kOffFps = 180;   // FPS argmax: score, index
constexpr int kOffMom1 = 182;  // m0, m1[3], wmax, wmax index
constexpr int kOffMom2 = 188;  // m2[6]
constexpr int kOffCnt = 194;   // partition: count[8], mass[8]



struct RoundNodes {  // per expanding node k of a round (ping-pong by round parity)
  int* tree_id;      // tree node being expanded (-1: virtual root)
  int* seg;          // entry segment start
  int* len;          // entry count
  int* tile0;        // first tile
  int* ntiles;
};

struct NodeFit {  // per expanding node k (current round only)
  double* mass;      // [K]
  double* ref;       // [K][3]  first entry's point
  double* mean;      // [K][3]
  double* scatter;   // [K][9]
  double* floorv;    // [K]
  double* seeds;     // [K][8][3] FPS seeds
  int* wmax_idx;     // [K]
  GComp* comps;      // [K][2][8]
  double* final_ll;  // [K][2]
  double* cmass;     // [K][2][8]
  int* kept;         // [K]
  int* ok;           // [K]
  int* ns;           // [K]
  int* surv;         // [K][8]
  double* smass;     // [K][8]  survivor (child) masses
  double* stotal;    // [K]
  int* next_seg;     // [K][8]  child segment start in next round (-1: not expanded)
  unsigned* arrive;  // [K]
};

struct BuildState {
  int round, J, done;
  int Kp[2], Tp[2], Ep[2];  // round sizes by parity
  int status_overflow;
  int need_E, need_K, need_T;
  // calibration
  int cal_pass;
  int root_count;
  int exp_base;  // expansions done in earlier rounds
  int n_exp;
  int lvl_start[9];
  double drift;
  int cal_done;  // sharded calibration: drift reached the stop test
  unsigned long long cal_evals;
  unsigned long long E_round[8];
  int K_round[8];
};

struct BuildParams {
  const double* pts;
  size_t n;
  int L, em_iters;
  double min_points, eps, abs_floor;
  // capacities
  int Kmax, Tmax, Emax;
  // round buffers (index by parity)
  double* ex[2];
  double* ey[2];
  double* ez[2];
  double* ew[2];
  RoundNodes rn[2];
  int* tile_node[2];
  int* tile_start[2];
  int* tile_len[2];
  NodeFit nf;
  double* partial;    // [kRec][Tmax] field-major: a field of a node's consecutive tiles is contiguous
  double* nodered;    // [Kmax][kRec] per-node reduced record
  unsigned* fdone;    // [Kmax] fields reduced (per phase)
  TreeMeta* meta;     // published by k_calibrate for work queued behind the build
  double* tile_base;  // [Tmax][8] child base offsets within node's child segment
  double* min_d2;     // [Emax]
  double* emit;       // [Emax][8]
  // tree
  DNode* nodes;
  double* cov;
  int capacity;
  // calibration association
  AssocParams a;
  double* cal_moments;  // [capacity] branch masses of a calibration pass
  long long* cal_acc;   // [3][capacity][10][3] exact leaf accumulators (trg_fx.cuh)
  unsigned long long* pmax_bits;  // max |coordinate| of the cloud (bits; k_init_entries)
  double* cta_drift;    // [G]
  unsigned* cal_arrive;  // [capacity + 1]; slot capacity: leaf arrivals of a calibration pass
  unsigned long long* drift_bits;  // [2] per-pass max drift (bits of a double >= 0)
  int* layout_scratch;  // [7 * 8 * Kmax]
  double* ll_trace;     // [capacity][2][em_iters + 1] per expansion, both candidates
  int* kept_exp;        // [capacity] kept candidate per expansion
  unsigned* bar;  // [0]: k_build's grid barrier, [8]: k_calibrate's (other grid size)
  BuildState* st;
  Timeline* tl;
  int* status;
  int want_traces;  // per-iteration log-likelihoods only feed BuildDiagnostics (gmm.cpp:240)
  // Point-sharded mode (trg_build_tree_sharded): seg >= 0 runs
  // one segment between two exchange points (k_build: the per-node phase
  // records; k_calibrate: the leaf moments) and exits; the host all-reduces
  // nodered (sums) and all-gathers xarg (argmax candidates) between launches.
  int seg;            // -1: whole build in one launch (single GPU)
  int n_ranks;        // shards contributing to the exchange
  double* xarg;       // [Kmax][8] this shard's (score, x, y, z) for wmax and FPS argmax
  double* xarg_all;   // [n_ranks][Kmax][8] gathered
  double* xcal;       // [capacity][10] calibration leaf moments (exchanged)
};


// ----------------------------------------------------------------- helpers

// One tile's partial record in the field-major buffer (field f of tile t at
// partial[f * Tmax + t]): the tile pass writes its fields, the per-node
// reduction then reads each field over the node's consecutive tiles with
// coalesced loads (tile-major records made every load a separate sector:
// 4x the bytes, from DRAM once the buffer outgrows L2).  Concurrently
// processed tiles are adjacent, so the scattered 8-byte writes still
// complete whole sectors in L2.
struct TileRec {
  double* base;   // partial + t
  size_t stride;  // Tmax
  __device__ __forceinline__ double& operator[](int f) const { return base[(size_t)f * stride]; }
};

// The scoring fields of a component: w, log w, mean, precision, log_norm,
// 1/lam_min (positive iff the covariance is PD).
__device__ __forceinline__ void comp_to_regs(const GComp& c, double r[13]) {
  r[0] = c.w;
  r[1] = c.lw;
#pragma unroll
  for (int i = 0; i < 3; ++i) r[2 + i] = c.mean[i];
#pragma unroll
  for (int i = 0; i < 6; ++i) r[5 + i] = c.prec[i];
  r[11] = c.log_norm;
  r[12] = c.il[2];
}

// Deterministic block sum of NV values per thread; results in out[0..NV) (smem).
template <int NV>
__device__ __forceinline__ void block_sum_vec(double v[NV], double (*wsum)[NV], double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1)
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] += __shfl_xor_sync(0xffffffffu, v[k], off);
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < NV; ++k) wsum[warp][k] = v[k];
  __syncthreads();
  if (threadIdx.x < NV) {
    double s = wsum[0][threadIdx.x];
    for (int w = 1; w < kTile / 32; ++w) s += wsum[w][threadIdx.x];
    out[threadIdx.x] = s;
  }
  __syncthreads();
}

// (score, index) argmax: larger score, then lower index.
__device__ __forceinline__ void argmax_merge(double& s, double& i, double s2, double i2) {
  if (s2 > s || (s2 == s && i2 < i)) {
    s = s2;
    i = i2;
  }
}

__device__ __forceinline__ void block_argmax(double s, double i, double (*ws)[2], double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double s2 = __shfl_xor_sync(0xffffffffu, s, off);
    const double i2 = __shfl_xor_sync(0xffffffffu, i, off);
    argmax_merge(s, i, s2, i2);
  }
  if (lane == 0) {
    ws[warp][0] = s;
    ws[warp][1] = i;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double bs = ws[0][0], bi = ws[0][1];
    for (int w = 1; w < kTile / 32; ++w) argmax_merge(bs, bi, ws[w][0], ws[w][1]);
    out[0] = bs;
    out[1] = bi;
  }
  __syncthreads();
}

struct Phase {
  bool mom1, mom2, pcount, pwrite, layout;
  bool emit;    // pcount: the partition is written next (not in the last round)
  int fps;      // FPS round 1..7 (0 = none)
  int mode[2];  // per candidate: 0 none, 1 EM, 2 final
  int em_it[2];
};

__device__ __forceinline__ Phase phase_of(int p, int I, bool last_round) {
  Phase ph{};
  if (p == 0) ph.mom1 = true;
  if (p == 1) ph.mom2 = true;
  if (p >= 1 && p <= 7) ph.fps = p;
  if (p >= 2 && p <= I + 1) {
    ph.mode[0] = 1;
    ph.em_it[0] = p - 1;
  }
  if (p == I + 2) ph.mode[0] = 2;
  if (p >= 8 && p <= I + 7) {
    ph.mode[1] = 1;
    ph.em_it[1] = p - 7;
  }
  if (p == I + 8) ph.mode[1] = 2;
  if (p == I + 9) {
    ph.pcount = true;
    ph.emit = !last_round;  // the last round's children are leaves: counts only
  }
  if (p == I + 10) ph.layout = true;
  if (p == I + 11 && !last_round) ph.pwrite = true;
  return ph;
}

struct BuildSmem {
  union {
    struct {
      double wsum[kTile / 32][16];
      double ws2[kTile / 32][2];
      double red[16];
      double am[2];
    } s;
    struct {                 // tile_comp_pass (entry-per-thread E-step)
      double gam[16][kTile];  // responsibilities (w * gamma outside the partition), component-major
      double lt[2][kTile];    // w * log-likelihood per entry and candidate
      int best;               // heaviest survivor (partition fallback)
    } g;
    typename cub::BlockScan<unsigned long long, kTile>::TempStorage scan;
  } u;
  int nitems;
  int item_off[192];
  int item_kind[192];
  int tnode, tstart, tlen, tidx;
  int probe;  // TRG_TILE_PROBE: this CTA's tiles of the probed phase are marked
#ifdef TRG_TILE_PROBE
  long long pclk[10];
#endif
  alignas(16) double ent[4][kTile + 2];  // the tile's entries (x, y, z, w): one bulk copy per tile
  uint64_t mbar;                          // completion of the tile's bulk copies
  unsigned mphase;                        // its phase parity (thread 0's copy)
  double sred[kTile / 32][11][33];  // per-warp cross-lane sums of tile_comp_pass (padded rows)
  double nref[3], nmean[3], seed[3];
  alignas(16) GComp comp[2][8];
  int cand_list[2];
  int ncand;
  int surv[8];
  int ns, kept;
  double floorv;
  double drift;
};

// ----------------------------------------------------------------- tile work
#ifdef TRG_TILE_PROBE
#ifndef TRG_TILE_PROBE_ROUND
#define TRG_TILE_PROBE_ROUND 0
#endif
// raw SM clocks into shared memory (no atomics inside the tile), flushed
// after the tile as labels 8100 + i carrying cycles since mark 8001
#define TPROBE(lab) if (sm.probe && threadIdx.x == 0) sm.pclk[(lab) - 8000] = clock64()
#else
#define TPROBE(lab)
#endif
// Thread-per-entry passes: list_moments 1/2 and one FPS round.
__device__ void tile_entry_pass(const BuildParams& p, BuildSmem& sm, const Phase& ph, int par,
                                TileRec rec) {
  const int tid = threadIdx.x;
  const int e = sm.tstart + tid;
  const bool act = tid < sm.tlen;
  double x0 = 0, x1 = 0, x2 = 0, w = 0;
  if (act) {
    x0 = sm.ent[0][tid];
    x1 = sm.ent[1][tid];
    x2 = sm.ent[2][tid];
    w = sm.ent[3][tid];
  }
  if (ph.mom1) {
    double v[4] = {0, 0, 0, 0};
    if (act) {
      v[0] = w;
      v[1] = w * (x0 - sm.nref[0]);
      v[2] = w * (x1 - sm.nref[1]);
      v[3] = w * (x2 - sm.nref[2]);
    }
    block_sum_vec<4>(v, (double(*)[4])sm.u.s.wsum, sm.u.s.red);
    if (tid < 4) rec[kOffMom1 + tid] = sm.u.s.red[tid];
    __syncthreads();
    block_argmax(act ? w : -INFINITY, act ? (double)e : 1e300, sm.u.s.ws2, sm.u.s.am);
    if (tid == 0) {
      rec[kOffMom1 + 4] = sm.u.s.am[0];
      rec[kOffMom1 + 5] = sm.u.s.am[1];
    }
    __syncthreads();
  }
  if (ph.mom2) {
    double v[6] = {0, 0, 0, 0, 0, 0};
    if (act) {
      const double d0 = x0 - sm.nmean[0], d1 = x1 - sm.nmean[1], d2 = x2 - sm.nmean[2];
      v[0] = w * (d0 * d0);
      v[1] = w * (d0 * d1);
      v[2] = w * (d0 * d2);
      v[3] = w * (d1 * d1);
      v[4] = w * (d1 * d2);
      v[5] = w * (d2 * d2);
    }
    block_sum_vec<6>(v, (double(*)[6])sm.u.s.wsum, sm.u.s.red);
    if (tid < 6) rec[kOffMom2 + tid] = sm.u.s.red[tid];
    __syncthreads();
  }
  if (ph.fps) {
    double sc = -INFINITY;
    if (act) {
      const double a = x0 - sm.seed[0], b = x1 - sm.seed[1], c = x2 - sm.seed[2];
      double d2 = a * a;
      d2 += b * b;
      d2 += c * c;
      const double md = ph.fps == 1 ? d2 : smin(__ldcg(&p.min_d2[e]), d2);
      p.min_d2[e] = md;
      sc = w * md;
    }
    block_argmax(sc, act ? (double)e : 1e300, sm.u.s.ws2, sm.u.s.am);
    if (tid == 0) {
      rec[kOffFps] = sm.u.s.am[0];
      rec[kOffFps + 1] = sm.u.s.am[1];
    }
    __syncthreads();
  }
}

// E-step over one tile (e_step_moments gmm.cpp:159-206, final pass
// :331-358, partition :430-454), in two block-wide steps:
//  (1) entry per thread: the 8 (or 16, both candidates) component
//      log-densities are independent (ILP, no shuffles), max / sum / log run
//      in component order exactly like the reference, responsibilities go to
//      shared memory component-major;
//  (2) (candidate, component) per warp, entries over the lanes: the moments
//      (mode 1), masses (mode 2) or survivor-normalised partition (mode 3),
//      then a fixed butterfly over the lanes.
__device__ void tile_comp_pass(const BuildParams& p, BuildSmem& sm, const Phase& ph, int par,
                               TileRec rec, bool pcount) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nc = pcount ? 1 : sm.ncand;
  const int tlen = sm.tlen;
  auto& G = sm.u.g;
  // ---- (1a) component per warp, entries over the lanes: the component's
  // parameters stay in registers for the whole tile (one shared-memory read
  // per component instead of per entry); the log-densities go to the gam
  // rows, which (1b) then turns into responsibilities in place.
  for (int item = warp; item < nc * 8; item += kTile / 32) {
    const int ci = item >> 3, k = item & 7;
    const int cand = pcount ? sm.kept : sm.cand_list[ci];
    // gmm.cpp:176-178 log w + log_density (-inf when w == 0), without
    // branches: the value is selected, the domain error (log_density on a
    // non-PD covariance) flagged once per component
    double r[13];
    comp_to_regs(sm.comp[cand][k], r);
    const bool live = r[0] > 0.0, pd = r[12] > 0.0;
    if (lane == 0 && live && !pd && tlen > 0) atomicCAS(p.status, 0, kEDomain);
    if (item == 0) TPROBE(8005);
#pragma unroll 4
    for (int e = lane; e < tlen; e += 32) {
      const double v =
          r[1] + __fma_rn(-0.5, fast_q(r + 2, r + 5, sm.ent[0][e], sm.ent[1][e], sm.ent[2][e]), r[11]);
      G.gam[item][e] = (live && pd) ? v : -INFINITY;
    }
    if (item == 0) TPROBE(8006);
  }
  __syncthreads();
  TPROBE(8003);
  // ---- (1b) entry per thread: max / sum / log in component order exactly
  // like the reference
  if (tid < tlen) {
    const double w = sm.ent[3][tid];
    for (int ci = 0; ci < nc; ++ci) {
      const int cand = pcount ? sm.kept : sm.cand_list[ci];
      const int mode = pcount ? 3 : (cand == 0 ? ph.mode[0] : ph.mode[1]);  // (no local-memory index)
      double lg[8];
      double m = -INFINITY;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        lg[k] = G.gam[ci * 8 + k][tid];
        m = fmax(m, lg[k]);
      }
      const bool fin = isfinite(m);
      double ek[8], s = 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        ek[k] = fin ? trg_exp(lg[k] - m) : 0.0;  // == exp(), bit for bit
        s += ek[k];
      }
      // gamma_k = exp(log_k - log_total) = e_k / s (gmm.cpp:189, 354): one
      // reciprocal per entry instead of a second exp per component
      const double rs = fin ? rcp_sum(s) : 0.0;
      // the moment passes use the weighted responsibility w * gamma (stored
      // instead of gamma: one shared-memory load less per entry and
      // component in (2), the same rounded product); the partition uses gamma
      if (pcount) {
#pragma unroll
        for (int k = 0; k < 8; ++k) G.gam[ci * 8 + k][tid] = ek[k] * rs;
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) G.gam[ci * 8 + k][tid] = (ek[k] * rs) * w;
      }
      // the per-iteration log-likelihood only feeds the diagnostics trace
      // (gmm.cpp:240); the final pass (mode 2) always needs it (gmm.cpp:394)
      const bool want_ll = mode == 2 || (mode == 1 && p.want_traces);
      G.lt[ci][tid] = (fin && want_ll) ? w * (m + log(s)) : 0.0;
    }
  }
  if (pcount && tid == 0) {  // heaviest survivor: the partition's fallback
    int best = 0;
    for (int s2 = 1; s2 < sm.ns; ++s2)
      if (__ldcg(&p.nf.cmass[(size_t)sm.tnode * 16 + sm.kept * 8 + sm.surv[s2]]) >
          __ldcg(&p.nf.cmass[(size_t)sm.tnode * 16 + sm.kept * 8 + sm.surv[best]]))
        best = s2;
    G.best = best;
  }
  __syncthreads();
  TPROBE(8004);
  // ---- (2)
  if (!pcount) {
    for (int item = warp; item < nc * 8; item += kTile / 32) {
      const int ci = item >> 3, k = item & 7;
      const int cand = sm.cand_list[ci];
      const int mode = cand == 0 ? ph.mode[0] : ph.mode[1];
      const double n0 = sm.nmean[0], n1 = sm.nmean[1], n2 = sm.nmean[2];
      double a[11];
#pragma unroll
      for (int q = 0; q < 11; ++q) a[q] = 0.0;
      // Per lane the entries e = lane, lane + 32, ... in order (two per
      // iteration for ILP); uniform control flow (mode and k are per warp; a
      // zero responsibility adds exact zeros, so no per-entry test).
      if (mode == 1) {
        auto acc = [&](int e) {
          const double g = G.gam[item][e];  // w * gamma
          const double d0 = sm.ent[0][e] - n0, d1 = sm.ent[1][e] - n1, d2 = sm.ent[2][e] - n2;
          a[0] += g;
          a[1] += g * d0;
          a[2] += g * d1;
          a[3] += g * d2;
          a[4] += g * (d0 * d0);
          a[5] += g * (d0 * d1);
          a[6] += g * (d0 * d2);
          a[7] += g * (d1 * d1);
          a[8] += g * (d1 * d2);
          a[9] += g * (d2 * d2);
        };
        int e = lane;
        for (; e + 32 < tlen; e += 64) {
          acc(e);
          acc(e + 32);
        }
        if (e < tlen) acc(e);
        if (item == 0) TPROBE(8007);
      } else {
        for (int e = lane; e < tlen; e += 32) a[0] += G.gam[item][e];  // child mass w * gamma (gmm.cpp:355)
      }
      if (k == 0)
        for (int e = lane; e < tlen; e += 32) a[10] += G.lt[ci][e];
      // Cross-lane sums through shared memory: lane q adds value q of all
      // 32 lanes in the halving tree (16, 8, 4, 2, 1) - the very tree lane
      // 0 of an xor butterfly computes, so the sums are bit-identical to it,
      // at ~half the issue slots of 11 x 5 double shuffles.
      double(*sr)[33] = sm.sred[warp];
#pragma unroll
      for (int q = 0; q < 11; ++q) sr[q][lane] = a[q];
      __syncwarp();
      const bool need = mode == 1 ? (lane < 10 || (lane == 10 && k == 0))
                                  : (lane == 0 || (lane == 10 && k == 0));
      if (need) {
        double t[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) t[i] = sr[lane][i] + sr[lane][i + 16];
#pragma unroll
        for (int o = 8; o > 0; o >>= 1)
#pragma unroll
          for (int i = 0; i < o; ++i) t[i] += t[i + o];
        if (mode == 1)
          rec[kOffEm + cand * 81 + (lane < 10 ? k * 10 + lane : 80)] = t[0];
        else
          rec[kOffFin + cand * 9 + (lane == 0 ? 1 + k : 0)] = t[0];
      }
      __syncwarp();
    }
  } else {
    // survivor-normalised soft partition (gmm.cpp:434-454): warp = survivor
    if (tid < 16) rec[kOffCnt + tid] = 0.0;
    __syncthreads();
    const int ns = sm.ns;
    if (warp < ns) {
      const int sv = warp, comp = sm.surv[sv], best = G.best;
      double cnt = 0.0, mass = 0.0;
      for (int e = lane; e < tlen; e += 32) {
        const double w = sm.ent[3][e];
        double denom = 0.0;
        for (int s2 = 0; s2 < ns; ++s2) denom += G.gam[sm.surv[s2]][e];
        double out = 0.0;
        if (denom > 0.0) {
          const double g = G.gam[comp][e] / denom;
          if (!(g < 1e-12)) {
            out = w * g;
            cnt += 1.0;
            mass += out;
          }
        } else if (sv == best) {  // all on pruned children, or no finite density
          out = w;
          cnt += 1.0;
          mass += w;
        }
        if (ph.emit) p.emit[(size_t)(sm.tstart + e) * 8 + sv] = out;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        mass += __shfl_xor_sync(0xffffffffu, mass, o);
      }
      if (lane == 0) {
        rec[kOffCnt + comp] = cnt;
        rec[kOffCnt + 8 + comp] = mass;
      }
    }
  }
  __syncthreads();
}

// ----------------------------------------------------------------- node work
#ifdef TRG_RP_PROBE
#define UPROBE(lab) if (k == 0 && (threadIdx.x & 31) == 0) tl_mark_any(p.tl, lab)
#else
#define UPROBE(lab)
#endif
// M-steps of node k (m_step gmm.cpp:208-232), the whole warp: lane
// 8 c + j fits component j of candidate c (when candidate c ran an EM
// iteration this phase), all lanes of the warp in one pass of the
// closed-form eigensolver (eig3_cf).
__device__ void node_mstep_warp(const BuildParams& p, const Phase& ph, int k, const double* red) {
  const int lane = threadIdx.x & 31;
  const int c = (lane >> 3) & 1, comp = lane & 7;
  bool act = lane < 16 && ph.mode[c] == 1;
  GComp& g = p.nf.comps[((size_t)k * 2 + c) * 8 + comp];
  const double* ac = red + kOffEm + c * 81;
  // every operand in one round trip (the loads do not depend on the tests)
  double tv[8], a[10], mn[3], flv = 1.0;
#pragma unroll
  for (int j = 0; j < 8; ++j) tv[j] = lane < 16 ? __ldcg(ac + j * 10) : 0.0;
#pragma unroll
  for (int q = 0; q < 10; ++q) a[q] = lane < 16 ? __ldcg(ac + comp * 10 + q) : 0.0;
#pragma unroll
  for (int i = 0; i < 3; ++i) mn[i] = lane < 16 ? __ldcg(&p.nf.mean[3 * k + i]) : 0.0;
  if (lane < 16) flv = __ldcg(&p.nf.floorv[k]);
  double total = 0.0;
  if (act) {
    for (int j = 0; j < 8; ++j) total += tv[j];
    if (!(total > 0.0)) {
      atomicCAS(p.status, 0, kERuntime);  // m_step: no responsibility mass
      act = false;
    }
  }
  if (act) {
    if (a[0] <= total * 1e-12) {
      g.w = 0.0;
      act = false;
    }
  }
  double sc[3][3];
  double fl = 1.0;
  if (act) {
    const double m0 = a[0];
    const double d[3] = {a[1] / m0, a[2] / m0, a[3] / m0};
    const double m2[3][3] = {{a[4], a[5], a[6]}, {a[5], a[7], a[8]}, {a[6], a[8], a[9]}};
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) sc[i][j] = m2[i][j] / m0 - d[i] * d[j];
    g.w = m0 / total;
    g.lw = log(g.w);
    for (int i = 0; i < 3; ++i) g.mean[i] = mn[i] + d[i];
    fl = flv;
  } else {
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) sc[i][j] = i == j ? 1.0 : 0.0;
  }
  GComp r;
  UPROBE(7110);
#ifdef TRG_RP_PROBE
  const long long c0 = clock64();
#endif
  const int rc = comp_set_cov_cf(r, sc, fl);
#ifdef TRG_RP_PROBE
  const long long c1 = clock64();
  if (k == 0 && (threadIdx.x & 31) == 0) {
    const int i = atomicAdd(&p.tl->n, 1);
    if (i < 1024) { p.tl->lab[i] = 7199; p.tl->t[i] = (unsigned long long)(c1 - c0); }
  }
#endif
  UPROBE(7111);
  if (!act) return;
  if (rc) {
    atomicCAS(p.status, 0, kEInval);
    return;
  }
  for (int i = 0; i < 9; ++i) {
    g.axT[i] = r.axT[i];
    g.cov[i] = r.cov[i];
  }
  for (int i = 0; i < 3; ++i) {
    g.lam[i] = r.lam[i];
    g.il[i] = r.il[i];
  }
  for (int i = 0; i < 6; ++i) g.prec[i] = r.prec[i];
  g.log_norm = r.log_norm;
}

// Candidate init (fit_candidate gmm.cpp:319-326) for component `comp`.
__device__ void cand_init(const BuildParams& p, int k, int c, const double seed[3], int comp) {
  GComp& g = p.nf.comps[((size_t)k * 2 + c) * 8 + comp];
  g.w = 1.0 / 8.0;
  g.lw = log(g.w);
  for (int i = 0; i < 3; ++i) g.mean[i] = seed[i];
  double cs[3][3];
  const double* S = p.nf.scatter + 9 * k;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) cs[i][j] = S[3 * i + j] / 4.0;
  // the initial axes only feed densities (basis-independent), so the
  // closed-form solver serves; the corner seeds keep the Jacobi's basis
  if (comp_set_cov_cf(g, cs, p.nf.floorv[k])) atomicCAS(p.status, 0, kEInval);
}

// Winner of an argmax field (score, entry index) of node k: its score, and
// the entry's point in xyz.  Single GPU: straight from the reduced record.
// Sharded: every shard's candidate (score, x, y, z) was all-gathered into
// xarg_all; the highest score wins, ties to the lowest shard (shards hold
// contiguous blocks of the cloud, so this is the lowest global position,
// like the reference's first-maximum scan).
__device__ double argmax_point(const BuildParams& p, int par, int k, const double* red, int off,
                               int slot, double xyz[3]) {
  if (p.seg < 0) {
    const int e = (int)__ldcg(red + off + 1);
    xyz[0] = p.ex[par][e];
    xyz[1] = p.ey[par][e];
    xyz[2] = p.ez[par][e];
    return __ldcg(red + off);
  }
  double best = -INFINITY;
  int br = 0;
  for (int r = 0; r < p.n_ranks; ++r) {
    const double sc = __ldcg(p.xarg_all + ((size_t)r * p.Kmax + k) * 8 + 4 * slot);
    if (sc > best) {
      best = sc;
      br = r;
    }
  }
  const double* c = p.xarg_all + ((size_t)br * p.Kmax + k) * 8 + 4 * slot;
  for (int i = 0; i < 3; ++i) xyz[i] = __ldcg(c + 1 + i);
  return best;
}

// Node work after phase ph, done by ONE warp (the warp that reduced the
// node's last field); `red` is the node's reduced record (global, L2).
__device__ void node_update_warp(const BuildParams& p, const Phase& ph, int k, int par,
                                 const double* red, int round) {
  const int lane = threadIdx.x & 31;
  const NodeFit& nf = p.nf;
  UPROBE(7100);
  if (ph.mom1 && lane == 0) {
    const double mass = __ldcg(red + kOffMom1);
    nf.mass[k] = mass;
    if (!(mass > 0.0)) atomicCAS(p.status, 0, kEInval);  // list_moments: no mass
    // sharded: a shard without entries in node k never staged its shift
    // point, so every shard recomputes it (same value everywhere)
    for (int i = 0; i < 3; ++i) {
      double r = nf.ref[3 * k + i];
      if (p.seg >= 0) {
        const int id = p.rn[par].tree_id[k];
        r = id >= 0 ? p.nodes[id].mean[i] : 0.0;
      }
      nf.mean[3 * k + i] = r + __ldcg(red + kOffMom1 + 1 + i) / mass;
    }
    double xyz[3];
    argmax_point(p, par, k, red, kOffMom1 + 4, 0, xyz);
    for (int i = 0; i < 3; ++i) nf.seeds[24 * k + i] = xyz[i];
  }
  if (ph.mom2) {
    if (lane == 0) {
      const double mass = __ldcg(&nf.mass[k]);
      double m[6];
      for (int q = 0; q < 6; ++q) m[q] = __ldcg(red + kOffMom2 + q);
      const double M[3][3] = {{m[0], m[1], m[2]}, {m[1], m[3], m[4]}, {m[2], m[4], m[5]}};
      double S[3][3];
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
          S[i][j] = M[i][j] / mass;
          nf.scatter[9 * k + 3 * i + j] = S[i][j];
        }
      nf.floorv[k] = cov_floor(S, p.eps, p.abs_floor);
    }
    __syncwarp();
    // corner seeds (gmm.cpp:248-261): lane c computes seed c
    if (lane < 8) {
      double S[3][3], lam[3], ax[3][3];
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) S[i][j] = nf.scatter[9 * k + 3 * i + j];
      if (eig_sym3_floored(S, nf.floorv[k], lam, ax)) atomicCAS(p.status, 0, kEInval);
      double off[3] = {0.0, 0.0, 0.0};
      for (int l = 0; l < 3; ++l) {
        const double sign = ((lane >> l) & 1) != 0 ? 1.0 : -1.0;
        const double sc = sign * 0.5 * sqrt(lam[l]);
        for (int i = 0; i < 3; ++i) off[i] = off[i] + sc * ax[i][l];
      }
      double seed[3];
      for (int i = 0; i < 3; ++i) seed[i] = nf.mean[3 * k + i] + off[i];
      cand_init(p, k, 0, seed, lane);
    }
    __syncwarp();
  }
  if (ph.fps && lane == 0) {
    double xyz[3];
    const double bs = argmax_point(p, par, k, red, kOffFps, 1, xyz);
    double* sd = nf.seeds + 24 * k;
    if (!(bs > 0.0)) {  // degenerate support: duplicate seed 0 (gmm.cpp:291-294)
      for (int i = 0; i < 3; ++i) sd[3 * ph.fps + i] = sd[i];
    } else {
      for (int i = 0; i < 3; ++i) sd[3 * ph.fps + i] = xyz[i];
    }
  }
  __syncwarp();
  if (ph.fps == 7 && lane < 8) {
    double seed[3];
    for (int i = 0; i < 3; ++i) seed[i] = nf.seeds[24 * k + 3 * lane + i];
    cand_init(p, k, 1, seed, lane);
  }
  // ll traces (BuildDiagnostics::node_ll_traces, gmm.cpp:240, 361)
  if (p.want_traces && lane < 2 && ph.mode[lane] != 0) {
    const int c = lane, I = p.em_iters;
    const int slot = ph.mode[c] == 1 ? ph.em_it[c] - 1 : I;
    const double ll = ph.mode[c] == 1 ? __ldcg(red + kOffEm + 81 * c + 80) : __ldcg(red + kOffFin + 9 * c);
    p.ll_trace[((size_t)(p.st->exp_base + k) * 2 + c) * (I + 1) + slot] = ll;
  }
  // M-steps: lanes 0-7 candidate 0, lanes 8-15 candidate 1
  __syncwarp();
  UPROBE(7101);
  if (ph.mode[0] == 1 || ph.mode[1] == 1) node_mstep_warp(p, ph, k, red);
  __syncwarp();
  UPROBE(7102);
  if (lane < 2 && ph.mode[lane] == 2) {
    const int c = lane;
    nf.final_ll[2 * k + c] = __ldcg(red + kOffFin + 9 * c);
    for (int j = 0; j < 8; ++j) nf.cmass[16 * k + 8 * c + j] = __ldcg(red + kOffFin + 9 * c + 1 + j);
  }
  __syncwarp();
  if (ph.mode[1] == 2 && lane == 0) {
    // candidate choice (gmm.cpp:394) and survivors (gmm.cpp:414-428)
    const int kept = (__ldcg(&nf.final_ll[2 * k + 1]) > __ldcg(&nf.final_ll[2 * k + 0])) ? 1 : 0;
    nf.kept[k] = kept;
    p.kept_exp[p.st->exp_base + k] = kept;
    const double* cm = nf.cmass + 16 * k + 8 * kept;
    const double thr = smax(4.0, __ldcg(&nf.mass[k]) * 1e-6);
    int ns = 0;
    for (int j = 0; j < 8; ++j)
      if (__ldcg(&cm[j]) > thr) nf.surv[8 * k + ns++] = j;
    int ok = 1;
    if (ns == 0) {
      if (round != 0) {
        ok = 0;
      } else {
        int best = 0;
        for (int j = 1; j < 8; ++j)
          if (__ldcg(&cm[j]) > __ldcg(&cm[best])) best = j;
        nf.surv[8 * k + ns++] = best;
      }
    }
    nf.ns[k] = ok ? ns : 0;
    nf.ok[k] = ok;
  }
  if (ph.pcount) {
    // per-child totals + per-tile child base offsets (stable order); lane s
    const int ns = nf.ns[k];
    // (tile_base / next_seg: the kind-2 reduction items; layout turns the
    // child entry counts into segments)
    if (lane < ns) {
      const int s = lane;
      const int comp = nf.surv[8 * k + s];
      nf.smass[8 * k + s] = __ldcg(red + kOffCnt + 8 + comp);
    }
    __syncwarp();
    if (lane == 0) {
      double total = 0.0;
      for (int s = 0; s < ns; ++s) total += nf.smass[8 * k + s];
      nf.stotal[k] = total;
    }
  }
  __syncwarp();
}

// Node-level context of the tile about to be processed (smem).
__device__ void load_tile_ctx(const BuildParams& p, BuildSmem& sm, const Phase& ph, int par,
                              int t) {
  const int tid = threadIdx.x;
  // every thread reads the tile's (node, start, len) (broadcast loads)
  const int k = __ldcg(&p.tile_node[par][t]);
  const int tstart = __ldcg(&p.tile_start[par][t]);
  const int tlen = __ldcg(&p.tile_len[par][t]);
  const bool need_comps = ph.mode[0] || ph.mode[1] || ph.pcount;
  // The tile's entries (x, y, z, w) and the node's 2 x 8 component table go
  // to shared memory as bulk copies (TMA engine, cp.async.bulk) completing on
  // the CTA's mbarrier: one thread issues them and the block's threads fetch
  // the node context meanwhile.  Segments start at even entries (the layout
  // pads them) so every copy is 16-byte aligned; the odd tail element copied
  // past a tile is never read.
  if (tid == 0) {
    sm.tidx = t;
    sm.tnode = k;
    sm.tstart = tstart;
    sm.tlen = tlen;
    const unsigned eb = (!ph.pwrite) ? (unsigned)((tlen + 1) & ~1) * 8u : 0u;
    const unsigned cb = need_comps ? 16u * (unsigned)sizeof(GComp) : 0u;
    if (eb + cb) {
      fence_proxy_async_shared();  // the previous tile's generic reads come first
      fence_proxy_async_global();  // other CTAs' writes (ordered by a grid barrier)
      mbar_arrive_tx(&sm.mbar, 4u * eb + cb);
      if (eb) {
        bulk_g2s(sm.ent[0], p.ex[par] + tstart, eb, &sm.mbar);
        bulk_g2s(sm.ent[1], p.ey[par] + tstart, eb, &sm.mbar);
        bulk_g2s(sm.ent[2], p.ez[par] + tstart, eb, &sm.mbar);
        bulk_g2s(sm.ent[3], p.ew[par] + tstart, eb, &sm.mbar);
      }
      if (cb) bulk_g2s(&sm.comp[0][0], p.nf.comps + (size_t)k * 16, cb, &sm.mbar);
    }
  }
  if (tid < 3) {
    if (ph.mom1) {
      // list_moments' shift point: the node's first entry (gmm.cpp); sharded,
      // a point every shard knows: the node's fitted mean (0 for the root)
      double v;
      if (p.seg < 0) {
        const int e0 = __ldcg(&p.rn[par].seg[k]);
        v = __ldcg(tid == 0 ? &p.ex[par][e0] : (tid == 1 ? &p.ey[par][e0] : &p.ez[par][e0]));
      } else {
        const int id = __ldcg(&p.rn[par].tree_id[k]);
        v = id >= 0 ? __ldcg(&p.nodes[id].mean[tid]) : 0.0;
      }
      sm.nref[tid] = v;
      p.nf.ref[3 * k + tid] = v;
    }
    sm.nmean[tid] = __ldcg(&p.nf.mean[3 * k + tid]);
    if (ph.fps) sm.seed[tid] = __ldcg(&p.nf.seeds[24 * k + 3 * (ph.fps - 1) + tid]);
  }
  if (tid == 32) {
    int nc = 0;
    for (int c = 0; c < 2; ++c)
      if (ph.mode[c]) sm.cand_list[nc++] = c;
    sm.ncand = nc;
    if (ph.pcount) {
      sm.kept = __ldcg(&p.nf.kept[k]);
      sm.ns = __ldcg(&p.nf.ns[k]);
      for (int s = 0; s < sm.ns; ++s) sm.surv[s] = __ldcg(&p.nf.surv[8 * k + s]);
    }
  }
  // one thread waits on the copies (the others block at the CTA barrier
  // instead of spinning: spinning warps took issue slots from the SM's
  // other CTAs, 5 % of all k_build instructions)
  if (tid == 0 && (!ph.pwrite || need_comps)) mbar_wait(&sm.mbar, sm.mphase);
  __syncthreads();
  if (tid == 0 && (!ph.pwrite || need_comps)) sm.mphase ^= 1u;
}

// Partition write (gmm.cpp:441-442): stable compaction of one tile into the
// next round's node-sorted entry buffer.
__device__ void tile_pwrite(const BuildParams& p, BuildSmem& sm, int par, int t) {
  const int tid = threadIdx.x;
  const int k = sm.tnode;
  const int ns = p.nf.ns[k];
  const bool act = tid < sm.tlen;
  const int e = sm.tstart + tid;
  double em[8];
  unsigned long long f0 = 0, f1 = 0;
  for (int s = 0; s < 8; ++s) {
    em[s] = (act && s < ns) ? p.emit[(size_t)e * 8 + s] : 0.0;
    const unsigned long long bit = em[s] > 0.0 ? 1ull : 0ull;
    if (s < 4) f0 |= bit << (16 * s);
    else f1 |= bit << (16 * (s - 4));
  }
  using Scan = cub::BlockScan<unsigned long long, kTile>;
  unsigned long long r0, r1;
  Scan(sm.u.scan).ExclusiveSum(f0, r0);
  __syncthreads();
  Scan(sm.u.scan).ExclusiveSum(f1, r1);
  __syncthreads();
  if (!act) return;
  const int npar = par ^ 1;
  for (int s = 0; s < ns; ++s) {
    if (!(em[s] > 0.0)) continue;
    const int cs = p.nf.next_seg[8 * k + s];
    if (cs < 0) continue;
    const unsigned long long rr = s < 4 ? r0 : r1;
    const int rank = (int)((rr >> (16 * (s & 3))) & 0xffffull);
    const int pos = cs + (int)p.tile_base[(size_t)t * 8 + s] + rank;
    p.ex[npar][pos] = p.ex[par][e];
    p.ey[npar][pos] = p.ey[par][e];
    p.ez[npar][pos] = p.ez[par][e];
    p.ew[npar][pos] = em[s];
  }
}

// Block-wide exclusive scan of n ints in place (one CTA, any n); returns
// the total.  Chunked per thread, then a warp/smem scan of chunk totals.
__device__ int block_exscan(int* a, int n, int* wtmp /* >= 33 ints smem */) {
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int per = (n + nt - 1) / nt;
  const int b = min(n, tid * per), e = min(n, b + per);
  int sum = 0;
  for (int i = b; i < e; ++i) sum += a[i];
  int x = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wtmp[warp] = x;
  __syncthreads();
  if (tid == 0) {
    int run = 0;
    for (int w = 0; w < nt / 32; ++w) {
      const int v = wtmp[w];
      wtmp[w] = run;
      run += v;
    }
    wtmp[32] = run;
  }
  __syncthreads();
  int run = wtmp[warp] + x - sum;
  for (int i = b; i < e; ++i) {
    const int v = a[i];
    a[i] = run;
    run += v;
  }
  const int total = wtmp[32];
  __syncthreads();
  return total;
}

// Last index i in [0, n) with a[i] <= v (a non-decreasing, a[0] <= v).
__device__ __forceinline__ int upper_index(const int* a, int n, int v) {
  int lo = 0, hi = n;  // a[lo] <= v < a[hi] (a[n] = +inf)
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] <= v) lo = mid; else hi = mid;
  }
  return lo;
}

// Layout (CTA 0, all threads): create this round's child tree nodes, choose
// the next round's expanding set (mass gate gmm.cpp:621-623), its entry
// segments and tiles.  Children are numbered node by node, survivor by
// survivor, exactly like build_tree's push_back order (gmm.cpp:629-641).
// Work is spread per child and per tile (a child finds its node, a tile its
// child, by binary search in the exclusive scans); the scratch arrays live
// in the idle tile scratch when they fit, else in global memory.
__device__ void round_layout(const BuildParams& p, BuildSmem& sm, int par, int round,
                             int* gscratch) {
  BuildState* st = p.st;
  const int tid = threadIdx.x, nt = blockDim.x;
  __shared__ int wtmp[33];
  __shared__ int sOvf;
  const int K = st->Kp[par];
  const int J0 = st->J;
  const int npar = par ^ 1;
  const bool last = round + 1 >= p.L;
  int* scratch = (size_t)(K + 6 * 8 * K) * sizeof(int) <= sizeof(sm.u)
                     ? reinterpret_cast<int*>(&sm.u) : gscratch;
  int* nbase = scratch;           // [K] child-id base per expanding node
  int* cgate = scratch + K;       // [NC] gated flag -> K2 position
  int* ngate = cgate + 8 * K;     // [NC] gated flag (kept)
  int* ccnt = ngate + 8 * K;      // [NC] padded entry count -> E2 offset
  int* ctil = ccnt + 8 * K;       // [NC] tile count -> T2 offset
  int* clen = ctil + 8 * K;       // [NC] entry count
  int* codd = clen + 8 * K;       // [NC] 1 when the child's entry count is odd
  for (int k = tid; k < K; k += nt) nbase[k] = p.nf.ok[k] ? p.nf.ns[k] : 0;
  __syncthreads();
  const int NC = block_exscan(nbase, K, wtmp);
  if (tid == 0) {
    sOvf = (J0 + NC > p.capacity) ? 1 : 0;
  }
  __syncthreads();
  if (sOvf) {
    if (tid == 0) atomicCAS(p.status, 0, kERuntime);
    return;
  }
  // (2) one child per thread: create the tree node, link the parent; the
  // child's gate / entry count / tiles
  for (int c = tid; c < NC; c += nt) {
    const int k = upper_index(nbase, K, c), s2 = c - nbase[k];
    const int ns = p.nf.ns[k];
    const int parent = p.rn[par].tree_id[k];
    const int id0 = J0 + nbase[k];
    if (s2 == 0 && parent >= 0) {
      p.nodes[parent].first_child = id0;
      p.nodes[parent].child_count = ns;
    }
    const int kept = p.nf.kept[k];
    const GComp& g = p.nf.comps[((size_t)k * 2 + kept) * 8 + p.nf.surv[8 * k + s2]];
    const double sm_c = p.nf.smass[8 * k + s2];
    const double w = sm_c / p.nf.stotal[k];
    write_dnode_from_comp(p.nodes[id0 + s2], p.cov + 9 * (size_t)(id0 + s2), g, w, round, parent);
    const int cnt = p.nf.next_seg[8 * k + s2];  // child entry count (from pcount)
    const bool gate = !last && !(sm_c < p.min_points);
    cgate[c] = gate ? 1 : 0;
    ngate[c] = gate ? 1 : 0;
    ccnt[c] = gate ? (cnt + 1) & ~1 : 0;  // segments start at even entries (16-byte bulk copies)
    codd[c] = gate ? cnt & 1 : 0;
    ctil[c] = gate ? (cnt + kTile - 1) / kTile : 0;
    clen[c] = gate ? cnt : 0;
  }
  __syncthreads();
  // (3) next round's expanding list: positions, entry offsets, tile offsets
  const int K2 = block_exscan(cgate, NC, wtmp);
  const int E2 = block_exscan(ccnt, NC, wtmp);
  const int T2 = block_exscan(ctil, NC, wtmp);
  const int pad2 = block_exscan(codd, NC, wtmp);  // E2 - pad2 = the entries (E_l)
  if (tid == 0) {
    sOvf = (!last && (K2 > p.Kmax || E2 > p.Emax || T2 > p.Tmax)) ? 1 : 0;
  }
  __syncthreads();
  if (sOvf) {
    if (tid == 0) {
      st->status_overflow = 1;
      st->need_K = K2;
      st->need_E = E2;
      st->need_T = T2;
      st->done = 1;
      __threadfence();
    }
    return;
  }
  for (int c = tid; c < NC; c += nt) {
    const int k = upper_index(nbase, K, c), s2 = c - nbase[k];
    if (!ngate[c]) {
      p.nf.next_seg[8 * k + s2] = -1;
      continue;
    }
    const int k2 = cgate[c], e2 = ccnt[c], cnt = clen[c];
    p.rn[npar].tree_id[k2] = J0 + c;
    p.rn[npar].seg[k2] = e2;
    p.rn[npar].len[k2] = cnt;
    p.rn[npar].tile0[k2] = ctil[c];
    p.rn[npar].ntiles[k2] = (cnt + kTile - 1) / kTile;
    p.nf.next_seg[8 * k + s2] = e2;
  }
  // (4) the next round's tiles, one per thread: its child by binary search
  // over the tile offsets (ungated children own no tiles)
  for (int t = tid; t < T2; t += nt) {
    const int c = upper_index(ctil, NC, t), q = t - ctil[c];
    p.tile_node[npar][t] = cgate[c];
    p.tile_start[npar][t] = ccnt[c] + q * kTile;
    p.tile_len[npar][t] = min(kTile, clen[c] - q * kTile);
  }
  __syncthreads();
  if (tid == 0) {
    st->exp_base += K;
    st->n_exp = st->exp_base;
    st->J = J0 + NC;
    if (round == 0) st->root_count = NC;
    if (round < 8) st->lvl_start[round] = J0;
    st->lvl_start[round + 1] = J0 + NC;
    st->round = round + 1;
    st->Kp[npar] = K2;
    st->Ep[npar] = E2;
    st->Tp[npar] = T2;
    if (round + 1 < 8) {
      st->E_round[round + 1] = (unsigned long long)(E2 - pad2);
      st->K_round[round + 1] = K2;
    }
    if (last || K2 == 0) {
      st->done = 1;
      for (int l = round + 1; l < 9; ++l) st->lvl_start[l] = J0 + NC;
    }
    __threadfence();
  }
  __syncthreads();
}

// reset_parents_to_child_moments (gmm.cpp:489-513), one CTA: levels bottom
// up, the parents of a level in parallel (each parent's sums run over its
// children in order, as in the reference).
__device__ void reset_parents(const BuildParams& p, const int* lvl_start) {
  for (int l = p.L - 2; l >= 0; --l) {
    for (int i = lvl_start[l] + threadIdx.x; i < lvl_start[l + 1]; i += blockDim.x) {
      DNode& nd = p.nodes[i];
      if (nd.child_count == 0) continue;
      double w = 0.0, mu[3] = {0.0, 0.0, 0.0};
      for (int c = 0; c < nd.child_count; ++c) {
        const DNode& ch = p.nodes[nd.first_child + c];
        w += ch.weight;
        for (int k = 0; k < 3; ++k) mu[k] = mu[k] + ch.weight * ch.mean[k];
      }
      if (!(w > 0.0)) continue;
      for (int k = 0; k < 3; ++k) mu[k] = mu[k] / w;
      double cov[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
      for (int c = 0; c < nd.child_count; ++c) {
        const int ci = nd.first_child + c;
        const DNode& ch = p.nodes[ci];
        const double d[3] = {ch.mean[0] - mu[0], ch.mean[1] - mu[1], ch.mean[2] - mu[2]};
        for (int r = 0; r < 3; ++r)
          for (int s = 0; s < 3; ++s)
            cov[3 * r + s] = cov[3 * r + s] + ch.weight * (p.cov[9 * (size_t)ci + 3 * r + s] + d[r] * d[s]);
      }
      for (int k = 0; k < 9; ++k) p.cov[9 * (size_t)i + k] = cov[k] / w;
      for (int k = 0; k < 3; ++k) nd.mean[k] = mu[k];
    }
    __syncthreads();
  }
}

// ----------------------------------------------------------------- kernel
// Field items reduced per node after a phase: (offset, kind 0 = sum,
// kind 1 = (score, index) argmax pair).
__device__ int phase_items(const Phase& ph, int* off, int* kind) {
  int n = 0;
  auto sum_range = [&](int o, int c) {
    for (int i = 0; i < c; ++i) {
      off[n] = o + i;
      kind[n++] = 0;
    }
  };
  if (ph.mom1) {
    sum_range(kOffMom1, 4);
    off[n] = kOffMom1 + 4;
    kind[n++] = 1;
  }
  if (ph.mom2) sum_range(kOffMom2, 6);
  if (ph.fps) {
    off[n] = kOffFps;
    kind[n++] = 1;
  }
  for (int c = 0; c < 2; ++c) {
    if (ph.mode[c] == 1) sum_range(kOffEm + 81 * c, 81);
    if (ph.mode[c] == 2) sum_range(kOffFin + 9 * c, 9);
  }
  if (ph.pcount) {
    sum_range(kOffCnt + 8, 8);
    for (int q = 0; q < (ph.emit ? 8 : 0); ++q) {  // per-survivor tile prefix (child base offsets)
      off[n] = q;
      kind[n++] = 2;
    }
  }
  return n;
}

// Sum (or argmax-merge) field item `f` of node k over its tiles, one warp;
// lane-strided then butterfly: fixed order, deterministic.
__device__ __forceinline__ void reduce_item(const BuildParams& p, int par, int k, int off,
                                            int kind) {
  // (the record loads are issued in batches of 8 ahead of their uses: the
  // cache-global loads are ordered volatile asm, so a load-then-add loop
  // would wait a full L2 round trip per tile; the sums keep their order)
  constexpr int B = 16;
  const int lane = threadIdx.x & 31;
  const int t0 = p.rn[par].tile0[k], nt = p.rn[par].ntiles[k];
  double* out = p.nodered + (size_t)k * kRec;
  const double* rec0 = p.partial + t0;  // field f of tile t0 + q: rec0[f * Tmax + q]
  const size_t TS = (size_t)p.Tmax;
  if (kind == 0) {
    double v = 0.0;
    for (int q0 = lane; q0 < nt; q0 += 32 * B) {
      double b[B];
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const int q = q0 + 32 * u;
        b[u] = q < nt ? __ldcg(rec0 + (size_t)off * TS + q) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < B; ++u)
        if (q0 + 32 * u < nt) v += b[u];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) out[off] = v;
  } else if (kind == 2) {
    // survivor `off`'s per-tile child base offsets: exclusive prefix over the
    // node's tiles of its integer entry counts (exact in any order), lanes
    // own contiguous tile runs
    const int s = off, ns = __ldcg(&p.nf.ns[k]);
    if (s >= ns) return;
    const int comp = __ldcg(&p.nf.surv[8 * k + s]);
    const double* cnt = rec0 + (size_t)(kOffCnt + comp) * TS;
    const int per = (nt + 31) / 32;
    const int q0 = min(nt, lane * per), q1 = min(nt, q0 + per);
    double loc = 0.0;
    for (int qb = q0; qb < q1; qb += B) {
      double b[B];
#pragma unroll
      for (int u = 0; u < B; ++u) b[u] = qb + u < q1 ? __ldcg(cnt + qb + u) : 0.0;
#pragma unroll
      for (int u = 0; u < B; ++u) loc += b[u];
    }
    double inc = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    double base = inc - loc;
    for (int qb = q0; qb < q1; qb += B) {
      double b[B];
#pragma unroll
      for (int u = 0; u < B; ++u) b[u] = qb + u < q1 ? __ldcg(cnt + qb + u) : 0.0;
#pragma unroll
      for (int u = 0; u < B; ++u) {
        if (qb + u < q1) p.tile_base[(size_t)(t0 + qb + u) * 8 + s] = base;
        base += b[u];
      }
    }
    if (lane == 31) p.nf.next_seg[8 * k + s] = (int)inc;  // child entry count
  } else {
    double bs = -INFINITY, bi = 1e300;
    for (int q0 = lane; q0 < nt; q0 += 32 * B) {
      double sc[B], ix[B];
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const int q = q0 + 32 * u;
        sc[u] = q < nt ? __ldcg(rec0 + (size_t)off * TS + q) : -INFINITY;
        ix[u] = q < nt ? __ldcg(rec0 + (size_t)(off + 1) * TS + q) : 1e300;
      }
#pragma unroll
      for (int u = 0; u < B; ++u) argmax_merge(bs, bi, sc[u], ix[u]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double s2 = __shfl_xor_sync(0xffffffffu, bs, o);
      const double i2 = __shfl_xor_sync(0xffffffffu, bi, o);
      argmax_merge(bs, bi, s2, i2);
    }
    if (lane == 0) {
      out[off] = bs;
      out[off + 1] = bi;
    }
  }
}


// Writes this shard's argmax candidates of the phase (score + the entry's
// point) for the all-gather (sharded mode).
__device__ void write_xarg(const BuildParams& p, const Phase& ph, int par, int K, int G, int cta) {
  const int gt = cta * blockDim.x + threadIdx.x, nt = G * blockDim.x;
  for (int k = gt; k < K; k += nt) {
    const double* red = p.nodered + (size_t)k * kRec;
    double* o = p.xarg + (size_t)k * 8;
    for (int slot = 0; slot < 2; ++slot) {
      const bool on = slot == 0 ? ph.mom1 : ph.fps != 0;
      if (!on) continue;
      const int off = slot == 0 ? kOffMom1 + 4 : kOffFps;
      const double sc = __ldcg(red + off), ix = __ldcg(red + off + 1);
      const bool valid = sc > -INFINITY && ix < 1e299;
      const int e = valid ? (int)ix : 0;
      o[4 * slot] = valid ? sc : -INFINITY;
      o[4 * slot + 1] = valid ? p.ex[par][e] : 0.0;
      o[4 * slot + 2] = valid ? p.ey[par][e] : 0.0;
      o[4 * slot + 3] = valid ? p.ez[par][e] : 0.0;
    }
  }
}

#ifndef TRG_KBUILD_MINB
#define TRG_KBUILD_MINB 3
#endif
// The build of one cloud on a group of G CTAs (this CTA: `cta` of them);
// every barrier and work split is over the group.  k_build runs it on the
// whole grid, k_build on one group per cloud.
__device__ __forceinline__ void build_run(const BuildParams& p, int G, int cta) {
  extern __shared__ __align__(16) unsigned char k_build_smem[];  // BuildSmem (> 48 KB static)
  BuildSmem& sm = *reinterpret_cast<BuildSmem*>(k_build_smem);
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  BuildState* st = p.st;
  const bool sharded = p.seg >= 0;
  if (sharded && (__ldcg(&st->done) || __ldcg(&st->status_overflow))) return;
  if (tid == 0) {
    mbar_init(&sm.mbar, 1);
    mbar_fence_init();
    sm.mphase = 0u;
  }
  __syncthreads();
  tl_mark(p.tl, -1);
  // Sharded segments: exchange point xp = the per-node reduction of a phase.
  // Segment q finishes exchange point q-1 (node updates from the all-reduced
  // record) and runs up to and including the reduction of exchange point q.
  int xp = 0;
  // ------------------------------------------------ expansion rounds
  for (int round = 0; round < p.L; ++round) {
    const int par = round & 1;
    const bool last_round = round + 1 >= p.L;
    const int nphase = p.em_iters + 12;
    for (int ph_i = 0; ph_i < nphase; ++ph_i) {
      const Phase ph = phase_of(ph_i, p.em_iters, last_round);
      if (!(ph.mom1 || ph.mom2 || ph.fps || ph.mode[0] || ph.mode[1] || ph.pcount || ph.layout ||
            ph.pwrite))
        continue;
      const bool mine = !sharded || xp == p.seg;  // this launch runs the phase's work
      if (ph.layout) {
        if (mine) {
          if (cta == 0) round_layout(p, sm, par, round, p.layout_scratch);
          grid_sync(p.bar, G);
          tl_mark(p.tl, round * 100 + ph_i);
        }
        continue;
      }
      if (ph.pwrite) {
        if (mine) {
          const int T = __ldcg(&st->Tp[par]);
          for (int t = cta; t < T; t += G) {
            load_tile_ctx(p, sm, ph, par, t);
            tile_pwrite(p, sm, par, t);
            __syncthreads();
          }
          grid_sync(p.bar, G);
          tl_mark(p.tl, round * 100 + ph_i);
        }
        continue;
      }
      if (mine) {
        // (a) tile pass (the phase's reduction items are listed first, off the
        // critical path: the lists live outside the tile scratch)
        if (tid == 0) sm.nitems = phase_items(ph, sm.item_off, sm.item_kind);
#ifdef TRG_TILE_PROBE
        if (tid == 0) sm.probe = cta == 0 && ph_i == TRG_TILE_PROBE && round == TRG_TILE_PROBE_ROUND;
        TPROBE(8000);
#endif
        const int T = __ldcg(&st->Tp[par]);
        int ntl = 0, nent = 0;
        for (int t = cta; t < T; t += G) {
          TPROBE(8001);
          load_tile_ctx(p, sm, ph, par, t);
          TPROBE(8002);
          const TileRec rec{p.partial + t, (size_t)p.Tmax};
          tile_entry_pass(p, sm, ph, par, rec);
          if (ph.mode[0] || ph.mode[1]) tile_comp_pass(p, sm, ph, par, rec, false);
          if (ph.pcount) tile_comp_pass(p, sm, ph, par, rec, true);
          ++ntl;
          nent += sm.tlen;
          __syncthreads();
          TPROBE(8009);
#ifdef TRG_TILE_PROBE
          if (sm.probe && tid == 0)
            for (int q = 0; q < 10; ++q)
              if (q != 0) {
                const int i = atomicAdd(&p.tl->n, 1);
                if (i < 1024) {
                  p.tl->lab[i] = 8100 + q;
                  p.tl->t[i] = (unsigned long long)(sm.pclk[q] - sm.pclk[1]);
                }
              }
#endif
        }
        grid_sync(p.bar, G);
        tl_mark(p.tl, round * 100 + ph_i);
        // (b) per-node reduction of the tile records (+ node update when the
        // whole cloud is here)
        const int NI = sm.nitems;
        const int K = __ldcg(&st->Kp[par]);
        // F consecutive fields per warp item, F chosen so that every warp has
        // at most one item: a warp that completes a node runs its update
        // (~5 us), and a second item queued behind it would delay that other
        // node's update in turn
        const int nw = G * (kTile / 32);
        const int F = max(1, (K * NI + nw - 1) / nw), IPN = (NI + F - 1) / F;
        for (int it = cta * (kTile / 32) + warp; it < K * IPN; it += nw) {
          const int k = it / IPN, f0 = (it % IPN) * F, f1 = min(f0 + F, NI);
          for (int f = f0; f < f1; ++f) reduce_item(p, par, k, sm.item_off[f], sm.item_kind[f]);
          if (sharded) continue;
          unsigned last = 0;
          if (lane == 0) {
            // release this item's sums, acquire the node's other items
            last = (atom_add_acq_rel(&p.fdone[k], 1u) == (unsigned)IPN - 1) ? 1u : 0u;
            if (last) p.fdone[k] = 0u;  // (ordered before the next phase by the grid barrier)
          }
          last = __shfl_sync(0xffffffffu, last, 0);
#ifdef TRG_RP_PROBE
          const bool probe = ph_i == TRG_RP_PROBE && k == 0 && lane == 0;
          if (probe) tl_mark_any(p.tl, 7000 + round * 10);
#endif
          if (last) {
#ifdef TRG_RP_PROBE
            if (probe) tl_mark_any(p.tl, 7001 + round * 10);
#endif
            node_update_warp(p, ph, k, par, p.nodered + (size_t)k * kRec, round);
#ifdef TRG_RP_PROBE
            if (probe) tl_mark_any(p.tl, 7002 + round * 10);
#endif
          }
        }
        if (sharded) {
          grid_sync(p.bar, G);
          if (ph.mom1 || ph.fps) write_xarg(p, ph, par, K, G, cta);
          return;  // exchange point: the host all-reduces nodered / gathers xarg
        }
        grid_sync(p.bar, G);
        tl_mark(p.tl, round * 100 + 50 + ph_i);
      } else if (xp == p.seg - 1) {
        // node updates of the previous segment's exchange point, from the
        // all-reduced records (every shard computes the same)
        const int K = __ldcg(&st->Kp[par]);
        for (int k = cta * (kTile / 32) + warp; k < K; k += G * (kTile / 32))
          node_update_warp(p, ph, k, par, p.nodered + (size_t)k * kRec, round);
        grid_sync(p.bar, G);
      }
      ++xp;
    }
    if (__ldcg(&st->done) || __ldcg(&st->status_overflow)) break;
  }
}

// Clouds per launch: k_build / k_calibrate take a batch of independent
// clouds, cloud i on CTAs [i * group, (i + 1) * group), its parameters in
// the launch's parameter space (dynamically indexed constant bank, no local
// copy).  A single build is a batch of one on the whole grid.  One kernel
// per body on purpose: with -fmad=true ptxas contracts FP64 mul/add pairs
// per compiled kernel, so two copies of the same body could round
// differently, and batched and single registrations must agree bitwise.
constexpr int kMaxBatch = kBatchInflightMax;
struct BuildBatch {
  int group, n;
  BuildParams p[kMaxBatch];
};
static_assert(sizeof(BuildBatch) <= 32000, "kernel parameter space");

__global__ void __launch_bounds__(kTile, TRG_KBUILD_MINB) k_build(const __grid_constant__ BuildBatch b) {
  const int i = blockIdx.x / b.group;
  if (i < b.n) build_run(b.p[i], b.group, blockIdx.x - i * b.group);
}

// Number of exchange points of a sharded build of depth L (k_build runs
// L * this + 1 segments).
inline int build_exchange_points_per_round(int em_iters) {
  int n = 0;
  for (int ph_i = 0; ph_i < em_iters + 12; ++ph_i) {
    // mirrors phase_of: every phase but layout and partition write reduces
    const int I = em_iters;
    const bool layout = ph_i == I + 10, pwrite = ph_i == I + 11;
    if (!layout && !pwrite) ++n;
  }
  return n;
}

// ----------------------------------------------------------------- calibration
// calibrate_pass (gmm.cpp:523-580) as a dataflow over the tree: after the
// pass's association (exact per-leaf accumulators) and one grid barrier,
// every node is finished by the thread that completes it:
//   leaf j (thread j / G of CTA j % G): branch mass = its m0, refit of mean
//     and floored covariance from its deposits (gmm.cpp:532-545), then
//     arrival on its parent's counter;
//   internal node P (by the thread whose arrival completes P's children):
//     branch mass = sum of the children's in child order (gmm.cpp:547-556),
//     reweight of P's octet (mass shares; a shadowed octet keeps its shares,
//     gmm.cpp:557-566), the moment match of P from its children
//     (reset_parents_to_child_moments, gmm.cpp:489-513), then arrival on P's
//     parent; P's refresh_eig (gmm.cpp:576-578) runs after the climb, since
//     nothing above P needs P's eigen fields;
//   the top octet is reweighted by the thread completing the level-0 set.
// The reference's loops run level by level; every value here comes from
// the same operands in the same order (child order for every sum), so the
// pass computes the same tree, with a critical path of one leaf refit, the
// chain of moment matches and the eigensolves of the completing thread.
// Drift is the max over all of it (atomicMax on the bits of a double >= 0).
// A second grid barrier closes the pass.
struct CalCtx {
  double* branch;    // [capacity] subtree deposit mass of this pass
  unsigned* arrive;  // [capacity + 1] (slot capacity: the top octet)
  int root_count;
};

__device__ __forceinline__ void cal_reweight(const BuildParams& p, const double* branch, int first,
                                             int count, double& drift) {
  double b[8], wo[8];  // every operand in one round trip (count <= 8)
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    b[c] = c < count ? __ldcg(&branch[first + c]) : 0.0;
    wo[c] = c < count ? __ldcg(&p.nodes[first + c].weight) : 0.0;
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < 8; ++c)
    if (c < count) s += b[c];
  if (!(s > 0.0)) return;  // shadowed octet: keep the fitted shares
#pragma unroll
  for (int c = 0; c < 8; ++c)
    if (c < count) {
      const double w = b[c] / s;
      drift = smax(drift, fabs(wo[c] - w));
      p.nodes[first + c].weight = w;
    }
}

// A node is final for this pass: arrive on its parent `par` (-1: the top
// octet), which has `need` children (both loaded by the caller ahead of
// time, off the climb's critical path).  Returns the parent when this
// arrival completed it (its node work is then this thread's), -1 otherwise
// (or after reweighting the top octet).
__device__ __forceinline__ int cal_arrive(const BuildParams& p, const CalCtx& cx, int par, int need,
                                          double& drift) {
  const int slot = par >= 0 ? par : p.capacity;
  const unsigned old = atom_add_acq_rel(&cx.arrive[slot], 1u);  // release mine, acquire siblings'
  if (old + 1 != (unsigned)need) return -1;
  cx.arrive[slot] = 0u;
  if (par < 0) {  // top octet (gmm.cpp:567-571)
    cal_reweight(p, cx.branch, 0, cx.root_count, drift);
    return -1;
  }
  return par;
}

// Sums of v[i] over lanes [0, cc) of the warp, each in lane (= child)
// order -- the reference's serial loop order; the N sums interleave (one
// shuffle round per child for all of them) and the results are uniform.
template <int N>
__device__ __forceinline__ void child_sums(const double (&v)[N], int cc, double (&out)[N]) {
#pragma unroll
  for (int i = 0; i < N; ++i) out[i] = 0.0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const double x = __shfl_sync(0xffffffffu, v[i], q);
      if (q < cc) out[i] += x;
    }
  }
}

// Internal node P, all children final, by one warp (lane c holds child c):
// branch mass, octet reweight, moment match of P (no eigensolve).  Every
// sum runs in child order.
__device__ void cal_internal(const BuildParams& p, const CalCtx& cx, int P, double& drift,
                             int& ppar, int& pneed) {
  const int lane = threadIdx.x & 31;
  const int f = __ldcg(&p.nodes[P].first_child), cc = __ldcg(&p.nodes[P].child_count);
  ppar = __ldcg(&p.nodes[P].parent);  // for the next arrival (with the children's loads)
  pneed = ppar >= 0 ? __ldcg(&p.nodes[ppar].child_count) : cx.root_count;
  const bool own = lane < cc;
  const int ci = f + (own ? lane : 0);
  const double cb = own ? __ldcg(&cx.branch[ci]) : 0.0;
  double cw = own ? __ldcg(&p.nodes[ci].weight) : 0.0;
  double cm[3], cv[9];
#pragma unroll
  for (int k = 0; k < 3; ++k) cm[k] = own ? __ldcg(&p.nodes[ci].mean[k]) : 0.0;
#pragma unroll
  for (int k = 0; k < 9; ++k) cv[k] = own ? __ldcg(&p.cov[9 * (size_t)ci + k]) : 0.0;
  const double bv[1] = {cb};
  double bb[1];
  child_sums<1>(bv, cc, bb);
  const double b = bb[0];  // branch (gmm.cpp:547-556) = the octet's share sum
  if (lane == 0) cx.branch[P] = b;
  if (b > 0.0 && own) {  // reweight (gmm.cpp:557-566); a shadowed octet keeps its shares
    const double nw = cb / b;
    drift = smax(drift, fabs(cw - nw));
    cw = nw;
    p.nodes[ci].weight = nw;
  }
  const double wv[4] = {cw, __dmul_rn(cw, cm[0]), __dmul_rn(cw, cm[1]), __dmul_rn(cw, cm[2])};
  double wm[4];
  child_sums<4>(wv, cc, wm);
  const double w = wm[0];
  if (!(w > 0.0)) return;
  double mu[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) mu[k] = wm[1 + k] / w;
  const double d[3] = {cm[0] - mu[0], cm[1] - mu[1], cm[2] - mu[2]};
  double t[9], cs[9];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int q = 0; q < 3; ++q)
      t[3 * r + q] = __dmul_rn(cw, __dadd_rn(cv[3 * r + q], __dmul_rn(d[r], d[q])));
  child_sums<9>(t, cc, cs);
  if (lane < 9) {
    double v = cs[0];
#pragma unroll
    for (int q = 1; q < 9; ++q) v = lane == q ? cs[q] : v;
    p.cov[9 * (size_t)P + lane] = v / w;
  }
  if (lane < 3) p.nodes[P].mean[lane] = mu[lane];
}

// Leaf refit (gmm.cpp:532-545) from the leaf's deposits m[10].
__device__ void cal_leaf(const BuildParams& p, const CalCtx& cx, int j, const double m[10],
                         double& drift) {
  cx.branch[j] = m[0];
  DNode& nd = p.nodes[j];
  if (!(m[0] > 0.0)) return;
  const double mu[3] = {m[1] / m[0], m[2] / m[0], m[3] / m[0]};
  const double M[3][3] = {{m[4], m[5], m[6]}, {m[5], m[7], m[8]}, {m[6], m[8], m[9]}};
  double S[3][3], S2[3][3];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) S[r][c] = M[r][c] / m[0] - mu[r] * mu[c];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) S2[r][c] = 0.5 * (S[r][c] + S[c][r]);
  double dm = (nd.mean[0] - mu[0]) * (nd.mean[0] - mu[0]);
  dm += (nd.mean[1] - mu[1]) * (nd.mean[1] - mu[1]);
  dm += (nd.mean[2] - mu[2]) * (nd.mean[2] - mu[2]);
  drift = smax(drift, sqrt(dm));
  double before[3][3];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) before[r][c] = p.cov[9 * (size_t)j + 3 * r + c];
  GComp g;
  g.w = nd.weight;
  for (int q = 0; q < 3; ++q) g.mean[q] = mu[q];
  if (comp_set_cov_cf(g, S2, cov_floor(S2, p.eps, p.abs_floor))) atomicCAS(p.status, 0, kEInval);
  double dc[3][3];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) dc[r][c] = g.cov[3 * r + c] - before[r][c];
  drift = smax(drift, norm33(dc));
  // every field but weight (the parent's octet reweight owns it this pass)
  for (int i = 0; i < 3; ++i) nd.mean[i] = g.mean[i];
  for (int i = 0; i < 9; ++i) {
    nd.axT[i] = g.axT[i];
    p.cov[9 * (size_t)j + i] = g.cov[i];
  }
  for (int i = 0; i < 3; ++i) {
    nd.lam[i] = g.lam[i];
    nd.il[i] = 1.0 / g.lam[i];
  }
  for (int i = 0; i < 6; ++i) nd.prec[i] = g.prec[i];
  nd.log_norm = g.log_norm;
  const double tr = (g.lam[0] + g.lam[1]) + g.lam[2];
  nd.cplx = tr > 0.0 ? g.lam[2] / tr : -1.0;
}

#ifndef TRG_PROBE_PASS
#define TRG_PROBE_PASS 10
#endif
#ifdef TRG_CAL_PROBE
#define CAL_PROBE(cond, lab) \
  if ((cond) && __ldcg(&p.st->cal_pass) == TRG_PROBE_PASS) tl_mark_any(p.tl, lab)
#else
#define CAL_PROBE(cond, lab)
#endif
// Leaf j final (its warp; lane 0 did the refit): climb as long as this warp
// completes ancestors, then the refresh_eig of every node it matched, one
// lane each.
__device__ void cal_finish_leaf(const BuildParams& p, const CalCtx& cx, int j, int par, int need,
                                double& drift) {
  const int lane = threadIdx.x & 31;
  int done[8];
  int nd = 0;
  int P = -1;
  if (lane == 0) P = cal_arrive(p, cx, par, need, drift);
  P = __shfl_sync(0xffffffffu, P, 0);
  CAL_PROBE(lane == 0 && j % 16 == 0, 5003);
  while (P >= 0) {
    int ppar, pneed;
    cal_internal(p, cx, P, drift, ppar, pneed);
    __syncwarp();
    CAL_PROBE(lane == 0, 5010);
    done[nd++] = P;
    if (lane == 0) P = cal_arrive(p, cx, ppar, pneed, drift);
    P = __shfl_sync(0xffffffffu, P, 0);
    CAL_PROBE(lane == 0, 5011);
  }
  if (nd) {  // the refreshes, one lane each (closed-form solver)
    int mine = -1;
    for (int k = 0; k < nd; ++k)
      if (lane == k) mine = done[k];
    double cv[9];
    for (int q = 0; q < 9; ++q) cv[q] = mine >= 0 ? __ldcg(&p.cov[9 * (size_t)mine + q]) : 0.0;
    if (refresh_node_cf(p.nodes[mine >= 0 ? mine : 0], cv, mine >= 0))
      atomicCAS(p.status, 0, kEInval);
    CAL_PROBE(lane == 0, 5030);
  }
  __syncwarp();
}

// Second persistent kernel of the build (launched right behind k_build on
// the same stream): parent moment match + refresh_eig, then the leaf
// calibration passes.
// Three CTAs per SM (80 registers): the association windows are bound by
// each SM's share of the descents, and 24 warps per SM hide their latency
// better than 16 (C2 stage 1 22.4 -> 19.3 us per pass); the leaf refits'
// spills cost less (stage 2 +0.8 us).
#ifndef TRG_KCAL_MINB
#define TRG_KCAL_MINB 3
#endif
__device__ __forceinline__ void calibrate_run(const BuildParams& p, int G, int cta) {
  __shared__ FxScale sc[3];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ int lvl[9];
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  BuildState* st = p.st;
  const bool sharded = p.seg >= 0;
  if (__ldcg(&st->status_overflow)) {
    if (cta == 0 && tid == 0) p.meta->ok = 0;
    return;
  }
  if (sharded && __ldcg(&st->cal_done)) return;
  const int J = __ldcg(&st->J);
  if (tid < 9) lvl[tid] = __ldcg(&st->lvl_start[tid]);
  if (tid == 0) {
    mbar_init(&mbar, 1);
    mbar_fence_init();
    assoc_scales(p.a.pmax, nullptr, sc);
  }
  __syncthreads();
  // ------------------------------------------------ rematch + refresh_eig
  if (!sharded || p.seg == 0) {
    tl_mark(p.tl, 900);
    if (cta == 0) reset_parents(p, lvl);
    grid_sync(p.bar + 8, G);
    tl_mark(p.tl, 901);
    for (int base = 0; base < J; base += G * blockDim.x) {  // refresh_eig
      const int j = base + cta * blockDim.x + tid;
      const bool act = j < J;
      if (refresh_node_cf(p.nodes[act ? j : 0], p.cov + 9 * (size_t)(act ? j : 0), act))
        atomicCAS(p.status, 0, kEInval);
    }
    grid_sync(p.bar + 8, G);
    tl_mark(p.tl, 902);
  }
  // ------------------------------------------------ leaf calibration
  // Sharded (p.seg >= 0): segment s runs stage 2 of pass s-1 (from the
  // all-reduced leaf moments in xcal) and stage 1 of pass s up to the local
  // leaf moments, then exits for the exchange.
  CalCtx cx;
  cx.branch = p.cal_moments;
  cx.arrive = p.cal_arrive;
  cx.root_count = lvl[1] - lvl[0];
  extern __shared__ __align__(128) unsigned char k_cal_stage[];  // upper levels for the descent
  DNode* cal_stage = reinterpret_cast<DNode*>(k_cal_stage);
  const int n_stage = min(p.L >= 2 ? lvl[p.L - 1] : 0, kStageNodes);
  const size_t accJ = (size_t)p.capacity * 30;  // limbs per accumulator buffer
  unsigned mphase = 0;
  constexpr int WPB = kTile / 32;
  for (int pass = 0; pass < 40; ++pass) {
    const bool run_s1 = !sharded || p.seg == pass;
    const bool run_s2 = !sharded || p.seg == pass + 1;
    if (!run_s1 && !run_s2) continue;
    AssocParams a = p.a;
    a.n_nodes = J;
    a.root_count = cx.root_count;
    a.snodes = cal_stage;
    a.n_snodes = n_stage;
    a.acc = p.cal_acc + (size_t)(pass % 3) * accJ;
#ifdef TRG_ASSOC_PROBE
    a.tl = pass == TRG_PROBE_PASS ? p.tl : nullptr;
    if (pass == TRG_PROBE_PASS && tid == 0 && cta % 32 == 0) tl_mark_any(p.tl, 5100);
#endif
    if (run_s1) {
      // the upper levels (stage 2 rewrote them) are copied while the drift
      // test's load is in flight
      stage_nodes_issue(cal_stage, p.nodes, n_stage, &mbar);
      bool stop = false;
      if (pass > 0) {
        const double dprev = __longlong_as_double((long long)__ldcg(&p.drift_bits[(pass - 1) & 1]));
        stop = !(dprev > 1e-13);  // gmm.cpp:652
      }
      stage_nodes_wait(n_stage, &mbar, mphase);  // (no copy may outlive the CTA)
      if (stop) {
        if (sharded && cta == 0 && tid == 0) st->cal_done = 1;
        break;
      }
      if (cta == 0 && tid == 0) p.drift_bits[pass & 1] = 0ull;
#ifdef TRG_ASSOC_PROBE
      if (pass == TRG_PROBE_PASS && tid == 0 && cta % 32 == 0) tl_mark_any(p.tl, 5103);
#endif
      // warp-major window order: the windows beyond one per warp land on
      // different SMs (the pass is bound by each SM's share of the descents)
      assoc_fx_pass<10>(a, nullptr, sc, G * WPB, warp * G + cta);
      grid_sync(p.bar + 8, G);
      tl_mark(p.tl, 1000 + pass * 10 + 1);
      if (sharded) {
        // this shard's leaf moments, for the all-reduce (rows zeroed for
        // the next segment)
        for (int j = cta * WPB + warp; j < J; j += G * WPB) {
          double m[10];
          fx_row<10>(a.acc, a.acc_stride, j, sc, m);
          __syncwarp();
          if (lane < 30) a.acc[(size_t)lane * a.acc_stride + j] = 0;
          if (lane == 0 && __ldcg(&p.nodes[j].child_count) == 0)
            for (int q = 0; q < 10; ++q) p.xcal[(size_t)j * 10 + q] = m[q];
        }
        return;
      }
    }
    if (!sharded) {
      // zero this CTA's slice of the buffer pass+2 writes
      long long* z = p.cal_acc + (size_t)((pass + 2) % 3) * accJ;
      for (size_t q = (size_t)cta * blockDim.x + tid; q < accJ; q += (size_t)G * blockDim.x) z[q] = 0;
    }
    double drift = 0.0;
    for (int j = warp * G + cta; j < J; j += G * WPB) {  // a warp per leaf, spread over SMs
      const int cc_j = __ldcg(&p.nodes[j].child_count), par_j = __ldcg(&p.nodes[j].parent);
      if (cc_j != 0) continue;  // leaves only
      // the parent's child count for the arrival, loaded under the refit
      const int need_j = par_j >= 0 ? __ldcg(&p.nodes[par_j].child_count) : cx.root_count;
      if (lane == 0) {
        CAL_PROBE(j % 16 == 0, 5000);
        double m[10];
        if (sharded) {
          for (int q = 0; q < 10; ++q) m[q] = __ldcg(p.xcal + (size_t)j * 10 + q);
        } else {
          fx_row<10>(a.acc, a.acc_stride, j, sc, m);
        }
        CAL_PROBE(j % 16 == 0, 5001);
        cal_leaf(p, cx, j, m, drift);
        CAL_PROBE(j % 16 == 0, 5002);
      }
      __syncwarp();
      cal_finish_leaf(p, cx, j, par_j, need_j, drift);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) drift = smax(drift, __shfl_xor_sync(0xffffffffu, drift, off));
    if (lane == 0 && drift > 0.0)
      atomicMax(&p.drift_bits[pass & 1], (unsigned long long)__double_as_longlong(drift));
    grid_sync(p.bar + 8, G);
    tl_mark(p.tl, 1000 + pass * 10 + 2);
    if (cta == 0 && tid == 0) {
      st->drift = __longlong_as_double((long long)__ldcg(&p.drift_bits[pass & 1]));
      st->cal_pass = pass + 1;
    }
  }
  if (cta == 0 && tid == 0) {
    st->cal_evals = __ldcg(&p.a.counters[1]);
    TreeMeta m;
    m.J = J;
    m.root_count = cx.root_count;
    m.n_upper = p.L >= 2 ? lvl[p.L - 1] : 0;
    m.ok = __ldcg(p.status) == 0 ? 1 : 0;
    *p.meta = m;
  }
}

__global__ void __launch_bounds__(kTile, TRG_KCAL_MINB) k_calibrate(const __grid_constant__ BuildBatch b) {
  const int i = blockIdx.x / b.group;
  if (i < b.n) calibrate_run(b.p[i], b.group, blockIdx.x - i * b.group);
}

__global__ void k_init_entries(const double* __restrict__ pts, size_t n, double* ex, double* ey,
                               double* ez, double* ew, int* tile_node, int* tile_start,
                               int* tile_len, int* status, unsigned long long* pmax_bits) {
  double am = 0.0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const double x = pts[3 * i], y = pts[3 * i + 1], z = pts[3 * i + 2];
    if (!isfinite(x) || !isfinite(y) || !isfinite(z)) atomicCAS(status, 0, kEInval);
    am = fmax(am, fmax(fabs(x), fmax(fabs(y), fabs(z))));
    ex[i] = x;
    ey[i] = y;
    ez[i] = z;
    ew[i] = 1.0;
    if (i % kTile == 0) {
      const size_t t = i / kTile;
      tile_node[t] = 0;
      tile_start[t] = (int)i;
      tile_len[t] = (int)min((size_t)kTile, n - i);
    }
  }
  am = block_max_nonneg(am);  // one atomic per block (per-warp atomics serialised on one word)
  if (threadIdx.x == 0 && am > 0.0) atomicMax(pmax_bits, (unsigned long long)__double_as_longlong(am));
}

}  // namespace trg

using namespace trg;

namespace trg {
int stage_points_public(trg_ctx* ctx, const double* xyz, size_t n, int on_device, int slot,
                        const double** dev);
}

namespace {

struct BuildAlloc {
  int Kmax, Tmax, Emax;
};

struct BuildJob {
  BuildParams p;
  trg_tree_dev* tree = nullptr;
  int G = 0, Gc = 0;
  BuildAlloc al;
};

// Everything up to the persistent launches: arena, parameters, initial
// state, entry buffer (k_init_entries).  `world` > 0 adds the sharded
// exchange buffers (seg mode) for that many shards.
int build_prepare(trg_ctx* ctx, const double* pts, size_t n, const trg_model_config* cfg,
                  BuildAlloc al, trg_build_diag* diag, int world, BuildJob* job) {
  const int L = cfg->max_level;
  const int cap = trg_tree_capacity(L);
  BuildParams p{};
  p.pts = pts;
  p.n = n;
  p.L = L;
  p.em_iters = cfg->em_iterations_per_node;
  p.min_points = (double)cfg->min_points_per_node;
  p.eps = cfg->cov_regularization_epsilon;
  p.abs_floor = cfg->cov_regularization_absolute;
  p.Kmax = al.Kmax;
  p.Tmax = al.Tmax;
  p.Emax = al.Emax;
  p.capacity = cap;
  // ---- one arena for everything
  const size_t E = (size_t)al.Emax, T = (size_t)al.Tmax, K = (size_t)al.Kmax;
  size_t off = 0;
  auto carve = [&](size_t bytes) {
    const size_t o = off;
    off += (bytes + 255) & ~size_t(255);
    return o;
  };
  size_t o_e[2][4], o_rn[2][5], o_tl[2][3];
  for (int b = 0; b < 2; ++b) {
    for (int q = 0; q < 4; ++q) o_e[b][q] = carve(sizeof(double) * (E + 2));  // + bulk-copy tail
    for (int q = 0; q < 5; ++q) o_rn[b][q] = carve(sizeof(int) * K);
    for (int q = 0; q < 3; ++q) o_tl[b][q] = carve(sizeof(int) * T);
  }
  const size_t o_mass = carve(sizeof(double) * K), o_ref = carve(sizeof(double) * 3 * K),
               o_mean = carve(sizeof(double) * 3 * K), o_sc = carve(sizeof(double) * 9 * K),
               o_fl = carve(sizeof(double) * K), o_seeds = carve(sizeof(double) * 24 * K),
               o_wmi = carve(sizeof(int) * K), o_comps = carve(sizeof(GComp) * 16 * K),
               o_fll = carve(sizeof(double) * 2 * K), o_cm = carve(sizeof(double) * 16 * K),
               o_kept = carve(sizeof(int) * K), o_ok = carve(sizeof(int) * K),
               o_ns = carve(sizeof(int) * K), o_surv = carve(sizeof(int) * 8 * K),
               o_sm = carve(sizeof(double) * 8 * K), o_st = carve(sizeof(double) * K),
               o_nseg = carve(sizeof(int) * 8 * K), o_arr = carve(sizeof(unsigned) * K),
               o_part = carve(sizeof(double) * kRec * T),
               o_nred = carve(sizeof(double) * kRec * K), o_fd = carve(sizeof(unsigned) * K),
               o_tb = carve(sizeof(double) * 8 * T),
               o_md = carve(sizeof(double) * E), o_emit = carve(sizeof(double) * 8 * E),
               o_calm = carve(sizeof(double) * 10 * cap), o_bar = carve(64),
               o_cacc = carve(sizeof(long long) * 3 * 30 * (size_t)cap), o_pmax = carve(64),
               o_lay = carve(sizeof(int) * 56 * K),
               o_llt = carve(sizeof(double) * (size_t)cap * 2 * (cfg->em_iterations_per_node + 1)),
               o_kex = carve(sizeof(int) * (size_t)cap),
               o_car = carve(sizeof(unsigned) * ((size_t)cap + 1)), o_dbits = carve(16),
               o_meta = carve(sizeof(TreeMeta)),
               o_state = carve(sizeof(BuildState));
  TRG_CU(set_dynamic_smem((const void*)k_build, sizeof(BuildSmem)));
  int G = persistent_grid(ctx, (const void*)k_build, kTile, sizeof(BuildSmem));
  {
    // CTAs per SM from the largest round's expected tile count (entries grow
    // ~4x per level): small clouds run fewer CTAs (cheaper grid barriers; C1
    // 2.90 -> 2.78 ms).  k_build's results do not depend on the grid (tile
    // records are reduced in tile order).
    const double est_tiles = (double)n * std::pow(4.0, (double)(L - 1)) / kTile;
    int per_sm = (int)std::min(3.0, std::max(1.0, std::ceil(est_tiles / (4.0 * ctx->sms))));
    G = std::min(G, ctx->sms * std::max(1, per_sm));
  }
  const size_t cal_smem = sizeof(DNode) * kStageNodes;
  TRG_CU(set_dynamic_smem((const void*)k_calibrate, cal_smem));
  int Gc = persistent_grid(ctx, (const void*)k_calibrate, kTile, cal_smem);
  {
    // CTAs per SM from the cloud size: each CTA's association tile should
    // hold ~200 points; small clouds run fewer, fuller CTAs (cheaper grid
    // barriers and per-leaf combines: C1 10k points 3.36 -> 2.89 ms build;
    // C2 76.8k stays at 3/SM, its optimum)
    int per_sm = (int)std::min<size_t>(3, std::max<size_t>(1, (n + 192 * (size_t)ctx->sms - 1) /
                                                                  (192 * (size_t)ctx->sms)));
    Gc = std::min(Gc, ctx->sms * std::max(1, per_sm));
  }
  const size_t o_cd = carve(sizeof(double) * std::max(G, Gc));
  const int W = std::max(world, 1);
  const size_t o_xa = carve(sizeof(double) * 8 * K), o_xaa = carve(sizeof(double) * 8 * K * W),
               o_xc = carve(sizeof(double) * 10 * (size_t)cap);
  void* arena = nullptr;
  TRG_TRY(ws_get(ctx, kSlotBuild0, off, &arena));
  char* A = static_cast<char*>(arena);
  for (int b = 0; b < 2; ++b) {
    p.ex[b] = (double*)(A + o_e[b][0]);
    p.ey[b] = (double*)(A + o_e[b][1]);
    p.ez[b] = (double*)(A + o_e[b][2]);
    p.ew[b] = (double*)(A + o_e[b][3]);
    p.rn[b].tree_id = (int*)(A + o_rn[b][0]);
    p.rn[b].seg = (int*)(A + o_rn[b][1]);
    p.rn[b].len = (int*)(A + o_rn[b][2]);
    p.rn[b].tile0 = (int*)(A + o_rn[b][3]);
    p.rn[b].ntiles = (int*)(A + o_rn[b][4]);
    p.tile_node[b] = (int*)(A + o_tl[b][0]);
    p.tile_start[b] = (int*)(A + o_tl[b][1]);
    p.tile_len[b] = (int*)(A + o_tl[b][2]);
  }
  p.nf.mass = (double*)(A + o_mass);
  p.nf.ref = (double*)(A + o_ref);
  p.nf.mean = (double*)(A + o_mean);
  p.nf.scatter = (double*)(A + o_sc);
  p.nf.floorv = (double*)(A + o_fl);
  p.nf.seeds = (double*)(A + o_seeds);
  p.nf.wmax_idx = (int*)(A + o_wmi);
  p.nf.comps = (GComp*)(A + o_comps);
  p.nf.final_ll = (double*)(A + o_fll);
  p.nf.cmass = (double*)(A + o_cm);
  p.nf.kept = (int*)(A + o_kept);
  p.nf.ok = (int*)(A + o_ok);
  p.nf.ns = (int*)(A + o_ns);
  p.nf.surv = (int*)(A + o_surv);
  p.nf.smass = (double*)(A + o_sm);
  p.nf.stotal = (double*)(A + o_st);
  p.nf.next_seg = (int*)(A + o_nseg);
  p.nf.arrive = (unsigned*)(A + o_arr);
  p.partial = (double*)(A + o_part);
  p.nodered = (double*)(A + o_nred);
  p.fdone = (unsigned*)(A + o_fd);
  p.meta = (TreeMeta*)(A + o_meta);
  p.tile_base = (double*)(A + o_tb);
  p.min_d2 = (double*)(A + o_md);
  p.emit = (double*)(A + o_emit);
  p.cal_moments = (double*)(A + o_calm);
  p.cal_acc = (long long*)(A + o_cacc);
  p.pmax_bits = (unsigned long long*)(A + o_pmax);
  p.layout_scratch = (int*)(A + o_lay);
  p.ll_trace = (double*)(A + o_llt);
  p.kept_exp = (int*)(A + o_kex);
  p.cal_arrive = (unsigned*)(A + o_car);
  p.drift_bits = (unsigned long long*)(A + o_dbits);
  p.bar = (unsigned*)(A + o_bar);
  p.st = (BuildState*)(A + o_state);
  p.cta_drift = (double*)(A + o_cd);
  p.status = ctx->status;
  p.tl = ctx->dev_timeline;
  p.seg = world > 0 ? 0 : -1;
  p.n_ranks = W;
  p.xarg = (double*)(A + o_xa);
  p.xarg_all = (double*)(A + o_xaa);
  p.xcal = (double*)(A + o_xc);
  p.want_traces = (diag && diag->ll_traces && diag->ll_trace_capacity > 0) ? 1 : 0;
  TRG_TRY(timeline_reset(ctx));
  // tree
  trg_tree_dev* tree = nullptr;
  TRG_TRY(tree_alloc(ctx, cap, &tree));
  tree->max_level = L;
  p.nodes = tree->nodes;
  p.cov = tree->cov;
  // calibration association (NM = 10, identity, lambda_c = 0, full depth)
  void* cnt;
  TRG_TRY(ws_get(ctx, kSlotCounters, 64, &cnt));
  p.a.nodes = tree->nodes;
  p.a.depth = L;
  p.a.lambda_c = 0.0;
  p.a.outlier_floor = 1e-300;
  p.a.pts = pts;
  p.a.n = n;
  p.a.Rt = nullptr;
  p.a.counters = (unsigned long long*)cnt;
  p.a.pmax = reinterpret_cast<const double*>(p.pmax_bits);
  p.a.acc_stride = (size_t)cap;
  p.a.status = ctx->status;
  // ---- initial state
  BuildState st{};
  st.Kp[0] = 1;
  st.Tp[0] = (int)((n + kTile - 1) / kTile);
  st.Ep[0] = (int)n;
  st.J = 0;
  st.drift = INFINITY;
  st.E_round[0] = n;
  st.K_round[0] = 1;
  TRG_CU(cudaMemsetAsync(A + o_bar, 0, 64, ctx->stream));
  TRG_CU(cudaMemsetAsync(A + o_arr, 0, sizeof(unsigned) * K, ctx->stream));
  TRG_CU(cudaMemsetAsync(A + o_fd, 0, sizeof(unsigned) * K, ctx->stream));
  TRG_CU(cudaMemsetAsync(A + o_car, 0, sizeof(unsigned) * ((size_t)cap + 1), ctx->stream));
  TRG_CU(cudaMemsetAsync(A + o_cacc, 0, sizeof(long long) * 3 * 30 * (size_t)cap, ctx->stream));
  TRG_CU(cudaMemsetAsync(A + o_pmax, 0, 64, ctx->stream));
  TRG_CU(cudaMemsetAsync(cnt, 0, 64, ctx->stream));
  // initial state through a dedicated pinned buffer: asynchronous copies, no
  // staging syncs (the previous build's copies completed at its collect)
  void* hinit = nullptr;
  TRG_TRY(host_ws_get(ctx, kSlotHostBuildInit, sizeof(BuildState) + 8 * sizeof(int), &hinit));
  std::memcpy(hinit, &st, sizeof st);
  int* h_rn = reinterpret_cast<int*>(static_cast<char*>(hinit) + sizeof(BuildState));
  const int rn0[5] = {-1, 0, (int)n, 0, st.Tp[0]};
  std::memcpy(h_rn, rn0, sizeof rn0);
  TRG_CU(trg_memcpy(ctx, p.st, hinit, sizeof st, cudaMemcpyHostToDevice));
  for (int q = 0; q < 5; ++q)
    TRG_CU(trg_memcpy(ctx, A + o_rn[0][q], &h_rn[q], sizeof(int), cudaMemcpyHostToDevice));
  k_init_entries<<<256, 256, 0, ctx->stream>>>(pts, n, p.ex[0], p.ey[0], p.ez[0], p.ew[0],
                                               p.tile_node[0], p.tile_start[0], p.tile_len[0],
                                               ctx->status, p.pmax_bits);
  ctx->launches += 1;
  // the calibration's association reads a spatially sorted copy (trg_sort.cu)
  TRG_TRY(morton_sorted_copy(ctx, pts, n, p.a.pmax, kSlotBuild2, kSlotBuild3, &p.a.pts));
  job->p = p;
  job->tree = tree;
  job->G = G;
  job->Gc = Gc;
  job->al = al;
  return TRG_OK;
}

// One k_build launch (seg = -1: the whole build; else one sharded segment).
// A batch of one on G CTAs (only p[0] is read).
std::unique_ptr<BuildBatch> single_batch(const BuildParams& p, int G) {
  std::unique_ptr<BuildBatch> b(new BuildBatch);
  b->group = G;
  b->n = 1;
  b->p[0] = p;
  return b;
}

int build_launch(trg_ctx* ctx, BuildJob* job, int seg) {
  job->p.seg = seg;
  auto b = single_batch(job->p, job->G);
  void* args[] = {b.get()};
  TRG_CU(launch_persistent(ctx, (const void*)k_build, job->G, kTile, args, sizeof(BuildSmem)));
  ctx->launches += 1;
  return TRG_OK;
}

int calibrate_launch(trg_ctx* ctx, BuildJob* job, int seg) {
  job->p.seg = seg;
  auto b = single_batch(job->p, job->Gc);
  void* args[] = {b.get()};
  TRG_CU(launch_persistent(ctx, (const void*)k_calibrate, job->Gc, kTile, args,
                           sizeof(DNode) * kStageNodes));
  ctx->launches += 1;
  return TRG_OK;
}

// Reads the build state back, checks status / overflow, fills diagnostics.
int build_collect(trg_ctx* ctx, BuildJob* job, const trg_model_config* cfg, trg_tree_dev** out,
                  trg_build_diag* diag, bool* overflow, BuildAlloc* need) {
  BuildParams& p = job->p;
  trg_tree_dev* tree = job->tree;
  const BuildAlloc al = job->al;
  const int L = cfg->max_level;
  // state and status word in one round trip (pinned, one synchronisation)
  void* hc = nullptr;
  TRG_TRY(host_ws_get(ctx, kSlotHostCollect, sizeof(BuildState) + 16, &hc));
  TRG_CU(cudaMemcpyAsync(hc, p.st, sizeof(BuildState), cudaMemcpyDeviceToHost, ctx->stream));
  int* hstatus = reinterpret_cast<int*>(static_cast<char*>(hc) + sizeof(BuildState));
  TRG_CU(cudaMemcpyAsync(hstatus, ctx->status, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  TRG_CU(cudaStreamSynchronize(ctx->stream));
  ctx->bytes_d2h += sizeof(BuildState) + sizeof(int);
  BuildState st;
  std::memcpy(&st, hc, sizeof st);
  int rc = status_result(ctx, *hstatus, ctx->status, "build_tree");
  if (rc == TRG_OK && st.status_overflow) {
    *overflow = true;
    need->Emax = std::max(al.Emax, st.need_E);
    need->Kmax = std::max(al.Kmax, st.need_K);
    need->Tmax = std::max(al.Tmax, st.need_T);
    trg_tree_free(ctx, tree);
    return TRG_OK;
  }
  if (rc != TRG_OK) {
    trg_tree_free(ctx, tree);
    return rc;
  }
  tree->n_nodes = st.J;
  tree->root_count = st.root_count;
  tree->n_upper = L >= 2 ? st.lvl_start[L - 1] : 0;
  TRG_TRY(timeline_fetch(ctx));
  if (diag) {
    for (int r = 0; r < 8; ++r) {
      diag->entries_per_round[r] = r < L ? st.E_round[r] : 0;
      diag->expanded_per_round[r] = r < L ? st.K_round[r] : 0;
    }
    diag->calibration_passes = st.cal_pass;
    diag->n_expansions = st.n_exp;
    if (diag->ll_traces && diag->ll_trace_capacity > 0) {
      const int I1 = cfg->em_iterations_per_node + 1;
      const int ne = std::min(st.n_exp, diag->ll_trace_capacity);
      std::vector<double> tr((size_t)std::max(1, ne) * 2 * I1);
      std::vector<int> kp(std::max(1, ne));
      if (ne > 0) {
        TRG_CU(trg_memcpy(ctx, tr.data(), p.ll_trace, sizeof(double) * tr.size(), cudaMemcpyDeviceToHost));
        TRG_CU(trg_memcpy(ctx, kp.data(), p.kept_exp, sizeof(int) * ne, cudaMemcpyDeviceToHost));
        TRG_CU(cudaStreamSynchronize(ctx->stream));
      }
      for (int e = 0; e < ne; ++e)
        for (int i = 0; i < I1; ++i)
          diag->ll_traces[(size_t)e * I1 + i] = tr[((size_t)e * 2 + kp[e]) * I1 + i];
    }
    diag->calibration_drift = st.drift;
    diag->calib_density_evaluations = st.cal_evals;
  }
  *out = tree;
  return TRG_OK;
}

int run_build(trg_ctx* ctx, const double* pts, size_t n, const trg_model_config* cfg,
              BuildAlloc al, trg_tree_dev** out, trg_build_diag* diag, bool* overflow,
              BuildAlloc* need) {
  BuildJob job;
  TRG_TRY(build_prepare(ctx, pts, n, cfg, al, diag, 0, &job));
  TRG_TRY(build_launch(ctx, &job, -1));
  TRG_TRY(calibrate_launch(ctx, &job, -1));
  return build_collect(ctx, &job, cfg, out, diag, overflow, need);
}

// validate_config gmm.cpp:465-477
int validate_model_config(const trg_model_config* cfg) {
  if (!cfg) {
    set_error("model config is null");
    return TRG_EINVAL;
  }
  if (cfg->max_level < 1) {
    set_error("max_level must be >= 1");
    return TRG_EINVAL;
  }
  if (cfg->max_level > 7) {
    set_error("max_level above 7 is not supported by this build");
    return TRG_EINVAL;
  }
  if (cfg->em_iterations_per_node < 1) {
    set_error("em_iterations_per_node must be >= 1");
    return TRG_EINVAL;
  }
  if (cfg->min_points_per_node < 1) {
    set_error("min_points_per_node must be >= 1");
    return TRG_EINVAL;
  }
  if (!(cfg->cov_regularization_epsilon >= 0.0) || !(cfg->cov_regularization_absolute > 0.0)) {
    set_error("covariance regularization must be positive");
    return TRG_EINVAL;
  }
  return TRG_OK;
}

// Initial entry-buffer capacity: soft-partition growth is data dependent
// (E_l/E_{l-1} ~2.5-5 on surfaces, at most 8).  Start from the largest ratio
// this context has seen (initially 12 x N for L >= 3) so repeated builds never
// take the overflow-and-retry path.
BuildAlloc initial_alloc(trg_ctx* ctx, size_t n, int L) {
  int kmax = 1;
  for (int l = 0; l + 1 < L; ++l) kmax *= 8;
  BuildAlloc al;
  al.Kmax = std::max(1, kmax);
  const double ratio = std::max(ctx->build_growth, L >= 3 ? 12.0 : (L == 2 ? 8.0 : 1.0));
  al.Emax = (int)std::min<double>((double)INT32_MAX / 16, ratio * (double)n + 1024.0);
  al.Tmax = al.Emax / kTile + al.Kmax + 8;
  return al;
}

}  // namespace

namespace trg {
int check_model_config(const trg_model_config* cfg) { return validate_model_config(cfg); }
}  // namespace trg

extern "C" int trg_build_tree(trg_ctx* ctx, const double* xyz, size_t n, int xyz_on_device,
                              const trg_model_config* cfg, trg_tree_dev** out,
                              trg_build_diag* diag) {
  trg::NvtxRange nvtx_range_("trg_build_tree");
  // validate_config gmm.cpp:465-477, validate_cloud :479-484
  TRG_TRY(validate_model_config(cfg));
  if (n == 0 || !xyz) {
    set_error("point cloud is empty");
    return TRG_EINVAL;
  }
  if (n > (size_t)INT32_MAX / 8) {
    set_error("point cloud too large for int32 entry indexing");
    return TRG_EINVAL;
  }
  TRG_CU(cudaSetDevice(ctx->device));
  const double* dev = nullptr;
  TRG_TRY(stage_points_public(ctx, xyz, n, xyz_on_device, kSlotPoints, &dev));
  BuildAlloc al = initial_alloc(ctx, n, cfg->max_level);
  for (int attempt = 0; attempt < 4; ++attempt) {
    bool overflow = false;
    BuildAlloc need = al;
    const int rc = run_build(ctx, dev, n, cfg, al, out, diag, &overflow, &need);
    if (rc != TRG_OK) {
      if (rc == TRG_EINVAL && trg_last_error()[0] == 'b') set_error("point cloud has non-finite coordinates or no mass");
      return rc;
    }
    if (!overflow) return TRG_OK;
    ctx->build_growth = std::max(ctx->build_growth, 1.25 * (double)need.Emax / (double)n);
    al.Emax = std::max(al.Emax * 2, need.Emax + 1024);
    al.Kmax = std::max(al.Kmax, need.Kmax);
    al.Tmax = al.Emax / kTile + al.Kmax + 8;
  }
  set_error("build_tree: entry buffer growth did not converge");
  return TRG_ERUNTIME;
}

// ------------------------------------------------------------ async build
namespace trg {

struct AsyncBuild {
  BuildJob job;
  BuildAlloc al;
  trg_model_config cfg;
  size_t n = 0;
};

int build_async_start(trg_ctx* ctx, const double* dev, size_t n, const trg_model_config* cfg,
                      AsyncBuild** h, trg_tree_dev** tree, const TreeMeta** meta, bool launch) {
  if (!*h) {  // first attempt: trg_build_tree's argument checks
    TRG_TRY(validate_model_config(cfg));
    if (n == 0 || !dev) {
      set_error("point cloud is empty");
      return TRG_EINVAL;
    }
    if (n > (size_t)INT32_MAX / 8) {
      set_error("point cloud too large for int32 entry indexing");
      return TRG_EINVAL;
    }
    *h = new AsyncBuild;
    (*h)->al = initial_alloc(ctx, n, cfg->max_level);
    (*h)->cfg = *cfg;
    (*h)->n = n;
  }
  AsyncBuild* b = *h;
  b->job = BuildJob{};
  TRG_TRY(build_prepare(ctx, dev, n, &b->cfg, b->al, nullptr, 0, &b->job));
  if (launch) {
    TRG_TRY(build_launch(ctx, &b->job, -1));
    TRG_TRY(calibrate_launch(ctx, &b->job, -1));
  }
  *tree = b->job.tree;
  *meta = b->job.p.meta;
  return TRG_OK;
}

int build_async_finish(trg_ctx* ctx, AsyncBuild* b, trg_tree_dev** out, bool* retry) {
  bool overflow = false;
  BuildAlloc need = b->al;
  *retry = false;
  const int rc = build_collect(ctx, &b->job, &b->cfg, out, nullptr, &overflow, &need);
  if (rc != TRG_OK) {
    if (rc == TRG_EINVAL && trg_last_error()[0] == 'b') set_error("point cloud has non-finite coordinates or no mass");
    return rc;
  }
  if (overflow) {  // as trg_build_tree's retry loop
    ctx->build_growth = std::max(ctx->build_growth, 1.25 * (double)need.Emax / (double)b->n);
    b->al.Emax = std::max(b->al.Emax * 2, need.Emax + 1024);
    b->al.Kmax = std::max(b->al.Kmax, need.Kmax);
    b->al.Tmax = b->al.Emax / kTile + b->al.Kmax + 8;
    *retry = true;
  }
  return TRG_OK;
}

void build_async_free(AsyncBuild* b) { delete b; }

// The builds of m prepared clouds (build_async_start without launch) as one
// k_build and one k_calibrate launch on ctx's stream, each cloud
// on an equal group of the co-resident grid.
int build_batch_launch(trg_ctx* ctx, AsyncBuild* const* hs, int m) {
  if (m < 1 || m > kMaxBatch) {
    set_error("build_batch_launch: bad batch size");
    return TRG_EINVAL;
  }
  std::unique_ptr<BuildBatch> b(new BuildBatch);
  b->n = m;
  for (int k = 0; k < m; ++k) {
    b->p[k] = hs[k]->job.p;
    b->p[k].seg = -1;
  }
  void* args[] = {b.get()};
  TRG_CU(set_dynamic_smem((const void*)k_build, sizeof(BuildSmem)));
  b->group = persistent_grid(ctx, (const void*)k_build, kTile, sizeof(BuildSmem)) / m;
  TRG_CU(launch_persistent(ctx, (const void*)k_build, b->group * m, kTile, args, sizeof(BuildSmem)));
  const size_t cal_smem = sizeof(DNode) * kStageNodes;
  TRG_CU(set_dynamic_smem((const void*)k_calibrate, cal_smem));
  b->group = persistent_grid(ctx, (const void*)k_calibrate, kTile, cal_smem) / m;
  TRG_CU(launch_persistent(ctx, (const void*)k_calibrate, b->group * m, kTile, args, cal_smem));
  ctx->launches += 2;
  return TRG_OK;
}

}  // namespace trg

// ------------------------------------------------------------ sharded build
namespace trg {

// The segmented build over a comm's shards (device-resident clouds, one per
// local shard).  trees[i] receives shard i's (identical) tree.
int build_sharded_dev(trg_comm* c, const double* const* dev, const size_t* n,
                      const trg_model_config* cfg, trg_tree_dev** trees, trg_build_diag* diag) {
  const int S = c->local;
  const int L = cfg->max_level;
  std::vector<BuildAlloc> al(S);
  for (int i = 0; i < S; ++i) al[i] = initial_alloc(c->shard_ctx[i], std::max<size_t>(n[i], 1), L);
  const int XP = cfg->em_iterations_per_node + 10;  // exchange points per round
  const int nseg = L * XP + 1;
  for (int attempt = 0; attempt < 4; ++attempt) {
    std::vector<BuildJob> job(S);
    for (int i = 0; i < S; ++i)
      TRG_TRY(build_prepare(c->shard_ctx[i], dev[i], n[i], cfg, al[i], i == 0 ? diag : nullptr,
                            c->world, &job[i]));
    std::vector<double*> red(S), xa(S), xaa(S), xc(S);
    for (int i = 0; i < S; ++i) {
      red[i] = job[i].p.nodered;
      xa[i] = job[i].p.xarg;
      xaa[i] = job[i].p.xarg_all;
      xc[i] = job[i].p.xcal;
    }
    // Exchanges are sized to the live nodes: the round's expanding nodes K_r
    // (read back once per round, after the segment that ran the previous
    // round's layout) and the tree's J for the calibration.
    size_t kr = 1;
    for (int q = 0; q < nseg; ++q) {
      for (int i = 0; i < S; ++i) TRG_TRY(build_launch(c->shard_ctx[i], &job[i], q));
      if (q + 1 == nseg) break;
      if (q % XP == 0 && q > 0) {
        int k2 = 0;
        TRG_CU(cudaMemcpyAsync(&k2, &job[0].p.st->Kp[(q / XP) & 1], sizeof(int),
                               cudaMemcpyDeviceToHost, c->shard_ctx[0]->stream));
        TRG_CU(cudaStreamSynchronize(c->shard_ctx[0]->stream));
        kr = (size_t)std::max(0, std::min(k2, job[0].p.Kmax));
      }
      TRG_TRY(comm_allreduce_sum(c, red.data(), kr * kRec));
      if (q % XP <= 7) TRG_TRY(comm_allgather(c, xa.data(), xaa.data(), (size_t)job[0].p.Kmax * 8));  // mom1 / FPS
    }
    int jn = 0;
    TRG_CU(cudaMemcpyAsync(&jn, &job[0].p.st->J, sizeof(int), cudaMemcpyDeviceToHost,
                           c->shard_ctx[0]->stream));
    TRG_CU(cudaStreamSynchronize(c->shard_ctx[0]->stream));
    const size_t nj = (size_t)std::max(0, std::min(jn, job[0].p.capacity));
    for (int s = 0; s <= 40; ++s) {
      for (int i = 0; i < S; ++i) TRG_TRY(calibrate_launch(c->shard_ctx[i], &job[i], s));
      if (s < 40) TRG_TRY(comm_allreduce_sum(c, xc.data(), nj * 10));
    }
    // consensus on errors / overflow (a shard that overflowed stopped early,
    // so the others' results are void too)
    std::vector<double> v((size_t)S * 6, 0.0);
    std::vector<int> rc(S);
    std::vector<bool> ovf(S);
    std::vector<BuildAlloc> need(S);
    std::vector<unsigned long long> eround((size_t)S * 8, 0);
    for (int i = 0; i < S; ++i) {
      bool o = false;
      need[i] = al[i];
      trg_build_diag d{};
      rc[i] = build_collect(c->shard_ctx[i], &job[i], cfg, &trees[i], i == 0 ? diag : &d, &o,
                            &need[i]);
      const trg_build_diag& di = i == 0 && diag ? *diag : d;
      for (int r = 0; r < 8; ++r) eround[(size_t)i * 8 + r] = di.entries_per_round[r];
      ovf[i] = o;
      v[(size_t)i * 6 + 0] = o ? 1.0 : 0.0;
      v[(size_t)i * 6 + 1] = rc[i] != TRG_OK ? (double)rc[i] : 0.0;
      v[(size_t)i * 6 + 2] = (double)need[i].Emax / (double)std::max<size_t>(n[i], 1);
      v[(size_t)i * 6 + 3] = (double)need[i].Kmax;
    }
    TRG_TRY(comm_host_reduce(c, v.data(), 6, 1));
    const bool any_ovf = v[0] > 0.0;
    if (!any_ovf && v[1] > 0.0) {
      int mine = TRG_OK;
      for (int i = 0; i < S; ++i)
        if (rc[i] != TRG_OK) mine = rc[i];
      for (int i = 0; i < S; ++i)
        if (rc[i] == TRG_OK && trees[i]) trg_tree_free(c->shard_ctx[i], trees[i]);
      if (mine == TRG_OK) {
        set_error("build_tree (sharded): another shard failed");
        return (int)v[1];
      }
      return mine;
    }
    if (!any_ovf) {
      if (diag) {
        std::vector<double> e((size_t)S * 8);
        for (size_t k = 0; k < e.size(); ++k) e[k] = (double)eround[k];
        TRG_TRY(comm_host_reduce(c, e.data(), 8, 0));
        for (int r = 0; r < 8; ++r) diag->entries_per_round[r] = (unsigned long long)e[r];
      }
      return TRG_OK;
    }
    for (int i = 0; i < S; ++i) {
      if (!ovf[i] && rc[i] == TRG_OK && trees[i]) trg_tree_free(c->shard_ctx[i], trees[i]);
      trees[i] = nullptr;
      trg_ctx* cx = c->shard_ctx[i];
      const double ratio = std::max(v[2], (double)need[i].Emax / (double)std::max<size_t>(n[i], 1));
      cx->build_growth = std::max(cx->build_growth, 1.25 * ratio);
      al[i].Emax = (int)std::min<double>((double)INT32_MAX / 16,
                                         std::max<double>(2.0 * al[i].Emax, 1.25 * ratio * (double)n[i] + 1024.0));
      al[i].Kmax = std::max(al[i].Kmax, (int)v[3]);
      al[i].Tmax = al[i].Emax / kTile + al[i].Kmax + 8;
    }
  }
  set_error("build_tree (sharded): entry buffer growth did not converge");
  return TRG_ERUNTIME;
}

}  // namespace trg

extern "C" int trg_build_tree_sharded(trg_comm* comm, const double* const* xyz, const size_t* n,
                                      int on_device, const trg_model_config* cfg,
                                      trg_tree_dev** out, trg_build_diag* diag) {
  trg::NvtxRange nvtx_range_("trg_build_tree_sharded");
  if (!comm || !xyz || !n || !out) {
    set_error("build_tree_sharded: bad argument");
    return TRG_EINVAL;
  }
  TRG_TRY(validate_model_config(cfg));
  const int S = comm->local;
  std::vector<double> tot((size_t)S, 0.0);
  for (int i = 0; i < S; ++i) {
    if (n[i] > (size_t)INT32_MAX / 8) {
      set_error("point cloud too large for int32 entry indexing");
      return TRG_EINVAL;
    }
    tot[i] = (double)n[i];
  }
  TRG_TRY(comm_host_reduce(comm, tot.data(), 1, 0));
  if (!(tot[0] > 0.0)) {
    set_error("point cloud is empty");
    return TRG_EINVAL;
  }
  TRG_CU(cudaSetDevice(comm->ctx->device));
  std::vector<const double*> dev(S);
  for (int i = 0; i < S; ++i)
    TRG_TRY(stage_points_public(comm->shard_ctx[i], xyz[i], n[i], on_device, kSlotPoints, &dev[i]));
  std::vector<trg_tree_dev*> trees(S, nullptr);
  TRG_TRY(build_sharded_dev(comm, dev.data(), n, cfg, trees.data(), diag));
  for (int i = 1; i < S; ++i) trg_tree_free(comm->shard_ctx[i], trees[i]);
  *out = trees[0];
  return TRG_OK;
}
