// The flat-mixture variant ("GMM J=n"): build_flat_gmm
// (gmm.cpp:659-736) and responsibilities_dense (association.cpp:54-89).
//
// k_flat_build: ONE persistent launch.  list_moments (two passes) ->
// D^2-weighted seeding (one seed per step: the CTA-0 search over per-CTA
// block sums + a block scan inside the chosen block; the reference's
// mt19937_64 stream reproduced on the device) -> J components at
// sigma^2 I -> em_iterations_per_node * max_level EM iterations, each: a
// point-major pass (warp per point, lanes over components, online
// log-sum-exp) writing the per-point log normaliser, then a component-major
// pass (lane per component, warps over point chunks) accumulating the
// centred moments, a fixed-order chunk reduction and the M-step (one thread
// per component).  No float atomics.
//
// Dense association (K12): pass 1 per point (warp, lanes over components)
// sums w_j N(y; j); pass 2 per component (lane) deposits gamma = score/sum
// into the epoch-stamped partial rows the tree path uses, so the same
// per-node combine and the registration M-step (k_register<true>) follow.
#include <cub/block/block_scan.cuh>

#include "trg_dense.cuh"
#include "trg_gmm.cuh"

namespace trg {

// ------------------------------------------------- mt19937_64 + libstdc++
// std::mt19937_64 and the libstdc++ (GCC 13) distributions the reference
// draws from: uniform_int_distribution<size_t> (Lemire's nearly divisionless
// downscaling, uniform_int_dist.h) and generate_canonical<double, 53> (one
// 64-bit draw / 2^64).  State lives in global memory; one thread draws.
struct Mt64 {
  unsigned long long mt[312];
  unsigned long long idx;
};

__device__ void mt_seed(Mt64* s, unsigned long long seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    s->mt[i] = 6364136223846793005ull * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (unsigned long long)i;
  s->idx = 312;
}

__device__ unsigned long long mt_next(Mt64* s) {
  if (s->idx >= 312) {
    const unsigned long long up = 0xFFFFFFFF80000000ull, lo = 0x7FFFFFFFull;
    for (int i = 0; i < 312; ++i) {
      const unsigned long long x = (s->mt[i] & up) | (s->mt[(i + 1) % 312] & lo);
      unsigned long long xa = x >> 1;
      if (x & 1ull) xa ^= 0xB5026F5AA96619E9ull;
      s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
    }
    s->idx = 0;
  }
  unsigned long long y = s->mt[s->idx++];
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= y >> 43;
  return y;
}

// uniform_int_distribution<size_t>(0, n - 1)(mt19937_64)
__device__ unsigned long long mt_index(Mt64* s, unsigned long long n) {
  const unsigned long long range = n;  // urange + 1
  unsigned long long g = mt_next(s);
  unsigned long long low = g * range, high = __umul64hi(g, range);
  if (low < range) {
    const unsigned long long threshold = (0ull - range) % range;
    while (low < threshold) {
      g = mt_next(s);
      low = g * range;
      high = __umul64hi(g, range);
    }
  }
  return high;
}

// generate_canonical<double, 53>(mt19937_64)
__device__ double mt_canonical(Mt64* s) {
  const double r = __ull2double_rn(mt_next(s)) / 18446744073709551616.0;
  return r >= 1.0 ? 0.99999999999999988898 : r;
}

// ------------------------------------------------------------------ build
struct FlatParams {
  const double* pts;  // N x 3 AoS
  size_t n;
  int J, iters;
  double eps, abs_floor;
  unsigned long long seed;
  DNode* nodes;      // [J] output mixture (flat: J roots)
  double* cov;       // [J][9]
  double* lw;        // [J] log weight (-inf when dormant)
  double* min_d2;    // [N]
  double* lt;        // [N] log normaliser per point (-inf: skipped)
  double* blk;       // [G][16] per-CTA partials
  double* part;      // [nchunks][J][10]
  double* acc;       // [J][10]
  double* seeds;     // [J][3]
  double* scal;      // [32] shared scalars
  double* ll_trace;  // [iters]
  Mt64* rng;
  unsigned* bar;
  int* status;
};

constexpr int kFB = 256;

// Deterministic block sum of NV doubles (fixed shuffle tree + warp order).
template <int NV>
__device__ void fblock_sum(double v[NV], double (*ws)[NV], double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < NV; ++k) ws[warp][k] = v[k];
  __syncthreads();
  if (threadIdx.x < NV) {
    double s = 0.0;
    for (int w = 0; w < kFB / 32; ++w) s += ws[w][threadIdx.x];
    out[threadIdx.x] = s;
  }
  __syncthreads();
}

// log w + log_density (gmm.cpp:37-47, 176-178) of component k at x.
__device__ __forceinline__ double flat_logp(const FlatParams& p, int k, double x0, double x1,
                                            double x2) {
  const double lwk = p.lw[k];
  if (!(lwk > -INFINITY)) return -INFINITY;
  const DNode& g = p.nodes[k];
  const double q = fast_q(g.mean, g.prec, x0, x1, x2);
  return lwk + __fma_rn(-0.5, q, g.log_norm);
}

__device__ __forceinline__ double sqd(const double* a, double x0, double x1, double x2) {
  const double d0 = x0 - a[0], d1 = x1 - a[1], d2 = x2 - a[2];
  double s = d0 * d0;
  s += d1 * d1;
  s += d2 * d2;
  return s;  // Eigen squaredNorm order
}

__global__ void __launch_bounds__(kFB, 2) k_flat_build(FlatParams p) {
  __shared__ double ws[kFB / 32][8];
  __shared__ double red[8];
  __shared__ double sref[3], smean[3];
  __shared__ typename cub::BlockScan<double, kFB>::TempStorage scan;
  __shared__ int s_found;
  const int G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const size_t n = p.n;
  const int J = p.J;
  const size_t per = (n + G - 1) / G;
  const size_t b0 = min(n, (size_t)cta * per), b1 = min(n, b0 + per);
  // ---------------- list_moments (gmm.cpp:92-136): ref = first point
  if (tid < 3) sref[tid] = p.pts[tid];
  __syncthreads();
  {
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    for (size_t i = b0 + tid; i < b1; i += kFB) {
      v[0] += 1.0;
      v[1] += p.pts[3 * i] - sref[0];
      v[2] += p.pts[3 * i + 1] - sref[1];
      v[3] += p.pts[3 * i + 2] - sref[2];
    }
    fblock_sum<4>(v, (double(*)[4])ws, red);
    if (tid < 4) p.blk[(size_t)cta * 16 + tid] = red[tid];
  }
  grid_sync(p.bar, G);
  if (tid == 0) {
    double m = 0.0, s1[3] = {0.0, 0.0, 0.0};
    for (int c = 0; c < G; ++c) {
      m += __ldcg(p.blk + (size_t)c * 16);
      for (int k = 0; k < 3; ++k) s1[k] += __ldcg(p.blk + (size_t)c * 16 + 1 + k);
    }
    for (int k = 0; k < 3; ++k) smean[k] = sref[k] + s1[k] / m;
    red[7] = m;
  }
  __syncthreads();
  const double mass = red[7];
  {
    double v[6] = {0, 0, 0, 0, 0, 0};
    for (size_t i = b0 + tid; i < b1; i += kFB) {
      const double d0 = p.pts[3 * i] - smean[0], d1 = p.pts[3 * i + 1] - smean[1],
                   d2 = p.pts[3 * i + 2] - smean[2];
      v[0] += d0 * d0;
      v[1] += d0 * d1;
      v[2] += d0 * d2;
      v[3] += d1 * d1;
      v[4] += d1 * d2;
      v[5] += d2 * d2;
    }
    __syncthreads();
    fblock_sum<6>(v, (double(*)[6])ws, red);
    if (tid < 6) p.blk[(size_t)cta * 16 + 4 + tid] = red[tid];
  }
  grid_sync(p.bar, G);
  // every CTA folds the same partials in the same order
  if (tid == 0) {
    double m2[6] = {0, 0, 0, 0, 0, 0};
    for (int c = 0; c < G; ++c)
      for (int k = 0; k < 6; ++k) m2[k] += __ldcg(p.blk + (size_t)c * 16 + 4 + k);
    const double S[3][3] = {{m2[0] / mass, m2[1] / mass, m2[2] / mass},
                            {m2[1] / mass, m2[3] / mass, m2[4] / mass},
                            {m2[2] / mass, m2[4] / mass, m2[5] / mass}};
    red[6] = cov_floor(S, p.eps, p.abs_floor);
    if (cta == 0)
      for (int k = 0; k < 3; ++k) p.scal[1 + k] = smean[k];
  }
  __syncthreads();
  const double floor_value = red[6];
  // ---------------- seeding (gmm.cpp:679-711)
  Mt64* rng = p.rng;
  if (cta == 0 && tid == 0) {
    mt_seed(rng, p.seed);
    const unsigned long long first = mt_index(rng, n);
    for (int k = 0; k < 3; ++k) p.seeds[k] = p.pts[3 * first + k];
  }
  grid_sync(p.bar, G);
  {
    const double s0[3] = {__ldcg(p.seeds), __ldcg(p.seeds + 1), __ldcg(p.seeds + 2)};
    double v[1] = {0.0};
    for (size_t i = b0 + tid; i < b1; i += kFB) {
      const double d = sqd(s0, p.pts[3 * i], p.pts[3 * i + 1], p.pts[3 * i + 2]);
      p.min_d2[i] = d;
      v[0] += d;
    }
    fblock_sum<1>(v, (double(*)[1])ws, red);
    if (tid == 0) p.blk[(size_t)cta * 16 + 10] = red[0];
  }
  grid_sync(p.bar, G);
  for (int k = 1; k < J; ++k) {
    if (cta == 0) {
      // total over the block sums in block order; draw; find the block
      if (tid == 0) {
        double total = 0.0;
        for (int c = 0; c < G; ++c) total += __ldcg(p.blk + (size_t)c * 16 + 10);
        long long chosen = -1;
        int b = -1;
        double t = 0.0;
        if (total > 0.0) {
          t = mt_canonical(rng) * total;  // uniform_real_distribution(0, total)
          for (int c = 0; c < G; ++c) {
            const double t2 = t - __ldcg(p.blk + (size_t)c * 16 + 10);
            if (t2 <= 0.0) {
              b = c;
              break;
            }
            t = t2;
          }
          if (b < 0) chosen = (long long)n - 1;
        } else {
          chosen = (long long)mt_index(rng, n);
        }
        red[0] = (double)chosen;
        red[1] = (double)b;
        red[2] = t;
      }
      __syncthreads();
      long long chosen = (long long)red[0];
      const int b = (int)red[1];
      if (chosen < 0 && b >= 0) {
        // first index in block b where the running target drops to <= 0
        const size_t c0 = min(n, (size_t)b * per), c1 = min(n, c0 + per);
        double t = red[2];
        chosen = (long long)c1 - 1;
        for (size_t base = c0; base < c1; base += kFB) {
          const size_t i = base + tid;
          const double d = i < c1 ? __ldcg(p.min_d2 + i) : 0.0;
          double pre, tot;
          cub::BlockScan<double, kFB>(scan).InclusiveSum(d, pre, tot);
          if (tid == 0) s_found = kFB;
          __syncthreads();
          if (i < c1 && t - pre <= 0.0) atomicMin(&s_found, tid);
          __syncthreads();
          if (s_found < kFB) {
            chosen = (long long)(base + s_found);
            break;
          }
          t -= tot;
          __syncthreads();
        }
      }
      if (tid == 0)
        for (int q = 0; q < 3; ++q) p.seeds[3 * k + q] = p.pts[3 * chosen + q];
    }
    grid_sync(p.bar, G);
    {
      const double sk[3] = {__ldcg(p.seeds + 3 * k), __ldcg(p.seeds + 3 * k + 1),
                            __ldcg(p.seeds + 3 * k + 2)};
      double v[1] = {0.0};
      for (size_t i = b0 + tid; i < b1; i += kFB) {
        const double d = sqd(sk, p.pts[3 * i], p.pts[3 * i + 1], p.pts[3 * i + 2]);
        const double m = smin(p.min_d2[i], d);
        p.min_d2[i] = m;
        v[0] += m;
      }
      fblock_sum<1>(v, (double(*)[1])ws, red);
      if (tid == 0) p.blk[(size_t)cta * 16 + 10] = red[0];
    }
    grid_sync(p.bar, G);
  }
  // sigma^2 = max(mean_d2 / 3, floor); components at sigma^2 I (gmm.cpp:712-722)
  if (tid == 0) {
    double s = 0.0;
    for (int c = 0; c < G; ++c) s += __ldcg(p.blk + (size_t)c * 16 + 10);
    red[5] = smax((s / (double)n) / 3.0, floor_value);
  }
  __syncthreads();
  const double sigma2 = red[5];
  for (int k = cta * kFB + tid; k < J; k += G * kFB) {
    double* c9 = p.cov + 9 * (size_t)k;
    for (int q = 0; q < 9; ++q) c9[q] = (q % 4 == 0) ? sigma2 : 0.0;
    DNode& d = p.nodes[k];
    for (int q = 0; q < 3; ++q) d.mean[q] = p.seeds[3 * k + q];
    d.weight = 1.0 / (double)J;
    d.pad = 0.0;
    d.first_child = -1;
    d.child_count = 0;
    d.level = 0;
    d.parent = -1;
    if (refresh_node(d, c9)) atomicCAS(p.status, 0, kEInval);
    p.lw[k] = log(d.weight);
  }
  grid_sync(p.bar, G);
  // ---------------- EM (run_em_iterations, gmm.cpp:225-242) about ref = mean
  const int nw = G * (kFB / 32), gw = cta * (kFB / 32) + warp;
  const int nb = (J + 31) / 32;
  const int nchunks = max(1, min(nw / nb, (int)((n + 7) / 8)));
  for (int it = 0; it < p.iters; ++it) {
    // pass 1: log normaliser per point (online log-sum-exp over the lanes)
    double ll = 0.0;
    for (size_t i = gw; i < n; i += nw) {
      const double x0 = p.pts[3 * i], x1 = p.pts[3 * i + 1], x2 = p.pts[3 * i + 2];
      double m = -INFINITY, s = 0.0;
      for (int k = lane; k < J; k += 32) {
        const double lg = flat_logp(p, k, x0, x1, x2);
        if (!(lg > -INFINITY)) continue;
        if (lg > m) {
          s = s * trg_exp(m - lg) + 1.0;
          m = lg;
        } else {
          s += trg_exp(lg - m);
        }
      }
      double M = m;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) M = fmax(M, __shfl_xor_sync(0xffffffffu, M, o));
      double sl = (m > -INFINITY) ? s * trg_exp(m - M) : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sl += __shfl_xor_sync(0xffffffffu, sl, o);
      const double ltot = isfinite(M) ? M + log(sl) : -INFINITY;
      if (lane == 0) {
        p.lt[i] = ltot;
        if (isfinite(M)) ll += ltot;  // entries carry w = 1
      }
    }
    {
      double v[1] = {ll};
      fblock_sum<1>(v, (double(*)[1])ws, red);
      if (tid == 0) p.blk[(size_t)cta * 16 + 11] = red[0];
    }
    grid_sync(p.bar, G);
    // pass 2: centred moments, lane per component, warps over point chunks
    {
      const double r0 = __ldcg(p.scal + 1), r1 = __ldcg(p.scal + 2), r2 = __ldcg(p.scal + 3);
      const int cb = gw % nb, chunk = gw / nb;
      if (chunk < nchunks) {
        const int k = cb * 32 + lane;
        const size_t c0 = (n * (size_t)chunk) / nchunks, c1 = (n * (size_t)(chunk + 1)) / nchunks;
        double a[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
        if (k < J) {
          for (size_t i = c0; i < c1; ++i) {
            const double lti = __ldcg(p.lt + i);
            if (!(lti > -INFINITY)) continue;
            const double x0 = p.pts[3 * i], x1 = p.pts[3 * i + 1], x2 = p.pts[3 * i + 2];
            const double lg = flat_logp(p, k, x0, x1, x2);
            const double g = lg > -INFINITY ? trg_exp(lg - lti) : 0.0;
            if (!(g > 0.0)) continue;
            const double d0 = x0 - r0, d1 = x1 - r1, d2 = x2 - r2;
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
          }
          double* o = p.part + ((size_t)chunk * J + k) * 10;
          for (int q = 0; q < 10; ++q) o[q] = a[q];
        }
      }
    }
    grid_sync(p.bar, G);
    // chunk reduction, fixed order
    for (int k = cta * kFB + tid; k < J; k += G * kFB) {
      double a[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
      for (int c = 0; c < nchunks; ++c)
        for (int q = 0; q < 10; ++q) a[q] += __ldcg(p.part + ((size_t)c * J + k) * 10 + q);
      for (int q = 0; q < 10; ++q) p.acc[(size_t)k * 10 + q] = a[q];
    }
    grid_sync(p.bar, G);
    // M-step (gmm.cpp:209-223): one thread per component
    {
      __shared__ double s_total;
      if (tid == 0) {
        double t = 0.0;
        for (int k = 0; k < J; ++k) t += __ldcg(p.acc + (size_t)k * 10);
        s_total = t;
        if (cta == 0) {
          double l = 0.0;
          for (int c = 0; c < G; ++c) l += __ldcg(p.blk + (size_t)c * 16 + 11);
          p.ll_trace[it] = l;
          if (!(t > 0.0)) atomicCAS(p.status, 0, kERuntime);  // m_step: no responsibility mass
        }
      }
      __syncthreads();
      const double total = s_total;
      const double r[3] = {__ldcg(p.scal + 1), __ldcg(p.scal + 2), __ldcg(p.scal + 3)};
      for (int k = cta * kFB + tid; k < J; k += G * kFB) {
        double a[10];
        for (int q = 0; q < 10; ++q) a[q] = __ldcg(p.acc + (size_t)k * 10 + q);
        if (!(total > 0.0)) continue;
        DNode& d = p.nodes[k];
        if (a[0] <= total * 1e-12) {  // dormant: weight 0, parameters kept
          d.weight = 0.0;
          p.lw[k] = -INFINITY;
          continue;
        }
        const double mu[3] = {a[1] / a[0], a[2] / a[0], a[3] / a[0]};
        const double M[3][3] = {{a[4], a[5], a[6]}, {a[5], a[7], a[8]}, {a[6], a[8], a[9]}};
        double S[3][3];
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) S[i][j] = M[i][j] / a[0] - mu[i] * mu[j];
        GComp g;
        g.w = a[0] / total;
        for (int i = 0; i < 3; ++i) g.mean[i] = r[i] + mu[i];
        if (comp_set_cov(g, S, floor_value)) atomicCAS(p.status, 0, kEInval);
        write_dnode_from_comp(d, p.cov + 9 * (size_t)k, g, g.w, 0, -1);
        p.lw[k] = log(g.w);
      }
    }
    grid_sync(p.bar, G);
  }
  if (cta == 0 && tid == 0) {
    p.scal[0] = mass;
    p.scal[4] = floor_value;
    p.scal[5] = sigma2;
  }
}

template <int NM>
__global__ void __launch_bounds__(256) k_dense(DenseParams p, const double* Rt_dev, unsigned* bar) {
  __shared__ double rt[12];
  if (Rt_dev && threadIdx.x < 12) rt[threadIdx.x] = Rt_dev[threadIdx.x];
  __syncthreads();
  const double* Rt = Rt_dev ? rt : nullptr;
  dense_pass1(p, Rt, gridDim.x, blockIdx.x);
  grid_sync(bar, gridDim.x);
  dense_pass2<NM>(p, Rt, gridDim.x, blockIdx.x);
}

template __global__ void k_dense<4>(DenseParams, const double*, unsigned*);
template __global__ void k_dense<10>(DenseParams, const double*, unsigned*);

}  // namespace trg

// ------------------------------------------------------------------ host
namespace trg {

int flat_build(trg_ctx* ctx, const double* dev, size_t n, size_t J, const trg_model_config* cfg,
               trg_tree_dev** out, trg_build_diag* diag) {
  TRG_TRY(check_model_config(cfg));
  if (n == 0) {
    set_error("point cloud is empty");
    return TRG_EINVAL;
  }
  if (J < 1 || J > n) {  // gmm.cpp:665-667
    set_error("component count out of range");
    return TRG_EINVAL;
  }
  if (J > (size_t)INT32_MAX / 64) {
    set_error("component count too large");
    return TRG_EINVAL;
  }
  TRG_CU(cudaSetDevice(ctx->device));
  const int G = persistent_grid(ctx, (const void*)k_flat_build, kFB, 0);
  const int iters = cfg->em_iterations_per_node * cfg->max_level;
  const size_t nw = (size_t)G * (kFB / 32);
  size_t off = 0;
  auto carve = [&](size_t bytes) {
    const size_t o = off;
    off += (bytes + 255) & ~size_t(255);
    return o;
  };
  const size_t o_lw = carve(8 * J), o_md = carve(8 * n), o_lt = carve(8 * n),
               o_blk = carve(8 * 16 * (size_t)G), o_part = carve(8 * 10 * J * nw),
               o_acc = carve(8 * 10 * J), o_seed = carve(8 * 3 * J), o_scal = carve(8 * 32),
               o_llt = carve(8 * (size_t)std::max(iters, 1)), o_rng = carve(sizeof(Mt64)),
               o_bar = carve(64);
  void* arena = nullptr;
  TRG_TRY(ws_get(ctx, kSlotBuild1, off, &arena));
  char* A = static_cast<char*>(arena);
  trg_tree_dev* tree = nullptr;
  TRG_TRY(tree_alloc(ctx, (int)J, &tree));
  FlatParams p{};
  p.pts = dev;
  p.n = n;
  p.J = (int)J;
  p.iters = iters;
  p.eps = cfg->cov_regularization_epsilon;
  p.abs_floor = cfg->cov_regularization_absolute;
  p.seed = cfg->rng_seed;
  p.nodes = tree->nodes;
  p.cov = tree->cov;
  p.lw = (double*)(A + o_lw);
  p.min_d2 = (double*)(A + o_md);
  p.lt = (double*)(A + o_lt);
  p.blk = (double*)(A + o_blk);
  p.part = (double*)(A + o_part);
  p.acc = (double*)(A + o_acc);
  p.seeds = (double*)(A + o_seed);
  p.scal = (double*)(A + o_scal);
  p.ll_trace = (double*)(A + o_llt);
  p.rng = (Mt64*)(A + o_rng);
  p.bar = (unsigned*)(A + o_bar);
  p.status = ctx->status;
  TRG_CU(cudaMemsetAsync(A + o_bar, 0, 64, ctx->stream));
  void* args[] = {&p};
  TRG_CU(launch_persistent(ctx, (const void*)k_flat_build, G, kFB, args));
  ctx->launches += 1;
  int rc = check_status(ctx, "build_flat_gmm");
  if (rc != TRG_OK) {
    trg_tree_free(ctx, tree);
    return rc;
  }
  tree->n_nodes = (int)J;
  tree->max_level = 1;
  tree->root_count = (int)J;
  if (diag) {
    double* traces = diag->ll_traces;
    const int tcap = diag->ll_trace_capacity;
    *diag = trg_build_diag{};
    diag->entries_per_round[0] = n;
    diag->expanded_per_round[0] = 1;
    diag->n_expansions = 0;
    diag->ll_traces = traces;
    diag->ll_trace_capacity = tcap;
    if (traces && iters > 0 &&
        (size_t)tcap * (size_t)(cfg->em_iterations_per_node + 1) >= (size_t)iters) {
      TRG_CU(cudaMemcpyAsync(traces, p.ll_trace, sizeof(double) * (size_t)iters,
                             cudaMemcpyDeviceToHost, ctx->stream));
      TRG_CU(cudaStreamSynchronize(ctx->stream));
      diag->flat_trace_len = iters;
    }
  }
  *out = tree;
  return TRG_OK;
}

}  // namespace trg

using namespace trg;

extern "C" int trg_build_flat_gmm(trg_ctx* ctx, const double* xyz, size_t n, int xyz_on_device,
                                  size_t J, const trg_model_config* cfg, trg_tree_dev** out,
                                  trg_build_diag* diag) {
  trg::NvtxRange nvtx_range_("trg_build_flat_gmm");
  if (!ctx || !cfg || !out) {
    set_error("build_flat_gmm: bad argument");
    return TRG_EINVAL;
  }
  if (n == 0 || !xyz) {
    set_error("point cloud is empty");
    return TRG_EINVAL;
  }
  TRG_CU(cudaSetDevice(ctx->device));
  const double* dev = nullptr;
  TRG_TRY(stage_points_public(ctx, xyz, n, xyz_on_device, kSlotPoints, &dev));
  TRG_TRY(check_finite_dev(ctx, dev, n, "point cloud has non-finite coordinates"));
  return flat_build(ctx, dev, n, J, cfg, out, diag);
}

extern "C" int trg_responsibilities_dense(trg_ctx* ctx, const trg_tree_dev* comps, const double* xyz,
                                          size_t n, int xyz_on_device, const double R[9],
                                          const double t[3], double outlier_floor,
                                          trg_moments* out) {
  trg::NvtxRange nvtx_range_("trg_responsibilities_dense");
  // association.cpp:43-50 validate_inputs
  if (n == 0 || !xyz) {
    set_error("association: empty point cloud");
    return TRG_EINVAL;
  }
  if (!comps || comps->n_nodes == 0) {
    set_error("association: empty model");
    return TRG_EINVAL;
  }
  TRG_CU(cudaSetDevice(ctx->device));
  const int nm = out->m2 ? 10 : 4;
  const int J = comps->n_nodes;
  const void* kern = nm == 4 ? (const void*)k_dense<4> : (const void*)k_dense<10>;
  const int G = persistent_grid(ctx, kern, 256, 0);
  const double* pts = nullptr;
  TRG_TRY(stage_points_public(ctx, xyz, n, xyz_on_device, kSlotPoints, &pts));
  TRG_TRY(check_finite_dev(ctx, pts, n, "association: non-finite point"));
  void *part, *stamps, *mom, *cnt, *ps;
  TRG_TRY(ws_get(ctx, kSlotPartials, sizeof(double) * nm * (size_t)J * G, &part));
  TRG_TRY(ws_get(ctx, kSlotStamps, sizeof(uint32_t) * (size_t)J * G, &stamps));
  TRG_TRY(ws_get(ctx, kSlotMoments, sizeof(double) * nm * (size_t)J, &mom));
  TRG_TRY(ws_get(ctx, kSlotCounters, 64 + 12 * sizeof(double) + 64, &cnt));
  TRG_TRY(ws_get(ctx, kSlotDense, sizeof(double) * n, &ps));
  double* rt = reinterpret_cast<double*>(static_cast<char*>(cnt) + 64);
  unsigned* bar = reinterpret_cast<unsigned*>(static_cast<char*>(cnt) + 64 + 12 * sizeof(double));
  double hrt[12];
  for (int k = 0; k < 9; ++k) hrt[k] = R[k];
  for (int k = 0; k < 3; ++k) hrt[9 + k] = t[k];
  TRG_CU(trg_memcpy(ctx, rt, hrt, sizeof hrt, cudaMemcpyHostToDevice));
  TRG_CU(cudaMemsetAsync(cnt, 0, 64, ctx->stream));
  TRG_CU(cudaMemsetAsync(bar, 0, 64, ctx->stream));
  DenseParams p{};
  p.pts = pts;
  p.n = n;
  p.comps = comps->nodes;
  p.J = J;
  p.outlier_floor = outlier_floor;
  p.psum = static_cast<double*>(ps);
  p.partials = static_cast<double*>(part);
  p.stamps = static_cast<uint32_t*>(stamps);
  p.epoch = ++ctx->epoch;
  p.counters = static_cast<unsigned long long*>(cnt);
  p.status = ctx->status;
  const double* rtc = rt;
  void* args[] = {&p, &rtc, &bar};
  TRG_CU(launch_persistent(ctx, kern, G, 256, args));
  ctx->launches += 1;
  TRG_TRY(launch_combine(ctx, p.partials, p.stamps, p.epoch, G, J, nm, static_cast<double*>(mom)));
  std::vector<double> hm((size_t)nm * J);
  unsigned long long hc[2];
  TRG_CU(trg_memcpy(ctx, hm.data(), mom, sizeof(double) * nm * J, cudaMemcpyDeviceToHost));
  TRG_CU(trg_memcpy(ctx, hc, cnt, sizeof hc, cudaMemcpyDeviceToHost));
  TRG_TRY(check_status(ctx, "responsibilities_dense"));
  double mass = 0.0;
  for (int j = 0; j < J; ++j) {
    const double* v = &hm[(size_t)nm * j];
    out->m0[j] = v[0];
    for (int k = 0; k < 3; ++k) out->m1[3 * j + k] = v[1 + k];
    if (nm == 10) {
      double* m2 = out->m2 + 9 * j;
      m2[0] = v[4];
      m2[1] = m2[3] = v[5];
      m2[2] = m2[6] = v[6];
      m2[4] = v[7];
      m2[5] = m2[7] = v[8];
      m2[8] = v[9];
    }
    mass += v[0];
  }
  out->total_points = n;
  out->outliers = hc[0];
  out->density_evaluations = hc[1];
  out->total_mass = mass;
  return TRG_OK;
}
