// Point-to-point ICP (register_icp_pt2pt, registration.cpp:211-298; SURVEY
// 8f rank 4: the side-by-side comparator).  ONE persistent launch for all
// iterations: per iteration every CTA matches its chunk of source points by
// an exact brute-force nearest-neighbour scan of the target cloud, staged
// through shared memory in tiles (squared distances in the reference's
// Eigen order, no FMA; the scan is in index order with a strict '<', so
// ties resolve to the lowest index exactly like KdTree3::nearest,
// kdtree.hpp:15); the cross-covariance sums are reduced per CTA and folded
// by every CTA in the same order; each CTA takes the Kabsch rotation from
// the same 3x3 SVD (the oracle shim's JacobiSVD: V from the eigenvectors of
// H^T H, U = H V / sigma) and updates the transform redundantly.  A second
// reduction gives the criterion after the update.  2 grid barriers per
// iteration, no host round trip.
#include "trg_solve.cuh"

namespace trg {

constexpr int kIcpBlock = 256;
constexpr int kIcpTile = 1024;  // target points per shared-memory tile
constexpr int kIcpAcc = 16;     // sum_y[3], sum_q[3], sum_yq[9], sq_dist

struct IcpState {
  double Rt[12];
  double trans_limit;
  int iterations, converged, done, pad;
};

struct IcpParams {
  const double* src;  // N_s x 3
  const double* tgt;  // N_t x 3
  size_t ns, nt;
  int max_iters;
  double rot_tol;
  IcpState* st;
  unsigned* corr;     // [N_s]
  double* part;       // [G][kIcpAcc]
  double* crit_before;
  double* crit_after;
  unsigned* bar;
};

// y = R p + t in the reference's order (geometry.hpp:31)
__device__ __forceinline__ void icp_apply(const double* Rt, double p0, double p1, double p2,
                                          double y[3]) {
  for (int i = 0; i < 3; ++i) {
    double s = __dmul_rn(Rt[3 * i], p0);
    s = __dadd_rn(s, __dmul_rn(Rt[3 * i + 1], p1));
    s = __dadd_rn(s, __dmul_rn(Rt[3 * i + 2], p2));
    y[i] = __dadd_rn(s, Rt[9 + i]);
  }
}

// (q - y).squaredNorm() in Eigen's order, no contraction
__device__ __forceinline__ double icp_d2(double dx, double dy, double dz) {
  return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
}

// Kabsch rotation of H = sum y q^T - n yc qc^T (registration.cpp:255-262)
// via the shim's JacobiSVD (oracle/shim/Eigen/Core:749-774).
__device__ void icp_rotation(const double H[3][3], double R[3][3]) {
  double ata[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double s = 0.0;
      for (int k = 0; k < 3; ++k) s += H[k][i] * H[k][j];
      ata[i][j] = s;
    }
  double ev[3], vec[3][3];
  jacobi_eig<3>(ata, ev, vec);  // ascending, sign-normalised columns
  double V[3][3], U[3][3], sv[3];
  for (int c = 0; c < 3; ++c) {
    const int k = 2 - c;
    sv[c] = sqrt(smax(ev[k], 0.0));
    for (int r = 0; r < 3; ++r) V[r][c] = vec[r][k];
  }
  for (int c = 0; c < 3; ++c) {
    double u[3];
    for (int r = 0; r < 3; ++r) u[r] = H[r][0] * V[0][c] + H[r][1] * V[1][c] + H[r][2] * V[2][c];
    const double n = sqrt(u[0] * u[0] + u[1] * u[1] + u[2] * u[2]);
    if (n > 1e-300 * (sv[0] + 1e-300) && n > 0.0) {
      for (int r = 0; r < 3; ++r) U[r][c] = u[r] / n;
    } else {  // Gram-Schmidt completion with unit vectors
      for (int e = 0; e < 3; ++e) {
        double cand[3] = {e == 0 ? 1.0 : 0.0, e == 1 ? 1.0 : 0.0, e == 2 ? 1.0 : 0.0};
        for (int q = 0; q < c; ++q) {
          const double d = cand[0] * U[0][q] + cand[1] * U[1][q] + cand[2] * U[2][q];
          for (int r = 0; r < 3; ++r) cand[r] -= U[r][q] * d;
        }
        const double cn = sqrt(cand[0] * cand[0] + cand[1] * cand[1] + cand[2] * cand[2]);
        if (cn > 1e-6) {
          for (int r = 0; r < 3; ++r) U[r][c] = cand[r] / cn;
          break;
        }
      }
    }
  }
  // r = V U^T, flipped in the last singular direction when det < 0
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) R[i][j] = V[i][0] * U[j][0] + V[i][1] * U[j][1] + V[i][2] * U[j][2];
  if (det33(R) < 0.0)
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) R[i][j] = V[i][0] * U[j][0] + V[i][1] * U[j][1] - V[i][2] * U[j][2];
}

__global__ void __launch_bounds__(kIcpBlock, 2) k_icp(IcpParams p) {
  __shared__ double tx[kIcpTile], ty[kIcpTile], tz[kIcpTile];
  __shared__ double rt[12];
  __shared__ double red[kIcpBlock / 32][kIcpAcc];
  __shared__ double fold[kIcpAcc + 1];
  __shared__ int s_done;
  const int G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  if (tid < 12) rt[tid] = __ldcg(&p.st->Rt[tid]);
  if (tid == 0) s_done = 0;
  __syncthreads();
  const double trans_limit = __ldcg(&p.st->trans_limit);
  const size_t per = (p.ns + G - 1) / G;
  const size_t b0 = min(p.ns, (size_t)cta * per), b1 = min(p.ns, b0 + per);
  const double dn = (double)p.ns;
  for (int it = 0; it < p.max_iters; ++it) {
    // ---- correspondences (exact NN) + per-CTA sums
    double acc[kIcpAcc];
#pragma unroll
    for (int k = 0; k < kIcpAcc; ++k) acc[k] = 0.0;
    for (size_t base = b0; base < b1; base += kIcpBlock) {
      const size_t i = base + tid;
      const bool act = i < b1;
      double y[3] = {0.0, 0.0, 0.0};
      if (act) icp_apply(rt, p.src[3 * i], p.src[3 * i + 1], p.src[3 * i + 2], y);
      double best = INFINITY;
      unsigned bi = 0;
      for (size_t t0 = 0; t0 < p.nt; t0 += kIcpTile) {
        const int tl = (int)min((size_t)kIcpTile, p.nt - t0);
        __syncthreads();
        for (int q = tid; q < tl; q += kIcpBlock) {
          tx[q] = p.tgt[3 * (t0 + q)];
          ty[q] = p.tgt[3 * (t0 + q) + 1];
          tz[q] = p.tgt[3 * (t0 + q) + 2];
        }
        __syncthreads();
        if (act)
          for (int q = 0; q < tl; ++q) {
            const double d2 = icp_d2(y[0] - tx[q], y[1] - ty[q], y[2] - tz[q]);
            if (d2 < best) {
              best = d2;
              bi = (unsigned)(t0 + q);
            }
          }
      }
      if (act) {
        p.corr[i] = bi;
        const double q0 = p.tgt[3 * (size_t)bi], q1 = p.tgt[3 * (size_t)bi + 1], q2 = p.tgt[3 * (size_t)bi + 2];
        const double q[3] = {q0, q1, q2};
        for (int k = 0; k < 3; ++k) {
          acc[k] += y[k];
          acc[3 + k] += q[k];
        }
        for (int r = 0; r < 3; ++r)
          for (int c = 0; c < 3; ++c) acc[6 + 3 * r + c] += y[r] * q[c];
        acc[15] += icp_d2(y[0] - q0, y[1] - q1, y[2] - q2);
      }
    }
    // block reduce (fixed butterfly + warp order) -> this CTA's partial row
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int k = 0; k < kIcpAcc; ++k) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], o);
    if (lane == 0)
      for (int k = 0; k < kIcpAcc; ++k) red[warp][k] = acc[k];
    __syncthreads();
    if (tid < kIcpAcc) {
      double s = 0.0;
      for (int w = 0; w < kIcpBlock / 32; ++w) s += red[w][tid];
      p.part[(size_t)cta * kIcpAcc + tid] = s;
    }
    grid_sync(p.bar, G);
    // ---- every CTA folds the rows in CTA order and solves (identical bits)
    if (tid < kIcpAcc) {
      double s = 0.0;
      for (int c = 0; c < G; ++c) s += __ldcg(p.part + (size_t)c * kIcpAcc + tid);
      fold[tid] = s;
    }
    __syncthreads();
    double dR[3][3], dt[3];
    {
      const double yc[3] = {fold[0] / dn, fold[1] / dn, fold[2] / dn};
      const double qc[3] = {fold[3] / dn, fold[4] / dn, fold[5] / dn};
      double H[3][3];
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) H[r][c] = fold[6 + 3 * r + c] - dn * (yc[r] * qc[c]);
      icp_rotation(H, dR);
      for (int r = 0; r < 3; ++r) dt[r] = qc[r] - (dR[r][0] * yc[0] + dR[r][1] * yc[1] + dR[r][2] * yc[2]);
    }
    // criterion after the update over the same correspondences
    double after = 0.0;
    for (size_t i = b0 + tid; i < b1; i += kIcpBlock) {
      double y[3], z[3];
      icp_apply(rt, p.src[3 * i], p.src[3 * i + 1], p.src[3 * i + 2], y);
      for (int r = 0; r < 3; ++r)
        z[r] = dR[r][0] * y[0] + dR[r][1] * y[1] + dR[r][2] * y[2] + dt[r];
      const unsigned bi = p.corr[i];
      after += icp_d2(z[0] - p.tgt[3 * (size_t)bi], z[1] - p.tgt[3 * (size_t)bi + 1],
                      z[2] - p.tgt[3 * (size_t)bi + 2]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) after += __shfl_xor_sync(0xffffffffu, after, o);
    __syncthreads();
    if (lane == 0) red[warp][0] = after;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int w = 0; w < kIcpBlock / 32; ++w) s += red[w][0];
      p.part[(size_t)G * kIcpAcc + cta] = s;  // after-criterion row
    }
    grid_sync(p.bar, G);
    if (tid == 0) {
      if (cta == 0) {
        double s = 0.0;
        for (int c = 0; c < G; ++c) s += __ldcg(p.part + (size_t)G * kIcpAcc + c);
        p.crit_before[it] = fold[15] / dn;
        p.crit_after[it] = s / dn;
      }
      // T = delta * T (geometry.hpp:42-47); convergence (registration.cpp:289-293)
      double nR[9], nt[3];
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
          double q = dR[i][0] * rt[j];
          q += dR[i][1] * rt[3 + j];
          q += dR[i][2] * rt[6 + j];
          nR[3 * i + j] = q;
        }
      for (int i = 0; i < 3; ++i) {
        double q = dR[i][0] * rt[9];
        q += dR[i][1] * rt[10];
        q += dR[i][2] * rt[11];
        nt[i] = q + dt[i];
      }
      for (int k = 0; k < 9; ++k) rt[k] = nR[k];
      for (int k = 0; k < 3; ++k) rt[9 + k] = nt[k];
      double cth = ((dR[0][0] + dR[1][1]) + dR[2][2] - 1.0) * 0.5;
      cth = cth < -1.0 ? -1.0 : (cth > 1.0 ? 1.0 : cth);
      const double tn = sqrt(dt[0] * dt[0] + dt[1] * dt[1] + dt[2] * dt[2]);
      if (acos(cth) < p.rot_tol && tn < trans_limit) s_done = 1;
      if (cta == 0) {
        p.st->iterations = it + 1;
        p.st->converged = s_done;
        for (int k = 0; k < 12; ++k) p.st->Rt[k] = rt[k];
      }
    }
    __syncthreads();
    if (s_done) break;
  }
}


// register_icp_pt2pt (registration.cpp:211-298) on device-resident clouds.
int register_icp_dev(trg_ctx* ctx, const double* tgt, size_t nt, const double* src, size_t ns,
                         const trg_reg_config* cfg, double diag, trg_reg_result* out) {
  const int G = persistent_grid(ctx, (const void*)k_icp, kIcpBlock, 0);
  const int K = cfg->max_em_iterations;
  void *corr, *part, *em, *tr;
  TRG_TRY(ws_get(ctx, kSlotPointNode, sizeof(unsigned) * std::max<size_t>(ns, 1), &corr));
  TRG_TRY(ws_get(ctx, kSlotPartials, sizeof(double) * ((size_t)G * kIcpAcc + G), &part));
  TRG_TRY(ws_get(ctx, kSlotEm, 256 + sizeof(IcpState), &em));
  TRG_TRY(ws_get(ctx, kSlotEmTrace, sizeof(double) * 2 * (size_t)K, &tr));
  IcpParams p{};
  p.src = src;
  p.tgt = tgt;
  p.ns = ns;
  p.nt = nt;
  p.max_iters = K;
  p.rot_tol = cfg->rotation_tol;
  p.bar = static_cast<unsigned*>(em);
  p.st = reinterpret_cast<IcpState*>(static_cast<char*>(em) + 64);
  p.corr = static_cast<unsigned*>(corr);
  p.part = static_cast<double*>(part);
  p.crit_before = static_cast<double*>(tr);
  p.crit_after = p.crit_before + K;
  IcpState st{};
  for (int k = 0; k < 9; ++k) st.Rt[k] = cfg->initial_R[k];
  for (int k = 0; k < 3; ++k) st.Rt[9 + k] = cfg->initial_t[k];
  st.trans_limit = cfg->translation_tol * diag;  // registration.cpp:221
  TRG_CU(cudaMemsetAsync(em, 0, 64, ctx->stream));
  TRG_CU(trg_memcpy(ctx, p.st, &st, sizeof st, cudaMemcpyHostToDevice));
  cudaEvent_t e0, e1;
  TRG_CU(cudaEventCreate(&e0));
  TRG_CU(cudaEventCreate(&e1));
  TRG_CU(cudaEventRecord(e0, ctx->stream));
  void* args[] = {&p};
  TRG_CU(launch_persistent(ctx, (const void*)k_icp, G, kIcpBlock, args));
  ctx->launches += 1;
  TRG_CU(cudaEventRecord(e1, ctx->stream));
  TRG_CU(trg_memcpy(ctx, &st, p.st, sizeof st, cudaMemcpyDeviceToHost));
  std::vector<double> cb(K), ca(K);
  TRG_CU(trg_memcpy(ctx, cb.data(), p.crit_before, sizeof(double) * K, cudaMemcpyDeviceToHost));
  TRG_CU(trg_memcpy(ctx, ca.data(), p.crit_after, sizeof(double) * K, cudaMemcpyDeviceToHost));
  TRG_CU(cudaEventSynchronize(e1));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  TRG_TRY(check_status(ctx, "register_icp_pt2pt"));
  for (int k = 0; k < 9; ++k) out->R[k] = st.Rt[k];
  for (int k = 0; k < 3; ++k) out->t[k] = st.Rt[9 + k];
  out->iterations = st.iterations;
  out->converged = st.converged;
  out->em_seconds = ms * 1e-3;
  out->model_build_seconds = 0.0;  // no model: the brute-force scan needs no index
  out->model_components = nt;
  const int m = std::min(st.iterations, out->trace_capacity);
  for (int i = 0; i < m; ++i) {
    if (out->criterion_trace) out->criterion_trace[i] = cb[i];
    if (out->criterion_after_trace) out->criterion_after_trace[i] = ca[i];
    if (out->eval_counts) out->eval_counts[i] = 0;  // registration.cpp:268
  }
  return TRG_OK;
}

}  // namespace trg
