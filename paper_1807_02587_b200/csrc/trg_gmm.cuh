// Shared device pieces of the GMM fits (tree build and flat mixture):
// the component record of a fit and the set_floored_cov / refresh_eig
// updates of gmm.cpp, writing the tree's DNode layout.
#pragma once
#include "trg_solve.cuh"

namespace trg {

// One mixture component during a node fit (gmm.hpp:12-23 + log weight).
struct GComp {
  double w, lw;
  double mean[3];
  double axT[9];
  double lam[3];
  double log_norm;
  double cov[9];
  double il[3];  // 1 / lam
  double prec[6];  // precision matrix for fast_q (set_prec)
};
static_assert(sizeof(GComp) == 288, "GComp layout");

// set_floored_cov (gmm.cpp:143-150) into a GComp.
static __device__ __noinline__ int comp_set_cov(GComp& g, const double sc[3][3], double floor_value,
                                            const double* warm = nullptr) {
  double lam[3], ax[3][3], cov[3][3];
  const int rc = eig_sym3_floored(sc, floor_value, lam, ax, warm);
  if (rc) return rc;
  reconstruct(lam, ax, cov);
  for (int i = 0; i < 3; ++i) {
    g.lam[i] = lam[i];
    g.il[i] = 1.0 / lam[i];
    for (int j = 0; j < 3; ++j) {
      g.axT[3 * i + j] = ax[j][i];
      g.cov[3 * i + j] = cov[i][j];
    }
  }
  g.log_norm = log_norm_of(lam);
  set_prec(g.axT, g.il, g.prec);
  return kOk;
}

__device__ __forceinline__ void write_dnode_from_comp(DNode& d, double* cov9, const GComp& g,
                                                      double w, int level, int parent) {
  for (int i = 0; i < 3; ++i) d.mean[i] = g.mean[i];
  for (int i = 0; i < 9; ++i) {
    d.axT[i] = g.axT[i];
    cov9[i] = g.cov[i];
  }
  for (int i = 0; i < 3; ++i) {
    d.lam[i] = g.lam[i];
    d.il[i] = 1.0 / g.lam[i];
  }
  for (int i = 0; i < 6; ++i) d.prec[i] = g.prec[i];
  d.pad = 0.0;
  d.log_norm = g.log_norm;
  d.weight = w;
  const double tr = (g.lam[0] + g.lam[1]) + g.lam[2];
  d.cplx = tr > 0.0 ? g.lam[2] / tr : -1.0;
  d.first_child = -1;
  d.child_count = 0;
  d.level = level;
  d.parent = parent;
}

// refresh_eig (gmm.cpp:31-35) of a tree node from its cov.
// warm: start the eigensolve from the node's current axes (calibration).
static __device__ __noinline__ int refresh_node(DNode& d, const double* cov9, bool warm = false) {
  double m[3][3], lam[3], ax[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) m[i][j] = cov9[3 * i + j];
  double w[9];
  if (warm)
    for (int i = 0; i < 9; ++i) w[i] = d.axT[i];
  const int rc = eig_sym3(m, lam, ax, warm ? w : nullptr);
  if (rc) return rc;
  for (int i = 0; i < 3; ++i) {
    d.lam[i] = lam[i];
    d.il[i] = 1.0 / lam[i];
    for (int j = 0; j < 3; ++j) d.axT[3 * i + j] = ax[j][i];
  }
  d.log_norm = log_norm_of(lam);
  set_prec(d.axT, d.il, d.prec);
  const double tr = (lam[0] + lam[1]) + lam[2];
  d.cplx = tr > 0.0 ? lam[2] / tr : -1.0;
  return kOk;
}

// Closed-form variants (trg_math.cuh eig_sym3*_cf): set_floored_cov of the
// M-steps and leaf refits, refresh_eig of the calibration's parents.  No
// warp collectives: any set of lanes may call.
__device__ __forceinline__ int comp_set_cov_cf(GComp& g, const double sc[3][3], double floor_value) {
  double lam[3], ax[3][3], cov[3][3];
  const int rc = eig_sym3_floored_cf(sc, floor_value, lam, ax);
  reconstruct(lam, ax, cov);
  for (int i = 0; i < 3; ++i) {
    g.lam[i] = lam[i];
    g.il[i] = 1.0 / lam[i];
    for (int j = 0; j < 3; ++j) {
      g.axT[3 * i + j] = ax[j][i];
      g.cov[3 * i + j] = cov[i][j];
    }
  }
  g.log_norm = log_norm_of(lam);
  set_prec(g.axT, g.il, g.prec);
  return rc;
}

// refresh_eig of a node from cov9 into its DNode fields (written only when
// `act` and the eigensolve succeeded).
__device__ __forceinline__ int refresh_node_cf(DNode& d, const double* cov9, bool act) {
  double m[3][3], lam[3], ax[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) m[i][j] = act ? cov9[3 * i + j] : (i == j ? 1.0 : 0.0);
  const int rc = eig_sym3_cf(m, lam, ax);
  if (!act || rc) return act ? rc : kOk;
  for (int i = 0; i < 3; ++i) {
    d.lam[i] = lam[i];
    d.il[i] = 1.0 / lam[i];
    for (int j = 0; j < 3; ++j) d.axT[3 * i + j] = ax[j][i];
  }
  d.log_norm = log_norm_of(lam);
  set_prec(d.axT, d.il, d.prec);
  const double tr = (lam[0] + lam[1]) + lam[2];
  d.cplx = tr > 0.0 ? lam[2] / tr : -1.0;
  return kOk;
}

}  // namespace trg
