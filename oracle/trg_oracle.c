/* TEST INFRASTRUCTURE ONLY — CPU restatement of the reference hot path.
 * See trg_oracle.h for scope.  Every function cites the reference lines it
 * restates; "shim order" means the evaluation order of oracle/shim/Eigen/Core
 * (products and sums left to right, norms over column-major storage).
 * Compiled with -ffp-contract=off (no FMA), like the reference's Release
 * build without -march. */
#include "trg_oracle.h"

#include <math.h>
#include <setjmp.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define CHUNK 4096 /* parallel.hpp:28 kChunkSize */
static const double kLog2Pi = 1.8378770664093453; /* gmm.cpp:18 */
static const double kMembershipTruncation = 1e-12; /* gmm.cpp:23 */
static const int kCalibrationPassLimit = 40;       /* gmm.cpp:28 */

static _Thread_local jmp_buf g_jmp;
static _Thread_local int g_code;
static _Thread_local char g_msg[256];

static void fail(int code, const char* msg) {
  g_code = code;
  snprintf(g_msg, sizeof g_msg, "%s", msg);
  longjmp(g_jmp, 1);
}
const char* trgo_last_error(void) { return g_msg; }

/* std::max / std::min semantics */
static inline double smax(double a, double b) { return (a < b) ? b : a; }
static inline double smin(double a, double b) { return (b < a) ? b : a; }

typedef struct {
  double w;
  double mean[3];
  double cov[3][3];
  double lam[3];
  double ax[3][3]; /* ax[r][c]: column c is the axis for lam[c] */
  double log_norm;
} comp_t;

/* ------------------------------------------------------------- 3x3 algebra */

/* Frobenius norm in column-major storage order (shim squaredNorm). */
static double norm33(const double m[3][3]) {
  double s = m[0][0] * m[0][0];
  for (int j = 0; j < 3; ++j)
    for (int i = 0; i < 3; ++i) {
      if (i == 0 && j == 0) continue;
      s += m[i][j] * m[i][j];
    }
  return sqrt(s);
}
static double norm3(const double v[3]) {
  double s = v[0] * v[0];
  s += v[1] * v[1];
  s += v[2] * v[2];
  return sqrt(s);
}
static double dot3(const double a[3], const double b[3]) {
  double s = a[0] * b[0];
  s += a[1] * b[1];
  s += a[2] * b[2];
  return s;
}
static void matmul33(const double a[3][3], const double b[3][3], double c[3][3]) {
  double t[3][3];
  for (int j = 0; j < 3; ++j)
    for (int i = 0; i < 3; ++i) {
      double s = a[i][0] * b[0][j];
      s += a[i][1] * b[1][j];
      s += a[i][2] * b[2][j];
      t[i][j] = s;
    }
  memcpy(c, t, sizeof t);
}
static double det33(const double g[3][3]) { /* shim determinant() */
  return g[0][0] * (g[1][1] * g[2][2] - g[2][1] * g[1][2]) -
         g[1][0] * (g[0][1] * g[2][2] - g[2][1] * g[0][2]) +
         g[2][0] * (g[0][1] * g[1][2] - g[1][1] * g[0][2]);
}
static int all_finite33(const double m[3][3]) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      if (!isfinite(m[i][j])) return 0;
  return 1;
}

/* Cyclic Jacobi, shim internal::jacobi_eig<N> (the oracle's stand-in for
 * Eigen::SelfAdjointEigenSolver). Eigenvalues ascending, vectors as
 * columns of v_out, sign: largest-|.| entry positive. */
static void jacobi_n(int n, const double* in /* row-major n*n */, double* evals, double* evecs /* row-major, col c = vec */) {
  double a[6][6], v[6][6];
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      a[i][j] = in[i * n + j];
      v[i][j] = (i == j) ? 1.0 : 0.0;
    }
  for (int sweep = 0; sweep < 64; ++sweep) {
    int rotated = 0;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = a[p][q];
        if (apq == 0.0) continue;
        const double app = a[p][p], aqq = a[q][q];
        const double g = 100.0 * fabs(apq);
        if (fabs(app) + g == fabs(app) && fabs(aqq) + g == fabs(aqq)) {
          a[p][q] = 0.0;
          a[q][p] = 0.0;
          continue;
        }
        rotated = 1;
        const double h = aqq - app;
        double t;
        if (fabs(h) + g == fabs(h)) {
          t = apq / h;
        } else {
          const double theta = 0.5 * h / apq;
          t = 1.0 / (fabs(theta) + sqrt(1.0 + theta * theta));
          if (theta < 0.0) t = -t;
        }
        const double c = 1.0 / sqrt(1.0 + t * t);
        const double s = t * c;
        const double tau = s / (1.0 + c);
        a[p][p] = app - t * apq;
        a[q][q] = aqq + t * apq;
        a[p][q] = 0.0;
        a[q][p] = 0.0;
        for (int r = 0; r < n; ++r) {
          if (r == p || r == q) continue;
          const double arp = a[r][p], arq = a[r][q];
          const double np = arp - s * (arq + arp * tau);
          const double nq = arq + s * (arp - arq * tau);
          a[r][p] = np;
          a[p][r] = np;
          a[r][q] = nq;
          a[q][r] = nq;
        }
        for (int r = 0; r < n; ++r) {
          const double vrp = v[r][p], vrq = v[r][q];
          v[r][p] = vrp - s * (vrq + vrp * tau);
          v[r][q] = vrq + s * (vrp - vrq * tau);
        }
      }
    if (!rotated) break;
  }
  int order[6];
  for (int i = 0; i < n; ++i) order[i] = i;
  for (int i = 1; i < n; ++i) {
    const int k = order[i];
    int j = i - 1;
    while (j >= 0 && a[order[j]][order[j]] > a[k][k]) {
      order[j + 1] = order[j];
      --j;
    }
    order[j + 1] = k;
  }
  for (int c = 0; c < n; ++c) {
    const int k = order[c];
    evals[c] = a[k][k];
    int big = 0;
    for (int r = 1; r < n; ++r)
      if (fabs(v[r][k]) > fabs(v[big][k])) big = r;
    const double sg = v[big][k] < 0.0 ? -1.0 : 1.0;
    for (int r = 0; r < n; ++r) evecs[r * n + c] = sg * v[r][k];
  }
}

/* geometry.cpp:40-79 eig_sym3 (strict) */
static void eig_sym3(const double m[3][3], double lam[3], double ax[3][3]) {
  if (!all_finite33(m)) fail(1, "eig_sym3: non-finite input matrix");
  const double scale = norm33(m);
  double d[3][3], sym[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) d[i][j] = m[i][j] - m[j][i];
  const double asym = norm33(d);
  if (asym > 1e-6 * smax(scale, 1e-300)) fail(1, "eig_sym3: matrix is not symmetric");
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) sym[i][j] = 0.5 * (m[i][j] + m[j][i]);
  double ev[3], vec[9];
  jacobi_n(3, &sym[0][0], ev, vec);
  for (int l = 0; l < 3; ++l) {
    lam[l] = ev[2 - l];
    for (int r = 0; r < 3; ++r) ax[r][l] = vec[r * 3 + (2 - l)];
  }
  const double neg_floor = -1e-10 * scale;
  for (int l = 0; l < 3; ++l)
    if (lam[l] < 0.0) {
      if (lam[l] < neg_floor) fail(1, "eig_sym3: strongly negative eigenvalue (corrupted covariance)");
      lam[l] = 0.0;
    }
  if (det33(ax) < 0.0)
    for (int r = 0; r < 3; ++r) ax[r][2] = -ax[r][2];
}

/* geometry.cpp:81-102 eig_sym3_floored */
static void eig_sym3_floored(const double m[3][3], double floor_value, double lam[3], double ax[3][3]) {
  if (!all_finite33(m)) fail(1, "eig_sym3_floored: non-finite input matrix");
  if (!(floor_value > 0.0)) fail(1, "eig_sym3_floored: floor must be positive");
  double sym[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) sym[i][j] = 0.5 * (m[i][j] + m[j][i]);
  double ev[3], vec[9];
  jacobi_n(3, &sym[0][0], ev, vec);
  for (int l = 0; l < 3; ++l) {
    lam[l] = smax(ev[2 - l], floor_value);
    for (int r = 0; r < 3; ++r) ax[r][l] = vec[r * 3 + (2 - l)];
  }
  if (det33(ax) < 0.0)
    for (int r = 0; r < 3; ++r) ax[r][2] = -ax[r][2];
}

/* geometry.hpp:18-20 EigenDecomp3::reconstruct = axes * diag(lam) * axes^T (shim order) */
static void reconstruct(const double lam[3], const double ax[3][3], double cov[3][3]) {
  double dg[3][3] = {{lam[0], 0, 0}, {0, lam[1], 0}, {0, 0, lam[2]}};
  double ad[3][3], axt[3][3];
  matmul33(ax, dg, ad);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) axt[i][j] = ax[j][i];
  matmul33(ad, axt, cov);
}

static double log_norm_of(const double lam[3]) { /* gmm.cpp:33-34, 148-149 */
  return -0.5 * (3.0 * kLog2Pi + log(lam[0]) + log(lam[1]) + log(lam[2]));
}

/* gmm.cpp:31-35 refresh_eig */
static void refresh_eig(comp_t* g) {
  eig_sym3(g->cov, g->lam, g->ax);
  g->log_norm = log_norm_of(g->lam);
}

/* gmm.cpp:143-150 set_floored_cov */
static void set_floored_cov(comp_t* g, const double scatter[3][3], double floor_value) {
  double lam[3], ax[3][3];
  eig_sym3_floored(scatter, floor_value, lam, ax);
  reconstruct(lam, ax, g->cov);
  memcpy(g->lam, lam, sizeof lam);
  memcpy(g->ax, ax, sizeof ax);
  g->log_norm = log_norm_of(lam);
}

/* gmm.cpp:152-155 cov_floor */
static double cov_floor(const double s[3][3], const trgo_model_cfg* cfg) {
  const double tr = s[0][0] + s[1][1] + s[2][2];
  return smax(cfg->abs_floor, cfg->eps * tr / 3.0);
}

/* gmm.cpp:37-47 log_density (shim order for axes^T d) */
static inline double log_density(const comp_t* g, const double x[3]) {
  if (!(g->lam[2] > 0.0)) fail(2, "log_density: covariance is not positive definite");
  const double d0 = x[0] - g->mean[0], d1 = x[1] - g->mean[1], d2 = x[2] - g->mean[2];
  double p[3];
  for (int l = 0; l < 3; ++l) {
    double s = g->ax[0][l] * d0;
    s += g->ax[1][l] * d1;
    s += g->ax[2][l] * d2;
    p[l] = s;
  }
  const double q = p[0] * p[0] / g->lam[0] + p[1] * p[1] / g->lam[1] + p[2] * p[2] / g->lam[2];
  return g->log_norm - 0.5 * q;
}

/* gmm.cpp:53-59 node_complexity */
static double node_complexity(const double lam[3]) {
  const double tr = (lam[0] + lam[1]) + lam[2];
  if (!(tr > 0.0)) fail(2, "node_complexity: covariance has no positive trace");
  return lam[2] / tr;
}

/* ------------------------------------------------------------ tree build */

typedef struct {
  size_t idx;
  double w;
} entry_t; /* gmm.cpp:73-76 */

typedef struct {
  double m0, m1[3], m2[3][3];
} accum_t; /* gmm.cpp:78-88 */

typedef struct {
  const double* pts;
  const trgo_model_cfg* cfg;
  trgo_build_stats* stats;
} bctx;

#define PT(c, i, k) ((c)->pts[3 * (i) + (k)])

/* gmm.cpp:92-137 list_moments */
static void list_moments(const bctx* c, const entry_t* e, size_t n, double* mass, double mean[3], double cov[3][3]) {
  if (n == 0) fail(1, "list_moments: empty point list");
  double ref[3] = {PT(c, e[0].idx, 0), PT(c, e[0].idx, 1), PT(c, e[0].idx, 2)};
  double tm = 0.0, tm1[3] = {0, 0, 0};
  for (size_t b = 0; b < n; b += CHUNK) {
    const size_t end = b + CHUNK < n ? b + CHUNK : n;
    double m0 = 0.0, m1[3] = {0, 0, 0};
    for (size_t i = b; i < end; ++i) {
      m0 += e[i].w;
      for (int k = 0; k < 3; ++k) m1[k] = m1[k] + e[i].w * (PT(c, e[i].idx, k) - ref[k]);
    }
    tm += m0;
    for (int k = 0; k < 3; ++k) tm1[k] = tm1[k] + m1[k];
  }
  *mass = tm;
  if (!(tm > 0.0)) fail(1, "list_moments: point list has no mass");
  for (int k = 0; k < 3; ++k) mean[k] = ref[k] + tm1[k] / tm;
  double tc[3][3] = {{0}};
  for (size_t b = 0; b < n; b += CHUNK) {
    const size_t end = b + CHUNK < n ? b + CHUNK : n;
    double m2[3][3] = {{0}};
    for (size_t i = b; i < end; ++i) {
      double d[3];
      for (int k = 0; k < 3; ++k) d[k] = PT(c, e[i].idx, k) - mean[k];
      for (int r = 0; r < 3; ++r)
        for (int s = 0; s < 3; ++s) m2[r][s] = m2[r][s] + e[i].w * (d[r] * d[s]);
    }
    for (int r = 0; r < 3; ++r)
      for (int s = 0; s < 3; ++s) tc[r][s] = tc[r][s] + m2[r][s];
  }
  for (int r = 0; r < 3; ++r)
    for (int s = 0; s < 3; ++s) cov[r][s] = tc[r][s] / tm;
}

/* Log-terms of one entry under the 8 components (gmm.cpp:174-184); returns 0 if not finite. */
static int entry_logs(const comp_t* comps, const double lw[8], const double x[3], double logs[8], double* log_total) {
  double m = -INFINITY;
  for (int k = 0; k < 8; ++k) {
    logs[k] = comps[k].w > 0.0 ? lw[k] + log_density(&comps[k], x) : -INFINITY;
    m = smax(m, logs[k]);
  }
  if (!isfinite(m)) return 0;
  double s = 0.0;
  for (int k = 0; k < 8; ++k) s += exp(logs[k] - m);
  *log_total = m + log(s);
  return 1;
}

/* gmm.cpp:159-206 e_step_moments (8 components, moments about ref) */
static double e_step_moments(const bctx* c, const entry_t* e, size_t n, const comp_t* comps, const double ref[3],
                             accum_t acc[8]) {
  double lw[8];
  for (int k = 0; k < 8; ++k) lw[k] = comps[k].w > 0.0 ? log(comps[k].w) : 0.0;
  memset(acc, 0, sizeof(accum_t) * 8);
  double ll = 0.0;
  for (size_t b = 0; b < n; b += CHUNK) {
    const size_t end = b + CHUNK < n ? b + CHUNK : n;
    accum_t local[8];
    memset(local, 0, sizeof local);
    double cll = 0.0;
    for (size_t i = b; i < end; ++i) {
      const double x[3] = {PT(c, e[i].idx, 0), PT(c, e[i].idx, 1), PT(c, e[i].idx, 2)};
      double logs[8], lt;
      if (!entry_logs(comps, lw, x, logs, &lt)) continue;
      cll += e[i].w * lt;
      const double d[3] = {x[0] - ref[0], x[1] - ref[1], x[2] - ref[2]};
      double outer[3][3];
      for (int r = 0; r < 3; ++r)
        for (int s = 0; s < 3; ++s) outer[r][s] = d[r] * d[s];
      for (int k = 0; k < 8; ++k) {
        const double g = exp(logs[k] - lt) * e[i].w;
        if (g <= 0.0) continue;
        local[k].m0 += g;
        for (int r = 0; r < 3; ++r) local[k].m1[r] = local[k].m1[r] + g * d[r];
        for (int r = 0; r < 3; ++r)
          for (int s = 0; s < 3; ++s) local[k].m2[r][s] = local[k].m2[r][s] + g * outer[r][s];
      }
    }
    ll += cll;
    for (int k = 0; k < 8; ++k) {
      acc[k].m0 += local[k].m0;
      for (int r = 0; r < 3; ++r) acc[k].m1[r] = acc[k].m1[r] + local[k].m1[r];
      for (int r = 0; r < 3; ++r)
        for (int s = 0; s < 3; ++s) acc[k].m2[r][s] = acc[k].m2[r][s] + local[k].m2[r][s];
    }
  }
  return ll;
}

/* gmm.cpp:211-230 m_step */
static void m_step(const accum_t acc[8], const double ref[3], double floor_value, comp_t comps[8]) {
  double total = 0.0;
  for (int k = 0; k < 8; ++k) total += acc[k].m0;
  if (!(total > 0.0)) fail(3, "m_step: no responsibility mass");
  for (int k = 0; k < 8; ++k) {
    const accum_t* a = &acc[k];
    if (a->m0 <= total * 1e-12) {
      comps[k].w = 0.0;
      continue;
    }
    double d[3], sc[3][3];
    for (int r = 0; r < 3; ++r) d[r] = a->m1[r] / a->m0;
    for (int r = 0; r < 3; ++r)
      for (int s = 0; s < 3; ++s) sc[r][s] = a->m2[r][s] / a->m0 - d[r] * d[s];
    comps[k].w = a->m0 / total;
    for (int r = 0; r < 3; ++r) comps[k].mean[r] = ref[r] + d[r];
    set_floored_cov(&comps[k], sc, floor_value);
  }
}

/* gmm.cpp:248-261 corner_seeds */
static void corner_seeds(const double mean[3], const double scatter[3][3], double floor_value, double seeds[8][3]) {
  double lam[3], ax[3][3];
  eig_sym3_floored(scatter, floor_value, lam, ax);
  for (int c = 0; c < 8; ++c) {
    double off[3] = {0, 0, 0};
    for (int l = 0; l < 3; ++l) {
      const double sign = ((c >> l) & 1) != 0 ? 1.0 : -1.0;
      const double s = sign * 0.5 * sqrt(lam[l]);
      for (int k = 0; k < 3; ++k) off[k] = off[k] + s * ax[k][l];
    }
    for (int k = 0; k < 3; ++k) seeds[c][k] = mean[k] + off[k];
  }
}

static inline double d2pt(const bctx* c, size_t idx, const double s[3]) {
  const double a = PT(c, idx, 0) - s[0], b = PT(c, idx, 1) - s[1], d = PT(c, idx, 2) - s[2];
  double r = a * a;
  r += b * b;
  r += d * d;
  return r;
}

/* gmm.cpp:267-303 farthest_point_seeds */
static void farthest_point_seeds(const bctx* c, const entry_t* e, size_t n, double seeds[8][3]) {
  size_t first = 0;
  for (size_t i = 1; i < n; ++i)
    if (e[i].w > e[first].w) first = i;
  for (int k = 0; k < 3; ++k) seeds[0][k] = PT(c, e[first].idx, k);
  int ns = 1;
  double* min_d2 = (double*)malloc(sizeof(double) * n);
  for (size_t i = 0; i < n; ++i) min_d2[i] = d2pt(c, e[i].idx, seeds[0]);
  while (ns < 8) {
    size_t best = 0;
    double best_score = -1.0;
    for (size_t i = 0; i < n; ++i) {
      const double score = e[i].w * min_d2[i];
      if (score > best_score) {
        best_score = score;
        best = i;
      }
    }
    if (!(best_score > 0.0)) {
      memcpy(seeds[ns++], seeds[0], sizeof(double) * 3);
      continue;
    }
    for (int k = 0; k < 3; ++k) seeds[ns][k] = PT(c, e[best].idx, k);
    ++ns;
    for (size_t i = 0; i < n; ++i) min_d2[i] = smin(min_d2[i], d2pt(c, e[i].idx, seeds[ns - 1]));
  }
  free(min_d2);
}

typedef struct {
  comp_t comps[8];
  double* gamma; /* n x 8 */
  double final_ll;
} cand_t;

/* gmm.cpp:314-364 fit_candidate */
static void fit_candidate(const bctx* c, const entry_t* e, size_t n, const double mean[3], const double scatter[3][3],
                          double floor_value, const double seeds[8][3], cand_t* fit) {
  double cs[3][3];
  for (int r = 0; r < 3; ++r)
    for (int s = 0; s < 3; ++s) cs[r][s] = scatter[r][s] / 4.0;
  for (int k = 0; k < 8; ++k) {
    fit->comps[k].w = 1.0 / 8.0;
    memcpy(fit->comps[k].mean, seeds[k], sizeof(double) * 3);
    set_floored_cov(&fit->comps[k], cs, floor_value);
  }
  accum_t acc[8];
  for (int it = 0; it < c->cfg->em_iterations_per_node; ++it) {
    e_step_moments(c, e, n, fit->comps, mean, acc);
    m_step(acc, mean, floor_value, fit->comps);
  }
  fit->gamma = (double*)calloc(n * 8, sizeof(double));
  double lw[8];
  for (int k = 0; k < 8; ++k) lw[k] = fit->comps[k].w > 0.0 ? log(fit->comps[k].w) : 0.0;
  double ll = 0.0;
  for (size_t b = 0; b < n; b += CHUNK) {
    const size_t end = b + CHUNK < n ? b + CHUNK : n;
    double cll = 0.0;
    for (size_t i = b; i < end; ++i) {
      const double x[3] = {PT(c, e[i].idx, 0), PT(c, e[i].idx, 1), PT(c, e[i].idx, 2)};
      double logs[8], lt;
      if (!entry_logs(fit->comps, lw, x, logs, &lt)) continue;
      cll += e[i].w * lt;
      for (int k = 0; k < 8; ++k) fit->gamma[i * 8 + k] = exp(logs[k] - lt);
    }
    ll += cll;
  }
  fit->final_ll = ll;
}

typedef struct {
  int ok, ns;
  comp_t children[8];
  entry_t* child_entries[8];
  size_t child_n[8];
} expansion_t;

/* gmm.cpp:378-463 expand_node */
static void expand_node(const bctx* c, const entry_t* e, size_t n, int must_survive, expansion_t* out) {
  memset(out, 0, sizeof *out);
  double mass, mean[3], scatter[3][3];
  list_moments(c, e, n, &mass, mean, scatter);
  const double floor_value = cov_floor(scatter, c->cfg);
  double seeds[8][3];
  cand_t kept, alt;
  corner_seeds(mean, scatter, floor_value, seeds);
  fit_candidate(c, e, n, mean, scatter, floor_value, seeds, &kept);
  farthest_point_seeds(c, e, n, seeds);
  fit_candidate(c, e, n, mean, scatter, floor_value, seeds, &alt);
  if (alt.final_ll > kept.final_ll) {
    free(kept.gamma);
    kept = alt;
  } else {
    free(alt.gamma);
  }
  const double* gamma = kept.gamma;
  double child_mass[8] = {0};
  for (size_t i = 0; i < n; ++i)
    for (int k = 0; k < 8; ++k) child_mass[k] += e[i].w * gamma[i * 8 + k];
  const double kMinChildMass = 4.0;
  int surv[8], ns = 0;
  for (int k = 0; k < 8; ++k)
    if (child_mass[k] > smax(kMinChildMass, mass * 1e-6)) surv[ns++] = k;
  if (ns == 0) {
    if (!must_survive) {
      free(kept.gamma);
      return;
    }
    int best = 0;
    for (int k = 1; k < 8; ++k)
      if (child_mass[k] > child_mass[best]) best = k;
    surv[ns++] = best;
  }
  double surv_mass[8] = {0};
  size_t cap[8];
  for (int s = 0; s < ns; ++s) {
    cap[s] = 16;
    out->child_entries[s] = (entry_t*)malloc(sizeof(entry_t) * cap[s]);
  }
#define PUSH(s, ix, ww)                                                                              \
  do {                                                                                               \
    if (out->child_n[s] == cap[s]) {                                                                 \
      cap[s] *= 2;                                                                                   \
      out->child_entries[s] = (entry_t*)realloc(out->child_entries[s], sizeof(entry_t) * cap[s]); \
    }                                                                                                \
    out->child_entries[s][out->child_n[s]].idx = (ix);                                               \
    out->child_entries[s][out->child_n[s]].w = (ww);                                                 \
    out->child_n[s]++;                                                                               \
  } while (0)
  for (size_t i = 0; i < n; ++i) {
    double denom = 0.0;
    for (int s = 0; s < ns; ++s) denom += gamma[i * 8 + surv[s]];
    if (denom > 0.0) {
      for (int s = 0; s < ns; ++s) {
        const double g = gamma[i * 8 + surv[s]] / denom;
        if (g < kMembershipTruncation) continue;
        PUSH(s, e[i].idx, e[i].w * g);
        surv_mass[s] += e[i].w * g;
      }
    } else {
      int best = 0;
      for (int s = 1; s < ns; ++s)
        if (child_mass[surv[s]] > child_mass[surv[best]]) best = s;
      PUSH(best, e[i].idx, e[i].w);
      surv_mass[best] += e[i].w;
    }
  }
#undef PUSH
  double total = 0.0;
  for (int s = 0; s < ns; ++s) total += surv_mass[s];
  for (int s = 0; s < ns; ++s) {
    out->children[s] = kept.comps[surv[s]];
    out->children[s].w = surv_mass[s] / total;
  }
  out->ns = ns;
  out->ok = 1;
  free(kept.gamma);
}

/* gmm.cpp:489-513 reset_parents_to_child_moments */
static void reset_parents(comp_t* nodes, const trgo_tree* t) {
  for (int l = t->max_level - 2; l >= 0; --l)
    for (int i = 0; i < t->n_nodes; ++i) {
      if (t->level[i] != l || t->child_count[i] == 0) continue;
      double w = 0.0, mu[3] = {0, 0, 0};
      for (int c = 0; c < t->child_count[i]; ++c) {
        const comp_t* ch = &nodes[t->first_child[i] + c];
        w += ch->w;
        for (int k = 0; k < 3; ++k) mu[k] = mu[k] + ch->w * ch->mean[k];
      }
      if (!(w > 0.0)) continue;
      for (int k = 0; k < 3; ++k) mu[k] = mu[k] / w;
      double cov[3][3] = {{0}};
      for (int c = 0; c < t->child_count[i]; ++c) {
        const comp_t* ch = &nodes[t->first_child[i] + c];
        double d[3];
        for (int k = 0; k < 3; ++k) d[k] = ch->mean[k] - mu[k];
        for (int r = 0; r < 3; ++r)
          for (int s = 0; s < 3; ++s) cov[r][s] = cov[r][s] + ch->w * (ch->cov[r][s] + d[r] * d[s]);
      }
      for (int r = 0; r < 3; ++r)
        for (int s = 0; s < 3; ++s) cov[r][s] = cov[r][s] / w;
      memcpy(nodes[i].mean, mu, sizeof mu);
      memcpy(nodes[i].cov, cov, sizeof cov);
    }
}

/* ------------------------------------------------------------ association */

typedef struct {
  double *m0, *m1, *m2; /* J, J*3, J*9 (row-major) */
  uint64_t total_points, outliers, evals;
  double total_mass;
} moments_t;

static void tf_apply(const double* R, const double* t, const double p[3], double y[3]) {
  for (int i = 0; i < 3; ++i) {
    double s = R[3 * i] * p[0];
    s += R[3 * i + 1] * p[1];
    s += R[3 * i + 2] * p[2];
    y[i] = s + t[i];
  }
}

/* association.cpp:91-157 associate_adaptive (+ accumulate/merge :10-39) */
static void associate(const comp_t* nodes, const trgo_tree* t, const double* pts, size_t n, const double* R,
                      const double* tr, double lambda_c, int max_level, moments_t* out, int* pnode, double* pw) {
  const int J = t->n_nodes;
  if (n == 0) fail(1, "association: empty point cloud");
  if (J == 0) fail(1, "association: empty model");
  if (!(lambda_c >= 0.0 && lambda_c <= 1.0 / 3.0)) fail(1, "association: lambda_c outside [0, 1/3]");
  const int depth = max_level == 0 ? t->max_level : max_level;
  if (depth < 1 || depth > t->max_level) fail(1, "association: search depth exceeds tree depth");
  int root_count = 0;
  while (root_count < J && t->level[root_count] == 0) ++root_count;
  memset(out->m0, 0, sizeof(double) * J);
  memset(out->m1, 0, sizeof(double) * J * 3);
  if (out->m2) memset(out->m2, 0, sizeof(double) * J * 9);
  out->total_points = out->outliers = out->evals = 0;
  out->total_mass = 0.0;
  double* c0 = (double*)malloc(sizeof(double) * J);
  double* c1 = (double*)malloc(sizeof(double) * J * 3);
  double* c2 = (double*)malloc(sizeof(double) * J * 9);
  for (size_t b = 0; b < n; b += CHUNK) {
    const size_t end = b + CHUNK < n ? b + CHUNK : n;
    memset(c0, 0, sizeof(double) * J);
    memset(c1, 0, sizeof(double) * J * 3);
    memset(c2, 0, sizeof(double) * J * 9);
    uint64_t ctot = 0, cout = 0, cev = 0;
    double cmass = 0.0;
    for (size_t i = b; i < end; ++i) {
      double y[3];
      tf_apply(R, tr, &pts[3 * i], y);
      ctot += 1;
      int node = -1;
      double path = 1.0;
      int outlier = 0;
      double scores[8];
      for (int l = 0; l < depth; ++l) {
        const int first = node < 0 ? 0 : t->first_child[node];
        const int count = node < 0 ? root_count : t->child_count[node];
        double sum = 0.0;
        for (int k = 0; k < count; ++k) {
          const comp_t* g = &nodes[first + k];
          scores[k] = g->w > 0.0 ? g->w * exp(log_density(g, y)) : 0.0;
          sum += scores[k];
        }
        cev += (uint64_t)count;
        if (l == 0 && !(sum > 1e-300)) {
          outlier = 1;
          break;
        }
        if (!(sum > 0.0)) break;
        int best = 0;
        for (int k = 1; k < count; ++k)
          if (scores[k] > scores[best]) best = k;
        node = first + best;
        path *= scores[best] / sum;
        if (t->child_count[node] == 0) break;
        if (node_complexity(nodes[node].lam) <= lambda_c) break;
      }
      if (pnode) {
        pnode[i] = (outlier || node < 0) ? -1 : node;
        pw[i] = (outlier || node < 0) ? 0.0 : path;
      }
      if (outlier || node < 0) {
        cout += 1;
        continue;
      }
      /* MomentSet::accumulate association.cpp:10-24 */
      if (!(path >= 0.0 && path <= 1.0)) fail(1, "MomentSet::accumulate: gamma outside [0,1]");
      if (!(isfinite(y[0]) && isfinite(y[1]) && isfinite(y[2]))) fail(1, "MomentSet::accumulate: non-finite point");
      c0[node] += path;
      for (int k = 0; k < 3; ++k) c1[3 * node + k] = c1[3 * node + k] + path * y[k];
      for (int r = 0; r < 3; ++r)
        for (int s = 0; s < 3; ++s) c2[9 * node + 3 * r + s] = c2[9 * node + 3 * r + s] + path * (y[r] * y[s]);
      cmass += path;
    }
    /* MomentSet::merge association.cpp:26-39, chunk order */
    for (int j = 0; j < J; ++j) {
      out->m0[j] += c0[j];
      for (int k = 0; k < 3; ++k) out->m1[3 * j + k] = out->m1[3 * j + k] + c1[3 * j + k];
      if (out->m2)
        for (int k = 0; k < 9; ++k) out->m2[9 * j + k] = out->m2[9 * j + k] + c2[9 * j + k];
    }
    out->total_points += ctot;
    out->total_mass += cmass;
    out->outliers += cout;
    out->evals += cev;
  }
  free(c0);
  free(c1);
  free(c2);
}

/* gmm.cpp:523-580 calibrate_pass */
static double calibrate_pass(const bctx* c, size_t n, comp_t* nodes, const trgo_tree* t) {
  const int J = t->n_nodes;
  moments_t m;
  m.m0 = (double*)malloc(sizeof(double) * J);
  m.m1 = (double*)malloc(sizeof(double) * J * 3);
  m.m2 = (double*)malloc(sizeof(double) * J * 9);
  const double I[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1}, z[3] = {0, 0, 0};
  associate(nodes, t, c->pts, n, I, z, 0.0, 0, &m, NULL, NULL);
  if (c->stats) c->stats->calib_density_evals += m.evals;
  double* branch = (double*)calloc(J, sizeof(double));
  double drift = 0.0;
  for (int j = 0; j < J; ++j) {
    if (t->child_count[j] != 0) continue;
    branch[j] = m.m0[j];
    if (!(m.m0[j] > 0.0)) continue;
    double mu[3], sc[3][3], sc2[3][3];
    for (int k = 0; k < 3; ++k) mu[k] = m.m1[3 * j + k] / m.m0[j];
    for (int r = 0; r < 3; ++r)
      for (int s = 0; s < 3; ++s) sc[r][s] = m.m2[9 * j + 3 * r + s] / m.m0[j] - mu[r] * mu[s];
    for (int r = 0; r < 3; ++r)
      for (int s = 0; s < 3; ++s) sc2[r][s] = 0.5 * (sc[r][s] + sc[s][r]);
    comp_t* g = &nodes[j];
    double dm[3] = {g->mean[0] - mu[0], g->mean[1] - mu[1], g->mean[2] - mu[2]};
    drift = smax(drift, norm3(dm));
    memcpy(g->mean, mu, sizeof mu);
    double before[3][3];
    memcpy(before, g->cov, sizeof before);
    set_floored_cov(g, sc2, cov_floor(sc2, c->cfg));
    double dc[3][3];
    for (int r = 0; r < 3; ++r)
      for (int s = 0; s < 3; ++s) dc[r][s] = g->cov[r][s] - before[r][s];
    drift = smax(drift, norm33(dc));
  }
  for (int l = t->max_level - 2; l >= 0; --l)
    for (int j = 0; j < J; ++j) {
      if (t->level[j] != l || t->child_count[j] == 0) continue;
      double s = 0.0;
      for (int q = 0; q < t->child_count[j]; ++q) s += branch[t->first_child[j] + q];
      branch[j] = s;
    }
#define REWEIGHT(first, count)                                   \
  do {                                                           \
    double s_ = 0.0;                                             \
    for (int q = 0; q < (count); ++q) s_ += branch[(first) + q]; \
    if (s_ > 0.0)                                                \
      for (int q = 0; q < (count); ++q) {                        \
        const double w_ = branch[(first) + q] / s_;              \
        drift = smax(drift, fabs(nodes[(first) + q].w - w_));    \
        nodes[(first) + q].w = w_;                               \
      }                                                          \
  } while (0)
  int top = 0;
  while (top < J && t->level[top] == 0) ++top;
  REWEIGHT(0, top);
  for (int j = 0; j < J; ++j)
    if (t->child_count[j] != 0) REWEIGHT(t->first_child[j], t->child_count[j]);
#undef REWEIGHT
  reset_parents(nodes, t);
  for (int j = 0; j < J; ++j)
    if (t->child_count[j] != 0) refresh_eig(&nodes[j]);
  free(branch);
  free(m.m0);
  free(m.m1);
  free(m.m2);
  return drift;
}

int trgo_tree_capacity(int max_level) {
  int cap = 0, p = 1;
  for (int l = 0; l < max_level; ++l) {
    p *= 8;
    cap += p;
  }
  return cap;
}

int trgo_tree_alloc(trgo_tree* t, int capacity) {
  memset(t, 0, sizeof *t);
  t->capacity = capacity;
  t->weight = (double*)calloc(capacity, sizeof(double));
  t->mean = (double*)calloc(capacity * 3, sizeof(double));
  t->cov = (double*)calloc(capacity * 9, sizeof(double));
  t->lambdas = (double*)calloc(capacity * 3, sizeof(double));
  t->axes = (double*)calloc(capacity * 9, sizeof(double));
  t->log_norm = (double*)calloc(capacity, sizeof(double));
  t->parent = (int*)calloc(capacity, sizeof(int));
  t->first_child = (int*)calloc(capacity, sizeof(int));
  t->child_count = (int*)calloc(capacity, sizeof(int));
  t->level = (int*)calloc(capacity, sizeof(int));
  return 0;
}

void trgo_tree_free(trgo_tree* t) {
  free(t->weight);
  free(t->mean);
  free(t->cov);
  free(t->lambdas);
  free(t->axes);
  free(t->log_norm);
  free(t->parent);
  free(t->first_child);
  free(t->child_count);
  free(t->level);
  memset(t, 0, sizeof *t);
}

static void export_nodes(const comp_t* nodes, trgo_tree* t) {
  for (int i = 0; i < t->n_nodes; ++i) {
    const comp_t* g = &nodes[i];
    t->weight[i] = g->w;
    t->log_norm[i] = g->log_norm;
    for (int r = 0; r < 3; ++r) {
      t->mean[3 * i + r] = g->mean[r];
      t->lambdas[3 * i + r] = g->lam[r];
      for (int s = 0; s < 3; ++s) {
        t->cov[9 * i + 3 * r + s] = g->cov[r][s];
        t->axes[9 * i + 3 * r + s] = g->ax[r][s];
      }
    }
  }
}

static comp_t* import_nodes(const trgo_tree* t) {
  comp_t* nodes = (comp_t*)calloc(t->n_nodes > 0 ? t->n_nodes : 1, sizeof(comp_t));
  for (int i = 0; i < t->n_nodes; ++i) {
    comp_t* g = &nodes[i];
    g->w = t->weight[i];
    g->log_norm = t->log_norm[i];
    for (int r = 0; r < 3; ++r) {
      g->mean[r] = t->mean[3 * i + r];
      g->lam[r] = t->lambdas[3 * i + r];
      for (int s = 0; s < 3; ++s) {
        g->cov[r][s] = t->cov[9 * i + 3 * r + s];
        g->ax[r][s] = t->axes[9 * i + 3 * r + s];
      }
    }
  }
  return nodes;
}

typedef struct {
  int node;
  entry_t* e;
  size_t n;
} pending_t;

/* gmm.cpp:584-657 build_tree */
int trgo_build_tree(const double* xyz, size_t n, const trgo_model_cfg* cfg, trgo_tree* out,
                    trgo_build_stats* stats) {
  comp_t* nodes = NULL;
  pending_t* frontier = NULL;
  pending_t* next = NULL;
  size_t nf = 0;
  if (setjmp(g_jmp)) {
    free(nodes);
    free(frontier);
    free(next);
    return g_code;
  }
  /* validate_config gmm.cpp:465-477, validate_cloud :479-484 */
  if (cfg->max_level < 1) fail(1, "max_level must be >= 1");
  if (cfg->em_iterations_per_node < 1) fail(1, "em_iterations_per_node must be >= 1");
  if (cfg->min_points_per_node < 1) fail(1, "min_points_per_node must be >= 1");
  if (!(cfg->eps >= 0.0) || !(cfg->abs_floor > 0.0)) fail(1, "covariance regularization must be positive");
  if (n == 0) fail(1, "point cloud is empty");
  for (size_t i = 0; i < 3 * n; ++i)
    if (!isfinite(xyz[i])) fail(1, "point cloud has non-finite coordinates");
  if (stats) memset(stats, 0, sizeof *stats);
  const int cap = trgo_tree_capacity(cfg->max_level);
  if (out->capacity < cap) fail(1, "tree capacity too small");
  nodes = (comp_t*)calloc(cap, sizeof(comp_t));
  bctx c = {xyz, cfg, stats};
  trgo_tree* t = out;
  t->max_level = cfg->max_level;
  t->n_nodes = 0;
  frontier = (pending_t*)malloc(sizeof(pending_t) * cap);
  next = (pending_t*)malloc(sizeof(pending_t) * cap);
  {
    entry_t* all = (entry_t*)malloc(sizeof(entry_t) * n);
    for (size_t i = 0; i < n; ++i) {
      all[i].idx = i;
      all[i].w = 1.0;
    }
    expansion_t root;
    expand_node(&c, all, n, 1, &root);
    if (stats) {
      stats->entries_per_round[0] = n;
      stats->expanded_per_round[0] = 1;
    }
    free(all);
    for (int s = 0; s < root.ns; ++s) {
      const int id = t->n_nodes++;
      nodes[id] = root.children[s];
      t->parent[id] = -1;
      t->first_child[id] = -1;
      t->child_count[id] = 0;
      t->level[id] = 0;
      frontier[nf].node = id;
      frontier[nf].e = root.child_entries[s];
      frontier[nf].n = root.child_n[s];
      ++nf;
    }
  }
  for (int l = 0; l + 1 < cfg->max_level; ++l) {
    size_t nn = 0;
    for (size_t f = 0; f < nf; ++f) {
      pending_t* p = &frontier[f];
      double mass = 0.0;
      for (size_t i = 0; i < p->n; ++i) mass += p->e[i].w;
      if (mass < (double)cfg->min_points_per_node) {
        free(p->e);
        p->e = NULL;
        continue;
      }
      expansion_t ex;
      expand_node(&c, p->e, p->n, 0, &ex);
      if (stats) {
        stats->entries_per_round[l + 1] += p->n;
        stats->expanded_per_round[l + 1] += 1;
      }
      free(p->e);
      p->e = NULL;
      if (!ex.ok) continue;
      t->first_child[p->node] = t->n_nodes;
      t->child_count[p->node] = ex.ns;
      for (int s = 0; s < ex.ns; ++s) {
        const int id = t->n_nodes++;
        nodes[id] = ex.children[s];
        t->parent[id] = p->node;
        t->first_child[id] = -1;
        t->child_count[id] = 0;
        t->level[id] = l + 1;
        next[nn].node = id;
        next[nn].e = ex.child_entries[s];
        next[nn].n = ex.child_n[s];
        ++nn;
      }
    }
    pending_t* tmp = frontier;
    frontier = next;
    next = tmp;
    nf = nn;
  }
  for (size_t f = 0; f < nf; ++f) free(frontier[f].e);
  nf = 0;
  reset_parents(nodes, t);
  for (int i = 0; i < t->n_nodes; ++i) refresh_eig(&nodes[i]);
  double drift = INFINITY;
  int pass = 0;
  for (; pass < kCalibrationPassLimit && drift > 1e-13; ++pass) drift = calibrate_pass(&c, n, nodes, t);
  if (stats) {
    stats->calibration_passes = pass;
    stats->calibration_drift = drift;
  }
  export_nodes(nodes, t);
  free(nodes);
  free(frontier);
  free(next);
  return 0;
}

int trgo_associate(const trgo_tree* t, const double* xyz, size_t n, const double* R, const double* tr,
                   double lambda_c, int max_level, double* m0, double* m1, double* m2, uint64_t* counters,
                   double* total_mass, int* point_node, double* point_weight) {
  comp_t* nodes = NULL;
  if (setjmp(g_jmp)) {
    free(nodes);
    return g_code;
  }
  nodes = import_nodes(t);
  moments_t m = {m0, m1, m2, 0, 0, 0, 0.0};
  associate(nodes, t, xyz, n, R, tr, lambda_c, max_level, &m, point_node, point_weight);
  counters[0] = m.total_points;
  counters[1] = m.outliers;
  counters[2] = m.evals;
  *total_mass = m.total_mass;
  free(nodes);
  return 0;
}

/* ------------------------------------------------------------- M-step */

typedef struct {
  double pi, mu[3];
  int j;
} vp_t; /* mstep.hpp:21-25 */

/* mstep.cpp:8-30 make_virtual_points */
static int make_vps(const double* m0, const double* m1, uint64_t total_points, int J, vp_t* vps) {
  if (total_points == 0) fail(1, "make_virtual_points: no points were associated");
  const double n = (double)total_points;
  const double floor_mass = 1e-8 * n;
  int nv = 0;
  for (int j = 0; j < J; ++j) {
    if (m0[j] <= floor_mass) continue;
    vps[nv].pi = m0[j] / n;
    for (int k = 0; k < 3; ++k) vps[nv].mu[k] = m1[3 * j + k] / m0[j];
    vps[nv].j = j;
    ++nv;
  }
  return nv;
}

/* mstep.cpp:32-47 criterion */
static double criterion(const comp_t* nodes, const vp_t* vps, int nv, const double* R, const double* t) {
  double total = 0.0;
  for (int v = 0; v < nv; ++v) {
    const comp_t* g = &nodes[vps[v].j];
    double y[3], d[3];
    tf_apply(R, t, vps[v].mu, y);
    for (int k = 0; k < 3; ++k) d[k] = y[k] - g->mean[k];
    for (int l = 0; l < 3; ++l) {
      const double lam = g->lam[l];
      if (!(lam > 0.0)) fail(2, "criterion: non-positive eigenvalue");
      const double ax[3] = {g->ax[0][l], g->ax[1][l], g->ax[2][l]};
      const double r = dot3(ax, d);
      total += vps[v].pi / lam * r * r;
    }
  }
  return total;
}

/* geometry.cpp:26-32 skew, 106-118 small_angle_rotation */
static void small_angle_rotation(const double w[3], double R[9]) {
  const double th = norm3(w);
  double k[3][3], kk[3][3];
  if (th < 1e-12) {
    const double s[3][3] = {{0.0, -w[2], w[1]}, {w[2], 0.0, -w[0]}, {-w[1], w[0], 0.0}};
    double hk[3][3];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) hk[i][j] = 0.5 * s[i][j];
    matmul33(hk, s, kk);
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) R[3 * i + j] = ((i == j ? 1.0 : 0.0) + s[i][j]) + kk[i][j];
    return;
  }
  const double a[3] = {w[0] / th, w[1] / th, w[2] / th};
  const double s[3][3] = {{0.0, -a[2], a[1]}, {a[2], 0.0, -a[0]}, {-a[1], a[0], 0.0}};
  const double st = sin(th), ct = 1.0 - cos(th);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) k[i][j] = ct * s[i][j];
  matmul33(k, s, kk);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) R[3 * i + j] = ((i == j ? 1.0 : 0.0) + st * s[i][j]) + kk[i][j];
}

/* LDLT with diagonal pivoting (shim Eigen::LDLT, right-looking) */
static void ldlt_solve6(const double A[6][6], const double b[6], double x[6]) {
  double a[6][6], l[6][6], d[6];
  int perm[6];
  memcpy(a, A, sizeof a);
  for (int i = 0; i < 6; ++i) {
    perm[i] = i;
    for (int j = 0; j < 6; ++j) l[i][j] = (i == j) ? 1.0 : 0.0;
  }
  for (int k = 0; k < 6; ++k) {
    int p = k;
    for (int i = k + 1; i < 6; ++i)
      if (fabs(a[i][i]) > fabs(a[p][p])) p = i;
    if (p != k) {
      int tp = perm[k];
      perm[k] = perm[p];
      perm[p] = tp;
      for (int j = 0; j < 6; ++j) {
        double t = a[k][j];
        a[k][j] = a[p][j];
        a[p][j] = t;
      }
      for (int i = 0; i < 6; ++i) {
        double t = a[i][k];
        a[i][k] = a[i][p];
        a[i][p] = t;
      }
      for (int j = 0; j < k; ++j) {
        double t = l[k][j];
        l[k][j] = l[p][j];
        l[p][j] = t;
      }
    }
    const double dk = a[k][k];
    d[k] = dk;
    for (int i = k + 1; i < 6; ++i) l[i][k] = (dk != 0.0) ? a[i][k] / dk : 0.0;
    for (int i = k + 1; i < 6; ++i)
      for (int j = k + 1; j < 6; ++j) a[i][j] = a[i][j] - l[i][k] * dk * l[j][k];
  }
  double y[6];
  for (int i = 0; i < 6; ++i) y[i] = b[perm[i]];
  for (int i = 0; i < 6; ++i) {
    double s = y[i];
    for (int j = 0; j < i; ++j) s -= l[i][j] * y[j];
    y[i] = s;
  }
  for (int i = 0; i < 6; ++i) y[i] = (d[i] != 0.0) ? y[i] / d[i] : 0.0;
  double z[6];
  for (int i = 5; i >= 0; --i) {
    double s = y[i];
    for (int j = i + 1; j < 6; ++j) s -= l[j][i] * z[j];
    z[i] = s;
  }
  for (int i = 0; i < 6; ++i) x[perm[i]] = z[i];
}

/* mstep.cpp:49-99 solve_mstep. Returns 0 ok, 5 degenerate. */
static int solve_mstep(const comp_t* nodes, const vp_t* vps, int nv, double omega[3], double trans[3], double dR[9],
                       double dt[3], double* cb, double* ca, double* cond_out) {
  if (nv < 3) {
    snprintf(g_msg, sizeof g_msg, "solve_mstep: fewer than 3 contributing components");
    return 5;
  }
  double ata[6][6] = {{0}}, atb[6] = {0};
  for (int v = 0; v < nv; ++v) {
    const comp_t* g = &nodes[vps[v].j];
    const double lf = 1e-6 * g->lam[0];
    for (int l = 0; l < 3; ++l) {
      const double lam = smax(g->lam[l], lf);
      if (!(lam > 0.0)) fail(2, "solve_mstep: non-positive eigenvalue");
      const double w = sqrt(vps[v].pi / lam);
      const double nr[3] = {g->ax[0][l], g->ax[1][l], g->ax[2][l]};
      const double* mu = vps[v].mu;
      const double cr[3] = {mu[1] * nr[2] - mu[2] * nr[1], mu[2] * nr[0] - mu[0] * nr[2], mu[0] * nr[1] - mu[1] * nr[0]};
      double row[6];
      for (int k = 0; k < 3; ++k) row[k] = w * cr[k];
      for (int k = 0; k < 3; ++k) row[3 + k] = w * nr[k];
      const double e[3] = {g->mean[0] - mu[0], g->mean[1] - mu[1], g->mean[2] - mu[2]};
      const double rhs = w * dot3(nr, e);
      for (int j = 0; j < 6; ++j)
        for (int i = 0; i < 6; ++i) ata[i][j] = ata[i][j] + row[i] * row[j];
      for (int i = 0; i < 6; ++i) atb[i] = atb[i] + row[i] * rhs;
    }
  }
  double ev[6], vec[36];
  jacobi_n(6, &ata[0][0], ev, vec);
  const double lmin = ev[0], lmax = ev[5];
  const double cond = lmin > 0.0 ? lmax / lmin : INFINITY;
  if (!(cond < 1e12)) {
    snprintf(g_msg, sizeof g_msg, "solve_mstep: normal equations condition estimate exceeds limit");
    return 5;
  }
  double x[6];
  ldlt_solve6(ata, atb, x);
  for (int k = 0; k < 3; ++k) {
    omega[k] = x[k];
    trans[k] = x[3 + k];
  }
  small_angle_rotation(omega, dR);
  for (int k = 0; k < 3; ++k) dt[k] = trans[k];
  *cond_out = cond;
  const double I[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1}, z[3] = {0, 0, 0};
  *cb = criterion(nodes, vps, nv, I, z);
  *ca = criterion(nodes, vps, nv, dR, dt);
  return 0;
}

int trgo_solve_mstep(const trgo_tree* t, const double* m0, const double* m1, uint64_t total_points, double* omega,
                     double* trans, double* dR, double* dt, double* scal, int* n_vps) {
  comp_t* nodes = NULL;
  vp_t* vps = NULL;
  if (setjmp(g_jmp)) {
    free(nodes);
    free(vps);
    return g_code;
  }
  nodes = import_nodes(t);
  vps = (vp_t*)malloc(sizeof(vp_t) * (t->n_nodes + 1));
  const int nv = make_vps(m0, m1, total_points, t->n_nodes, vps);
  *n_vps = nv;
  const int rc = solve_mstep(nodes, vps, nv, omega, trans, dR, dt, &scal[0], &scal[1], &scal[2]);
  free(nodes);
  free(vps);
  return rc;
}

/* registration.cpp:140-151 tree_extent_estimate */
static double tree_extent_estimate(const comp_t* nodes, const trgo_tree* t) {
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int i = 0; i < t->n_nodes; ++i) {
    if (t->child_count[i] != 0) continue;
    const double r = 3.0 * sqrt(smax(nodes[i].lam[0], 0.0));
    for (int k = 0; k < 3; ++k) {
      lo[k] = smin(lo[k], nodes[i].mean[k] - r);
      hi[k] = smax(hi[k], nodes[i].mean[k] + r);
    }
  }
  const double d[3] = {hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]};
  return norm3(d);
}

/* registration.cpp:47-82 em_loop + 153-172 register_with_tree */
int trgo_register_with_tree(const trgo_tree* t, const double* xyz, size_t n, int tree_variant, double lambda_c,
                            int max_iters, double rot_tol, double trans_tol, double target_diag, double* R,
                            double* tr, int* iters, int* converged, double* crit_before, double* crit_after,
                            uint64_t* evals) {
  comp_t* nodes = NULL;
  vp_t* vps = NULL;
  moments_t m = {0};
  if (setjmp(g_jmp)) {
    free(nodes);
    free(vps);
    free(m.m0);
    free(m.m1);
    return g_code;
  }
  if (n == 0) fail(1, "register: bad source cloud");
  for (size_t i = 0; i < 3 * n; ++i)
    if (!isfinite(xyz[i])) fail(1, "register: bad source cloud");
  nodes = import_nodes(t);
  const int J = t->n_nodes;
  vps = (vp_t*)malloc(sizeof(vp_t) * (J + 1));
  m.m0 = (double*)malloc(sizeof(double) * J);
  m.m1 = (double*)malloc(sizeof(double) * J * 3);
  m.m2 = NULL;
  const double diag = target_diag > 0.0 ? target_diag : tree_extent_estimate(nodes, t);
  const double lc = tree_variant ? 0.0 : lambda_c;
  const double trans_limit = trans_tol * diag;
  /* initial transform = identity */
  double TR[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1}, Tt[3] = {0, 0, 0};
  int fails = 0;
  *iters = 0;
  *converged = 0;
  for (int it = 0; it < max_iters; ++it) {
    associate(nodes, t, xyz, n, TR, Tt, lc, 0, &m, NULL, NULL);
    evals[it] = m.evals;
    const int nv = make_vps(m.m0, m.m1, m.total_points, J, vps);
    ++*iters;
    double om[3], trn[3], dR[9], dt[3], cb, ca, cond;
    const int rc = solve_mstep(nodes, vps, nv, om, trn, dR, dt, &cb, &ca, &cond);
    if (rc == 0) {
      crit_before[it] = cb;
      crit_after[it] = ca;
      /* T = delta * T (geometry.hpp:42-47) */
      double nR[9], nt[3];
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
          double s = dR[3 * i] * TR[j];
          s += dR[3 * i + 1] * TR[3 + j];
          s += dR[3 * i + 2] * TR[6 + j];
          nR[3 * i + j] = s;
        }
      for (int i = 0; i < 3; ++i) {
        double s = dR[3 * i] * Tt[0];
        s += dR[3 * i + 1] * Tt[1];
        s += dR[3 * i + 2] * Tt[2];
        nt[i] = s + dt[i];
      }
      memcpy(TR, nR, sizeof nR);
      memcpy(Tt, nt, sizeof nt);
      fails = 0;
      /* geometry.cpp:17-20 rotation_angle */
      double c = ((dR[0] + dR[4]) + dR[8] - 1.0) * 0.5;
      c = c < -1.0 ? -1.0 : (c > 1.0 ? 1.0 : c);
      if (acos(c) < rot_tol && norm3(trn) < trans_limit) {
        *converged = 1;
        break;
      }
    } else {
      const double I[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1}, z[3] = {0, 0, 0};
      const double before = criterion(nodes, vps, nv, I, z);
      crit_before[it] = before;
      crit_after[it] = before;
      if (++fails >= 3) break;
    }
  }
  memcpy(R, TR, sizeof TR);
  memcpy(tr, Tt, sizeof Tt);
  free(nodes);
  free(vps);
  free(m.m0);
  free(m.m1);
  return 0;
}

int trgo_eig_sym3(const double* m, int floored, double floor_value, double* lambdas, double* axes) {
  if (setjmp(g_jmp)) return g_code;
  double a[3][3], lam[3], ax[3][3];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) a[r][c] = m[3 * r + c];
  if (floored)
    eig_sym3_floored(a, floor_value, lam, ax);
  else
    eig_sym3(a, lam, ax);
  for (int r = 0; r < 3; ++r) {
    lambdas[r] = lam[r];
    for (int c = 0; c < 3; ++c) axes[3 * r + c] = ax[r][c];
  }
  return 0;
}

double trgo_bbox_diagonal(const double* xyz, size_t n) {
  if (n == 0) return 0.0;
  double lo[3] = {xyz[0], xyz[1], xyz[2]}, hi[3] = {xyz[0], xyz[1], xyz[2]};
  for (size_t i = 0; i < n; ++i)
    for (int k = 0; k < 3; ++k) {
      lo[k] = smin(lo[k], xyz[3 * i + k]);
      hi[k] = smax(hi[k], xyz[3 * i + k]);
    }
  const double d[3] = {hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]};
  return norm3(d);
}
