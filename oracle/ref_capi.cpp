// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the reference's OWN C++ API (namespace treereg), so
// the unmodified reference sources compiled into oracle/_ref/libtreereg_ref.so
// can be driven from Python (ctypes) as the parity oracle and as the CPU
// baseline arm of bench.py.  Every entry point forwards to one reference
// function; the file:line each one wraps is given beside it.  Matrices cross
// this boundary ROW-MAJOR.
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "treereg/association.hpp"
#include "treereg/cloud_io.hpp"
#include "treereg/gmm.hpp"
#include "treereg/mstep.hpp"
#include "treereg/parallel.hpp"
#include "treereg/registration.hpp"
#include "treereg/synthetic.hpp"

using namespace treereg;

namespace {
thread_local std::string g_err;

// Error codes mirror include/treereg_b200.h (TRG_E*).
int map_exc(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const DegenerateGeometryError*>(&e)) return 5;
  if (dynamic_cast<const std::out_of_range*>(&e)) return 4;
  if (dynamic_cast<const std::invalid_argument*>(&e)) return 1;
  if (dynamic_cast<const std::domain_error*>(&e)) return 2;
  if (dynamic_cast<const std::runtime_error*>(&e)) return 3;
  return 3;
}

#define GUARD(body)                     \
  try {                                 \
    body;                               \
    return 0;                           \
  } catch (const std::exception& e) {   \
    return map_exc(e);                  \
  }

PointCloud to_cloud(const double* xyz, std::size_t n) {
  PointCloud c;
  c.points.resize(n);
  for (std::size_t i = 0; i < n; ++i) c.points[i] = Vec3(xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]);
  return c;
}
void from_cloud(const PointCloud& c, double* xyz) {
  for (std::size_t i = 0; i < c.size(); ++i)
    for (int k = 0; k < 3; ++k) xyz[3 * i + k] = c.points[i](k);
}
RigidTransform to_tf(const double* R, const double* t) {
  RigidTransform tf;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) tf.rotation(r, c) = R[3 * r + c];
  for (int k = 0; k < 3; ++k) tf.translation(k) = t[k];
  return tf;
}
void from_tf(const RigidTransform& tf, double* R, double* t) {
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) R[3 * r + c] = tf.rotation(r, c);
  for (int k = 0; k < 3; ++k) t[k] = tf.translation(k);
}

struct RefTree {
  GmmTree tree;
  BuildDiagnostics diag;
};
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// parallel.hpp:22 set_max_threads
void ref_set_threads(unsigned n) { parallel::set_max_threads(n); }

// synthetic.cpp:46-165 generators (kind: blobs|plane|sphere|scene|lumpy)
int ref_synthetic(const char* kind, std::size_t n, std::uint64_t seed, double* out) {
  GUARD({
    const std::string k(kind);
    PointCloud c;
    if (k == "blobs") c = synthetic_blobs(n, 0.01, seed);
    else if (k == "plane") c = synthetic_plane(n, seed);
    else if (k == "sphere") c = synthetic_sphere(n, seed);
    else if (k == "scene") c = synthetic_scene(n, seed);
    else if (k == "lumpy") c = synthetic_lumpy(n, seed);
    else throw std::invalid_argument("unknown kind");
    from_cloud(c, out);
  })
}

// cloud_io.cpp:48-57 unit_normalized (in place)
int ref_unit_normalized(double* xyz, std::size_t n) {
  GUARD({
    const PointCloud c = unit_normalized(to_cloud(xyz, n));
    from_cloud(c, xyz);
  })
}

// point_cloud bbox_diagonal (cloud_io.cpp:30-33)
double ref_bbox_diagonal(const double* xyz, std::size_t n) {
  return to_cloud(xyz, n).bbox_diagonal();
}

// cloud_io.cpp:511-532 random_rigid_transform
int ref_random_rigid_transform(double rot_deg, double trans, std::uint64_t seed, int trial,
                               double* R, double* t) {
  GUARD({
    SyntheticTransformSpec s;
    s.rot_range_deg = rot_deg;
    s.trans_range = trans;
    s.seed = seed;
    s.trials = trial + 1;
    from_tf(random_rigid_transform(s, trial), R, t);
  })
}

// cloud_io subsample (selection sampling)
int ref_subsample(const double* xyz, std::size_t n, std::size_t m, std::uint64_t seed, double* out) {
  GUARD({ from_cloud(subsample(to_cloud(xyz, n), m, seed), out); })
}

// gmm.cpp:584-657 build_tree
int ref_build_tree(const double* xyz, std::size_t n, int max_level, int em_iters,
                   std::size_t min_points, double eps, double abs_floor, void** out) {
  GUARD({
    ModelConfig cfg;
    cfg.max_level = max_level;
    cfg.em_iterations_per_node = em_iters;
    cfg.min_points_per_node = min_points;
    cfg.cov_regularization_epsilon = eps;
    cfg.cov_regularization_absolute = abs_floor;
    auto* h = new RefTree;
    try {
      h->tree = build_tree(to_cloud(xyz, n), cfg, &h->diag);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  })
}

// build_flat_gmm (gmm.cpp:659-736) as a depth-1 handle of J roots, so the
// tree export / dense association wrappers serve it too.
int ref_build_flat_gmm(const double* xyz, std::size_t n, std::size_t j, int max_level,
                       int em_iters, double eps, double abs_floor, std::uint64_t seed,
                       void** out) {
  GUARD({
    ModelConfig cfg;
    cfg.max_level = max_level;
    cfg.em_iterations_per_node = em_iters;
    cfg.cov_regularization_epsilon = eps;
    cfg.cov_regularization_absolute = abs_floor;
    cfg.rng_seed = seed;
    auto* h = new RefTree;
    try {
      h->tree.nodes = build_flat_gmm(to_cloud(xyz, n), j, cfg, &h->diag);
    } catch (...) {
      delete h;
      throw;
    }
    const std::size_t J = h->tree.nodes.size();
    h->tree.parent.assign(J, -1);
    h->tree.first_child.assign(J, -1);
    h->tree.child_count.assign(J, 0);
    h->tree.level.assign(J, 0);
    h->tree.max_level = 1;
    *out = h;
  })
}

// responsibilities_dense (association.cpp:54-89) over the handle's nodes.
int ref_responsibilities_dense(void* h, const double* xyz, std::size_t n, const double* R,
                               const double* t, double floor, double* m0, double* m1, double* m2,
                               std::uint64_t* counters, double* total_mass) {
  GUARD({
    const MomentSet m = responsibilities_dense(to_cloud(xyz, n), static_cast<RefTree*>(h)->tree.nodes,
                                               to_tf(R, t), floor);
    for (std::size_t q = 0; q < m.components(); ++q) {
      m0[q] = m.m0[q];
      for (int r = 0; r < 3; ++r) {
        m1[3 * q + r] = m.m1[q](r);
        for (int c = 0; c < 3; ++c) m2[9 * q + 3 * r + c] = m.m2[q](r, c);
      }
    }
    counters[0] = m.total_points;
    counters[1] = m.outliers;
    counters[2] = m.density_evaluations;
    *total_mass = m.total_mass;
  })
}

// read_cloud (cloud_io.cpp:401-427): format 0 = by content, 1 = ply ascii,
// 2 = ply binary_le, 3 = xyz.  Returns the point count, fills at most cap.
long long ref_read_cloud(const char* path, int format, double* out, std::size_t cap) {
  try {
    const PointCloud c = format == 0 ? read_cloud(path)
                                     : read_cloud(path, format == 1   ? CloudFormat::kPlyAscii
                                                        : format == 2 ? CloudFormat::kPlyBinaryLe
                                                                      : CloudFormat::kXyzText);
    for (std::size_t i = 0; i < c.size() && i < cap; ++i)
      for (int k = 0; k < 3; ++k) out[3 * i + k] = c.points[i](k);
    return static_cast<long long>(c.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// gmm.cpp:769-796 save_tree / 798-896 load_tree
int ref_save_tree(void* h, const char* path) {
  GUARD({ save_tree(static_cast<RefTree*>(h)->tree, path); })
}

int ref_load_tree(const char* path, void** out) {
  GUARD({
    auto* t = new RefTree;
    try {
      t->tree = load_tree(path);
    } catch (...) {
      delete t;
      throw;
    }
    *out = t;
  })
}

void ref_tree_free(void* h) { delete static_cast<RefTree*>(h); }
int ref_tree_size(void* h) { return static_cast<int>(static_cast<RefTree*>(h)->tree.size()); }
int ref_tree_max_level(void* h) { return static_cast<RefTree*>(h)->tree.max_level; }
double ref_tree_calibration_drift(void* h) { return static_cast<RefTree*>(h)->diag.calibration_drift; }
int ref_tree_num_traces(void* h) { return static_cast<int>(static_cast<RefTree*>(h)->diag.node_ll_traces.size()); }
int ref_tree_trace(void* h, int i, double* out, int cap) {
  const auto& tr = static_cast<RefTree*>(h)->diag.node_ll_traces.at(i);
  const int n = static_cast<int>(tr.size());
  for (int k = 0; k < n && k < cap; ++k) out[k] = tr[k];
  return n;
}

// Node layout per gmm.hpp:12-23 / 56-67; cov and axes ROW-MAJOR.
int ref_tree_export(void* h, double* weight, double* mean, double* cov, double* lambdas,
                    double* axes, double* log_norm, int* parent, int* first_child,
                    int* child_count, int* level) {
  const GmmTree& t = static_cast<RefTree*>(h)->tree;
  for (std::size_t i = 0; i < t.size(); ++i) {
    const GaussianComponent& g = t.nodes[i];
    weight[i] = g.weight;
    for (int r = 0; r < 3; ++r) {
      mean[3 * i + r] = g.mean(r);
      lambdas[3 * i + r] = g.eig.lambdas(r);
      for (int c = 0; c < 3; ++c) {
        cov[9 * i + 3 * r + c] = g.cov(r, c);
        axes[9 * i + 3 * r + c] = g.eig.axes(r, c);
      }
    }
    log_norm[i] = g.log_norm;
    parent[i] = t.parent[i];
    first_child[i] = t.first_child[i];
    child_count[i] = t.child_count[i];
    level[i] = t.level[i];
  }
  return 0;
}

// Builds a tree handle from arrays (e.g. the GPU's tree) so the reference's
// own association / EM can run on exactly that model.
int ref_tree_import(int n_nodes, int max_level, const double* weight, const double* mean,
                    const double* cov, const double* lambdas, const double* axes,
                    const double* log_norm, const int* parent, const int* first_child,
                    const int* child_count, const int* level, void** out) {
  GUARD({
    auto* h = new RefTree;
    GmmTree& t = h->tree;
    t.max_level = max_level;
    t.nodes.resize(n_nodes);
    t.parent.assign(parent, parent + n_nodes);
    t.first_child.assign(first_child, first_child + n_nodes);
    t.child_count.assign(child_count, child_count + n_nodes);
    t.level.assign(level, level + n_nodes);
    for (int i = 0; i < n_nodes; ++i) {
      GaussianComponent& g = t.nodes[i];
      g.weight = weight[i];
      for (int r = 0; r < 3; ++r) {
        g.mean(r) = mean[3 * i + r];
        g.eig.lambdas(r) = lambdas[3 * i + r];
        for (int c = 0; c < 3; ++c) {
          g.cov(r, c) = cov[9 * i + 3 * r + c];
          g.eig.axes(r, c) = axes[9 * i + 3 * r + c];
        }
      }
      g.log_norm = log_norm[i];
    }
    *out = h;
  })
}

// association.cpp:91-157 associate_adaptive. m1 J×3, m2 J×9 row-major (may be null).
int ref_associate(void* h, const double* xyz, std::size_t n, const double* R, const double* t,
                  double lambda_c, int max_level, double* m0, double* m1, double* m2,
                  std::uint64_t* counters /*total_points, outliers, density_evaluations*/,
                  double* total_mass) {
  GUARD({
    AssocConfig ac;
    ac.lambda_c = lambda_c;
    ac.max_level = max_level;
    const MomentSet m = associate_adaptive(to_cloud(xyz, n), static_cast<RefTree*>(h)->tree,
                                           to_tf(R, t), ac);
    for (std::size_t j = 0; j < m.components(); ++j) {
      m0[j] = m.m0[j];
      for (int r = 0; r < 3; ++r) {
        if (m1) m1[3 * j + r] = m.m1[j](r);
        if (m2)
          for (int c = 0; c < 3; ++c) m2[9 * j + 3 * r + c] = m.m2[j](r, c);
      }
    }
    counters[0] = m.total_points;
    counters[1] = m.outliers;
    counters[2] = m.density_evaluations;
    *total_mass = m.total_mass;
  })
}

// Per-point deposits of associate_adaptive, by running the reference on
// one-point clouds: node = the only component with m0 > 0 (-1 = outlier),
// weight = its m0 (the path product, association.cpp:143, 151).
int ref_associate_points(void* h, const double* xyz, std::size_t n, const double* R,
                         const double* t, double lambda_c, int* node, double* weight) {
  GUARD({
    AssocConfig ac;
    ac.lambda_c = lambda_c;
    const GmmTree& tree = static_cast<RefTree*>(h)->tree;
    const RigidTransform tf = to_tf(R, t);
    PointCloud one;
    one.points.resize(1);
    for (std::size_t i = 0; i < n; ++i) {
      one.points[0] = Vec3(xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]);
      const MomentSet m = associate_adaptive(one, tree, tf, ac);
      node[i] = -1;
      weight[i] = 0.0;
      for (std::size_t j = 0; j < m.components(); ++j) {
        if (m.m0[j] > 0.0) {
          node[i] = static_cast<int>(j);
          weight[i] = m.m0[j];
        }
      }
    }
  })
}

// mstep.cpp:8-99 make_virtual_points + solve_mstep over a moment set.
// out: omega[3], translation[3], deltaR[9], deltat[3]; scal: crit_before, crit_after, cond
int ref_solve_mstep(void* h, const double* m0, const double* m1, std::uint64_t total_points,
                    double* omega, double* trans, double* dR, double* dt, double* scal,
                    int* n_vps) {
  GUARD({
    const GmmTree& tree = static_cast<RefTree*>(h)->tree;
    MomentSet m(tree.size());
    for (std::size_t j = 0; j < tree.size(); ++j) {
      m.m0[j] = m0[j];
      m.m1[j] = Vec3(m1[3 * j], m1[3 * j + 1], m1[3 * j + 2]);
    }
    m.total_points = total_points;
    const VirtualPointSet vps = make_virtual_points(m, tree.nodes);
    *n_vps = static_cast<int>(vps.size());
    const MStepSolution s = solve_mstep(vps);
    for (int k = 0; k < 3; ++k) {
      omega[k] = s.omega(k);
      trans[k] = s.translation(k);
    }
    from_tf(s.delta, dR, dt);
    scal[0] = s.criterion_before;
    scal[1] = s.criterion_after;
    scal[2] = s.condition_estimate;
  })
}

// registration.cpp:153-172 register_with_tree. variant_kind 0 adaptive, 1 tree.
// out_T: R[9], t[3]; iters/converged; traces (cap max_iters) for criterion
// before/after and eval counts.
int ref_register_with_tree(void* h, const double* xyz, std::size_t n, int variant_kind,
                           double lambda_c, int max_iters, double rot_tol, double trans_tol,
                           double target_diag, double* R, double* t, int* iters,
                           int* converged, double* crit_before, double* crit_after,
                           std::uint64_t* evals, double* em_seconds) {
  GUARD({
    RegistrationConfig cfg;
    cfg.variant.kind = variant_kind == 3   ? Variant::Kind::kIcpPointToPoint
                       : variant_kind == 2 ? Variant::Kind::kFlatGmm
                       : variant_kind == 1 ? Variant::Kind::kGmmTree
                                           : Variant::Kind::kAdaptive;
    cfg.variant.param = static_cast<RefTree*>(h)->tree.max_level;
    cfg.lambda_c = lambda_c;
    cfg.max_em_iterations = max_iters;
    cfg.rotation_tol = rot_tol;
    cfg.translation_tol = trans_tol;
    const RegistrationResult r = register_with_tree(static_cast<RefTree*>(h)->tree,
                                                    to_cloud(xyz, n), cfg, target_diag);
    from_tf(r.transform, R, t);
    *iters = r.iterations;
    *converged = r.converged ? 1 : 0;
    for (std::size_t k = 0; k < r.criterion_trace.size(); ++k) {
      crit_before[k] = r.criterion_trace[k];
      crit_after[k] = r.criterion_after_trace[k];
    }
    for (std::size_t k = 0; k < r.eval_counts.size(); ++k) evals[k] = r.eval_counts[k];
    *em_seconds = r.em_seconds;
  })
}

// registration.cpp:174-209 register_clouds (adaptive:L / tree:L).
int ref_register_clouds(const double* tgt, std::size_t nt, const double* src, std::size_t ns,
                        int variant_kind, int level, double lambda_c, int max_iters,
                        double* R, double* t, int* iters, int* converged, double* build_s,
                        double* em_s) {
  GUARD({
    RegistrationConfig cfg;
    cfg.variant.kind = variant_kind == 3   ? Variant::Kind::kIcpPointToPoint
                       : variant_kind == 2 ? Variant::Kind::kFlatGmm
                       : variant_kind == 1 ? Variant::Kind::kGmmTree
                                           : Variant::Kind::kAdaptive;
    cfg.variant.param = level;
    cfg.lambda_c = lambda_c;
    cfg.max_em_iterations = max_iters;
    const RegistrationResult r = register_clouds(to_cloud(tgt, nt), to_cloud(src, ns), cfg);
    from_tf(r.transform, R, t);
    *iters = r.iterations;
    *converged = r.converged ? 1 : 0;
    *build_s = r.model_build_seconds;
    *em_s = r.em_seconds;
  })
}

// geometry.cpp:40-79 / 81-102 eigensolvers (row-major in/out)
int ref_eig_sym3(const double* m, int floored, double floor_value, double* lambdas, double* axes) {
  GUARD({
    Mat3 a;
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) a(r, c) = m[3 * r + c];
    const EigenDecomp3 e = floored ? eig_sym3_floored(a, floor_value) : eig_sym3(a);
    for (int r = 0; r < 3; ++r) {
      lambdas[r] = e.lambdas(r);
      for (int c = 0; c < 3; ++c) axes[3 * r + c] = e.axes(r, c);
    }
  })
}

}  // extern "C"
