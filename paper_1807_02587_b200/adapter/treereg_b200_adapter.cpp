// treereg -> B200 drop-in adapter.
//
// Defines the reference's hot-path C++ API (namespace treereg, declared in
// the reference's own headers proj/core/include/treereg/*.hpp) on top of the
// C-ABI in include/treereg_b200.h.  A treereg maintainer compiles this file
// into their build in place of the hot-path definitions of gmm.cpp,
// association.cpp, mstep.cpp and registration.cpp; every
// call then runs on the GPU.  Exceptions are rethrown as the reference's
// types (std::invalid_argument, std::domain_error, std::runtime_error,
// std::out_of_range, DegenerateGeometryError).
//
// Replaced entry points (reference file:line):
//   build_tree              gmm.hpp:69-70          -> trg_build_tree
//   associate_adaptive      association.hpp:54-56  -> trg_associate
//   make_virtual_points     mstep.hpp:46-47        -> trg_make_virtual_points
//   solve_mstep             mstep.hpp:67           -> trg_solve_mstep_vps
//   register_with_tree      registration.hpp:59-62 -> trg_register_with_tree
//   register_clouds         registration.hpp:53-55 -> trg_register_clouds
//                           (adaptive:L, tree:L, flat:J, icp)
//   register_icp_pt2pt      registration.hpp:64-66 -> trg_register_clouds (icp)
//   build_flat_gmm          gmm.hpp:74-76          -> trg_build_flat_gmm
//   responsibilities_dense  association.hpp:44-47  -> trg_responsibilities_dense
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "treereg/association.hpp"
#include "treereg/gmm.hpp"
#include "treereg/mstep.hpp"
#include "treereg/registration.hpp"
#include "treereg_b200.h"

namespace treereg {

namespace {

[[noreturn]] void raise(int rc, const char* where) {
  const std::string msg = std::string(where) + ": " + trg_last_error();
  switch (rc) {
    case TRG_EINVAL:
      throw std::invalid_argument(msg);
    case TRG_EDOMAIN:
      throw std::domain_error(msg);
    case TRG_ERANGE:
      throw std::out_of_range(msg);
    case TRG_EDEGENERATE:
      throw DegenerateGeometryError(msg);
    default:
      throw std::runtime_error(msg);
  }
}

void check(int rc, const char* where) {
  if (rc != TRG_OK) raise(rc, where);
}

// One context PER THREAD (device from TRG_DEVICE, default 0): a context owns
// a stream, growable workspaces and pinned buffers, so the reference's free
// functions -- callable from several threads at once -- must not share one.
std::atomic<unsigned long long> g_launches{0};  // finished threads' kernel launches

struct CtxHolder {
  trg_ctx* c = nullptr;
  ~CtxHolder() {
    if (!c) return;
    g_launches += trg_kernel_launches(c);
    trg_ctx_destroy(c);
  }
};

trg_ctx* ctx() {
  thread_local CtxHolder h;
  if (!h.c) {
    const char* d = std::getenv("TRG_DEVICE");
    check(trg_ctx_create(d ? std::atoi(d) : 0, &h.c), "trg_ctx_create");
    static std::once_flag once;
    std::call_once(once, [] {
      if (std::getenv("TRG_ADAPTER_REPORT"))
        std::atexit([] {
          std::fprintf(stderr, "trg adapter: %llu kernel launches on the B200 path\n",
                       static_cast<unsigned long long>(g_launches.load()));
        });
    });
  }
  return h.c;
}

// PointCloud::points is std::vector<Eigen::Vector3d>: 3 contiguous doubles
// per point, exactly the C-ABI's N*3 AoS layout.
const double* xyz(const PointCloud& c) {
  static_assert(sizeof(Vec3) == 3 * sizeof(double), "Vec3 must be 3 packed doubles");
  return c.points.empty() ? nullptr : c.points.front().data();
}

struct HostTree {
  std::vector<double> weight, mean, cov, lambdas, axes, log_norm;
  std::vector<int> parent, first_child, child_count, level;
  trg_tree t{};
  explicit HostTree(int cap)
      : weight(cap), mean(3 * cap), cov(9 * cap), lambdas(3 * cap), axes(9 * cap),
        log_norm(cap), parent(cap), first_child(cap), child_count(cap), level(cap) {
    t.capacity = cap;
    t.weight = weight.data();
    t.mean = mean.data();
    t.cov = cov.data();
    t.lambdas = lambdas.data();
    t.axes = axes.data();
    t.log_norm = log_norm.data();
    t.parent = parent.data();
    t.first_child = first_child.data();
    t.child_count = child_count.data();
    t.level = level.data();
  }
};

struct DevTree {
  trg_tree_dev* h = nullptr;
  ~DevTree() {
    if (h) trg_tree_free(ctx(), h);
  }
};

void upload(const GmmTree& tree, DevTree& out) {
  const int J = static_cast<int>(tree.size());
  HostTree ht(std::max(J, 1));
  ht.t.n_nodes = J;
  ht.t.max_level = tree.max_level;
  for (int i = 0; i < J; ++i) {
    const GaussianComponent& g = tree.nodes[i];
    ht.weight[i] = g.weight;
    ht.log_norm[i] = g.log_norm;
    for (int r = 0; r < 3; ++r) {
      ht.mean[3 * i + r] = g.mean(r);
      ht.lambdas[3 * i + r] = g.eig.lambdas(r);
      for (int c = 0; c < 3; ++c) {
        ht.cov[9 * i + 3 * r + c] = g.cov(r, c);
        ht.axes[9 * i + 3 * r + c] = g.eig.axes(r, c);
      }
    }
    ht.parent[i] = tree.parent[i];
    ht.first_child[i] = tree.first_child[i];
    ht.child_count[i] = tree.child_count[i];
    ht.level[i] = tree.level[i];
  }
  check(trg_tree_upload(ctx(), &ht.t, &out.h), "tree upload");
}

GmmTree download(trg_tree_dev* h) {
  const int J = trg_tree_size(h);
  HostTree ht(std::max(J, 1));
  check(trg_tree_download(ctx(), h, &ht.t), "tree download");
  GmmTree tree;
  tree.max_level = ht.t.max_level;
  tree.nodes.resize(J);
  tree.parent.assign(ht.parent.begin(), ht.parent.begin() + J);
  tree.first_child.assign(ht.first_child.begin(), ht.first_child.begin() + J);
  tree.child_count.assign(ht.child_count.begin(), ht.child_count.begin() + J);
  tree.level.assign(ht.level.begin(), ht.level.begin() + J);
  for (int i = 0; i < J; ++i) {
    GaussianComponent& g = tree.nodes[i];
    g.weight = ht.weight[i];
    g.log_norm = ht.log_norm[i];
    for (int r = 0; r < 3; ++r) {
      g.mean(r) = ht.mean[3 * i + r];
      g.eig.lambdas(r) = ht.lambdas[3 * i + r];
      for (int c = 0; c < 3; ++c) {
        g.cov(r, c) = ht.cov[9 * i + 3 * r + c];
        g.eig.axes(r, c) = ht.axes[9 * i + 3 * r + c];
      }
    }
  }
  return tree;
}

trg_model_config model_cfg(const ModelConfig& m) {
  trg_model_config c{};
  c.em_iterations_per_node = m.em_iterations_per_node;
  c.min_points_per_node = m.min_points_per_node;
  c.cov_regularization_epsilon = m.cov_regularization_epsilon;
  c.cov_regularization_absolute = m.cov_regularization_absolute;
  c.rng_seed = m.rng_seed;
  c.max_level = m.max_level;
  return c;
}

trg_reg_config reg_cfg(const RegistrationConfig& cfg) {
  trg_reg_config c{};
  c.variant_kind = cfg.variant.kind == Variant::Kind::kGmmTree          ? TRG_VARIANT_TREE
                   : cfg.variant.kind == Variant::Kind::kFlatGmm        ? TRG_VARIANT_FLAT
                   : cfg.variant.kind == Variant::Kind::kIcpPointToPoint ? TRG_VARIANT_ICP
                                                                        : TRG_VARIANT_ADAPTIVE;
  c.variant_param = cfg.variant.param;
  c.lambda_c = cfg.lambda_c;
  c.max_em_iterations = cfg.max_em_iterations;
  c.rotation_tol = cfg.rotation_tol;
  c.translation_tol = cfg.translation_tol;
  for (int r = 0; r < 3; ++r) {
    c.initial_t[r] = cfg.initial_transform.translation(r);
    for (int k = 0; k < 3; ++k) c.initial_R[3 * r + k] = cfg.initial_transform.rotation(r, k);
  }
  c.model_config = model_cfg(cfg.model_config);
  return c;
}

RegistrationResult result_of(const trg_reg_result& r, const std::vector<double>& cb,
                             const std::vector<double>& ca, const std::vector<uint64_t>& ev) {
  RegistrationResult out;
  for (int i = 0; i < 3; ++i) {
    out.transform.translation(i) = r.t[i];
    for (int k = 0; k < 3; ++k) out.transform.rotation(i, k) = r.R[3 * i + k];
  }
  out.iterations = r.iterations;
  out.converged = r.converged != 0;
  out.criterion_trace.assign(cb.begin(), cb.begin() + r.iterations);
  out.criterion_after_trace.assign(ca.begin(), ca.begin() + r.iterations);
  out.eval_counts.assign(ev.begin(), ev.begin() + r.iterations);
  out.model_build_seconds = r.model_build_seconds;
  out.em_seconds = r.em_seconds;
  out.model_components = r.model_components;
  return out;
}

}  // namespace

GmmTree build_tree(const PointCloud& cloud, const ModelConfig& config,
                   BuildDiagnostics* diagnostics) {
  trg_model_config c = model_cfg(config);
  trg_build_diag d{};
  const int I1 = config.em_iterations_per_node + 1;
  int cap = 1;
  for (int l = 1, p = 8; l < config.max_level; ++l, p *= 8) cap += p;
  std::vector<double> traces;
  if (diagnostics && config.max_level >= 1 && config.max_level <= 7 && I1 > 0) {
    traces.assign(static_cast<size_t>(cap) * I1, 0.0);
    d.ll_traces = traces.data();
    d.ll_trace_capacity = cap;
  }
  DevTree t;
  check(trg_build_tree(ctx(), xyz(cloud), cloud.size(), 0, &c, &t.h, &d), "build_tree");
  GmmTree tree = download(t.h);
  if (diagnostics) {
    diagnostics->calibration_drift = d.calibration_drift;
    diagnostics->node_ll_traces.clear();
    for (int e = 0; e < d.n_expansions && e < cap; ++e)
      diagnostics->node_ll_traces.emplace_back(traces.begin() + static_cast<size_t>(e) * I1,
                                               traces.begin() + static_cast<size_t>(e + 1) * I1);
  }
  return tree;
}

MomentSet associate_adaptive(const PointCloud& cloud, const GmmTree& tree,
                             const RigidTransform& t, const AssocConfig& config) {
  if (cloud.empty()) throw std::invalid_argument("association: empty point cloud");
  if (tree.size() == 0) throw std::invalid_argument("association: empty model");
  DevTree dt;
  upload(tree, dt);
  const int J = static_cast<int>(tree.size());
  std::vector<double> m0(J), m1(3 * J), m2(9 * J);
  trg_moments m{};
  m.m0 = m0.data();
  m.m1 = m1.data();
  m.m2 = m2.data();
  double R[9], tr[3];
  for (int i = 0; i < 3; ++i) {
    tr[i] = t.translation(i);
    for (int k = 0; k < 3; ++k) R[3 * i + k] = t.rotation(i, k);
  }
  trg_assoc_config ac{config.lambda_c, config.max_level, config.outlier_floor,
                      config.deterministic ? 1 : 0};
  check(trg_associate(ctx(), dt.h, xyz(cloud), cloud.size(), 0, R, tr, &ac, &m, nullptr, nullptr),
        "associate_adaptive");
  MomentSet out(J);
  for (int j = 0; j < J; ++j) {
    out.m0[j] = m0[j];
    for (int r = 0; r < 3; ++r) {
      out.m1[j](r) = m1[3 * j + r];
      for (int c = 0; c < 3; ++c) out.m2[j](r, c) = m2[9 * j + 3 * r + c];
    }
  }
  out.total_points = m.total_points;
  out.total_mass = m.total_mass;
  out.outliers = m.outliers;
  out.density_evaluations = m.density_evaluations;
  return out;
}

VirtualPointSet make_virtual_points(const MomentSet& moments,
                                    const std::vector<GaussianComponent>& components) {
  if (moments.components() != components.size())
    throw std::invalid_argument("make_virtual_points: moment/component count mismatch");
  const int J = static_cast<int>(components.size());
  std::vector<double> m1(3 * J), pi(J), mu(3 * J);
  std::vector<int> idx(J);
  for (int j = 0; j < J; ++j)
    for (int r = 0; r < 3; ++r) m1[3 * j + r] = moments.m1[j](r);
  int n = 0;
  check(trg_make_virtual_points(ctx(), J, moments.m0.data(), m1.data(), moments.total_points,
                                idx.data(), pi.data(), mu.data(), &n),
        "make_virtual_points");
  VirtualPointSet vps;
  vps.points.resize(n);
  for (int v = 0; v < n; ++v) {
    vps.points[v].pi_star = pi[v];
    vps.points[v].mu_star = Vec3(mu[3 * v], mu[3 * v + 1], mu[3 * v + 2]);
    vps.points[v].component = &components[idx[v]];
  }
  return vps;
}

MStepSolution solve_mstep(const VirtualPointSet& vps) {
  const int n = static_cast<int>(vps.size());
  std::vector<double> pi(n), mu(3 * n), mean(3 * n), lam(3 * n), axes(9 * n);
  for (int v = 0; v < n; ++v) {
    const VirtualPoint& vp = vps.points[v];
    const GaussianComponent& g = *vp.component;
    pi[v] = vp.pi_star;
    for (int r = 0; r < 3; ++r) {
      mu[3 * v + r] = vp.mu_star(r);
      mean[3 * v + r] = g.mean(r);
      lam[3 * v + r] = g.eig.lambdas(r);
      for (int c = 0; c < 3; ++c) axes[9 * v + 3 * r + c] = g.eig.axes(r, c);
    }
  }
  trg_mstep_solution s{};
  const int rc = trg_solve_mstep_vps(ctx(), n, pi.data(), mu.data(), mean.data(), lam.data(),
                                     axes.data(), &s);
  if (rc != TRG_OK) raise(rc, "solve_mstep");
  MStepSolution out;
  for (int i = 0; i < 3; ++i) {
    out.omega(i) = s.omega[i];
    out.translation(i) = s.translation[i];
    out.delta.translation(i) = s.delta_t[i];
    for (int k = 0; k < 3; ++k) out.delta.rotation(i, k) = s.delta_R[3 * i + k];
  }
  out.criterion_before = s.criterion_before;
  out.criterion_after = s.criterion_after;
  out.condition_estimate = s.condition_estimate;
  return out;
}

RegistrationResult register_with_tree(const GmmTree& tree, const PointCloud& source,
                                      const RegistrationConfig& config, double target_diag) {
  if (source.empty() || !source.all_finite())
    throw std::invalid_argument("register: bad source cloud");
  DevTree dt;
  upload(tree, dt);
  trg_reg_config c = reg_cfg(config);
  const int K = std::max(1, config.max_em_iterations);
  std::vector<double> cb(K), ca(K);
  std::vector<uint64_t> ev(K);
  trg_reg_result r{};
  r.criterion_trace = cb.data();
  r.criterion_after_trace = ca.data();
  r.eval_counts = ev.data();
  r.trace_capacity = K;
  check(trg_register_with_tree(ctx(), dt.h, xyz(source), source.size(), 0, &c, target_diag, &r),
        "register_with_tree");
  return result_of(r, cb, ca, ev);
}

std::vector<GaussianComponent> build_flat_gmm(const PointCloud& cloud, std::size_t j,
                                              const ModelConfig& config,
                                              BuildDiagnostics* diagnostics) {
  if (cloud.empty()) throw std::invalid_argument("point cloud is empty");
  if (!cloud.all_finite()) throw std::invalid_argument("point cloud has non-finite coordinates");
  const trg_model_config mc = model_cfg(config);
  DevTree dt;
  // the flat fit's per-iteration log-likelihoods (gmm.cpp:729-734)
  const int iters = std::max(1, config.em_iterations_per_node * config.max_level);
  std::vector<double> trace(static_cast<size_t>(iters));
  trg_build_diag d{};
  d.ll_traces = trace.data();
  d.ll_trace_capacity = (iters + config.em_iterations_per_node) / (config.em_iterations_per_node + 1);
  check(trg_build_flat_gmm(ctx(), xyz(cloud), cloud.size(), 0, j, &mc, &dt.h,
                           diagnostics != nullptr ? &d : nullptr),
        "build_flat_gmm");
  if (diagnostics != nullptr)
    diagnostics->node_ll_traces.emplace_back(trace.begin(), trace.begin() + d.flat_trace_len);
  return download(dt.h).nodes;
}

MomentSet responsibilities_dense(const PointCloud& cloud,
                                 const std::vector<GaussianComponent>& components,
                                 const RigidTransform& t, double outlier_floor) {
  if (cloud.empty()) throw std::invalid_argument("association: empty point cloud");
  if (components.empty()) throw std::invalid_argument("association: empty model");
  GmmTree flat;
  flat.nodes = components;
  const std::size_t J = components.size();
  flat.parent.assign(J, -1);
  flat.first_child.assign(J, -1);
  flat.child_count.assign(J, 0);
  flat.level.assign(J, 0);
  flat.max_level = 1;
  DevTree dt;
  upload(flat, dt);
  std::vector<double> m0(J), m1(3 * J), m2(9 * J);
  trg_moments m{};
  m.m0 = m0.data();
  m.m1 = m1.data();
  m.m2 = m2.data();
  double R[9], tr[3];
  for (int i = 0; i < 3; ++i) {
    tr[i] = t.translation(i);
    for (int k = 0; k < 3; ++k) R[3 * i + k] = t.rotation(i, k);
  }
  check(trg_responsibilities_dense(ctx(), dt.h, xyz(cloud), cloud.size(), 0, R, tr, outlier_floor,
                                   &m),
        "responsibilities_dense");
  MomentSet out(J);
  for (std::size_t q = 0; q < J; ++q) {
    out.m0[q] = m0[q];
    for (int r = 0; r < 3; ++r) {
      out.m1[q](r) = m1[3 * q + r];
      for (int c = 0; c < 3; ++c) out.m2[q](r, c) = m2[9 * q + 3 * r + c];
    }
  }
  out.total_points = m.total_points;
  out.total_mass = m.total_mass;
  out.outliers = m.outliers;
  out.density_evaluations = m.density_evaluations;
  return out;
}

RegistrationResult register_clouds(const PointCloud& target, const PointCloud& source,
                                   const RegistrationConfig& config) {
  if (target.empty() || source.empty()) throw std::invalid_argument("register: empty cloud");
  if (!target.all_finite() || !source.all_finite())
    throw std::invalid_argument("register: non-finite coordinates");
  trg_reg_config c = reg_cfg(config);
  const int K = std::max(1, config.max_em_iterations);
  std::vector<double> cb(K), ca(K);
  std::vector<uint64_t> ev(K);
  trg_reg_result r{};
  r.criterion_trace = cb.data();
  r.criterion_after_trace = ca.data();
  r.eval_counts = ev.data();
  r.trace_capacity = K;
  check(trg_register_clouds(ctx(), xyz(target), target.size(), xyz(source), source.size(), 0, &c,
                            &r),
        "register_clouds");
  return result_of(r, cb, ca, ev);
}

RegistrationResult register_icp_pt2pt(const PointCloud& target, const PointCloud& source,
                                      const RegistrationConfig& config) {
  RegistrationConfig c = config;
  c.variant.kind = Variant::Kind::kIcpPointToPoint;
  return register_clouds(target, source, c);
}

}  // namespace treereg
