// Model files: save_tree / load_tree (gmm.cpp:769-896) in native code with
// the reference's own JSON library (nlohmann/json, header-only), so the bytes
// written and the parse errors raised are the reference's.  Host side of the
// model interchange; the eigen fields of a loaded model are computed on the
// device (trg_tree_upload_refresh).
#include <cmath>
#include <cstring>
#include <exception>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "json.hpp"
#include "treereg_b200.h"

namespace trg {
void set_error(const std::string& msg);
}

namespace {

// A runtime_error ("bad model file ...") or an invalid-argument style
// failure; mapped to TRG_ERUNTIME / TRG_EINVAL by the C entry points.
struct FileError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void save_host(const trg_tree* t, const char* path) {
  nlohmann::json j;
  j["format"] = "gmm-tree";
  j["version"] = 1;
  j["max_level"] = t->max_level;
  nlohmann::json nodes = nlohmann::json::array();
  for (int i = 0; i < t->n_nodes; ++i) {
    nlohmann::json node;
    node["level"] = t->level[i];
    node["parent"] = t->parent[i];
    node["weight"] = t->weight[i];
    node["mean"] = {t->mean[3 * i], t->mean[3 * i + 1], t->mean[3 * i + 2]};
    node["cov"] = std::vector<double>(t->cov + 9 * (size_t)i, t->cov + 9 * (size_t)i + 9);  // row-major
    nodes.push_back(std::move(node));
  }
  j["nodes"] = std::move(nodes);
  std::ofstream out(path);
  if (!out) throw FileError(std::string("cannot open for writing: ") + path);
  out << j.dump(1) << '\n';
  if (!out) throw FileError(std::string("write failed: ") + path);
}

// gmm.cpp:798-887 (everything but refresh_eig): parse and validate in the
// reference's order, fill the host tree (capacity permitting).
int load_host(const char* path, trg_tree* t) {
  std::ifstream in(path);
  if (!in) throw FileError(std::string("cannot open file: ") + path);
  nlohmann::json j;
  try {
    in >> j;
  } catch (const std::exception& e) {
    throw FileError(std::string("bad model file ") + path + ": " + e.what());
  }
  const auto fail = [&](const std::string& msg) {
    return FileError(std::string("bad model file ") + path + ": " + msg);
  };
  try {
    if (j.at("format") != "gmm-tree") throw fail("unknown format tag");
    if (j.at("version") != 1) throw fail("unsupported version");
    const int L = j.at("max_level").get<int>();
    if (L < 1) throw fail("max_level must be >= 1");
    const auto& nodes = j.at("nodes");
    if (!nodes.is_array() || nodes.empty()) throw fail("empty node array");
    const int n = static_cast<int>(nodes.size());
    std::vector<int> level(n), parent(n), first(n, -1), count(n, 0);
    std::vector<double> weight(n), mean(3 * (size_t)n), cov(9 * (size_t)n);
    for (int i = 0; i < n; ++i) {
      const auto& node = nodes[i];
      level[i] = node.at("level").get<int>();
      parent[i] = node.at("parent").get<int>();
      weight[i] = node.at("weight").get<double>();
      const auto& m = node.at("mean");
      const auto& c = node.at("cov");
      if (m.size() != 3 || c.size() != 9) throw fail("node " + std::to_string(i) + " has malformed moments");
      bool finite = std::isfinite(weight[i]) && weight[i] >= 0.0;
      for (int k = 0; k < 3; ++k) {
        mean[3 * (size_t)i + k] = m[k].get<double>();
        finite = finite && std::isfinite(mean[3 * (size_t)i + k]);
      }
      for (int k = 0; k < 9; ++k) {
        cov[9 * (size_t)i + k] = c[k].get<double>();
        finite = finite && std::isfinite(cov[9 * (size_t)i + k]);
      }
      if (!finite) throw fail("node " + std::to_string(i) + " has non-finite values");
      const int p = parent[i];
      if (p >= i || p < -1) throw fail("node " + std::to_string(i) + " has invalid parent");
      if (p == -1) {
        if (level[i] != 0) throw fail("node " + std::to_string(i) + " is an orphan");
      } else {
        if (level[i] != level[p] + 1) throw fail("node " + std::to_string(i) + " has inconsistent level");
        if (first[p] == -1) {
          first[p] = i;
        } else if (i != first[p] + count[p]) {
          throw fail("children of node " + std::to_string(p) + " are not contiguous");
        }
        ++count[p];
      }
      if (level[i] < 0 || level[i] >= L) throw fail("node " + std::to_string(i) + " level out of range");
    }
    double root = 0.0;
    for (int i = 0; i < n; ++i)
      if (level[i] == 0) root += weight[i];
    if (std::abs(root - 1.0) > 1e-9) throw fail("top-level weights do not sum to 1");
    for (int i = 0; i < n; ++i) {
      if (count[i] == 0) continue;
      double s = 0.0;
      for (int c = 0; c < count[i]; ++c) s += weight[first[i] + c];
      if (std::abs(s - 1.0) > 1e-9)
        throw fail("children of node " + std::to_string(i) + " have weights not summing to 1");
    }
    t->n_nodes = n;
    t->max_level = L;
    if (t->capacity < n) return TRG_ERANGE;  // two-call pattern: n_nodes is the size needed
    for (int i = 0; i < n; ++i) {
      t->weight[i] = weight[i];
      t->level[i] = level[i];
      t->parent[i] = parent[i];
      t->first_child[i] = first[i];
      t->child_count[i] = count[i];
      for (int k = 0; k < 3; ++k) t->mean[3 * (size_t)i + k] = mean[3 * (size_t)i + k];
      for (int k = 0; k < 9; ++k) t->cov[9 * (size_t)i + k] = cov[9 * (size_t)i + k];
    }
    return TRG_OK;
  } catch (const nlohmann::json::exception& e) {
    throw fail(e.what());
  }
}

}  // namespace

extern "C" {

int trg_save_tree_host(const trg_tree* host, const char* path) {
  if (!host || !path || host->n_nodes <= 0) {
    trg::set_error("save_tree: empty model");
    return TRG_EINVAL;
  }
  try {
    save_host(host, path);
    return TRG_OK;
  } catch (const std::exception& e) {
    trg::set_error(e.what());
    return TRG_ERUNTIME;
  }
}

int trg_load_tree_host(const char* path, trg_tree* host) {
  if (!host || !path) {
    trg::set_error("load_tree: null argument");
    return TRG_EINVAL;
  }
  try {
    const int rc = load_host(path, host);
    if (rc == TRG_ERANGE) trg::set_error("load_tree: host capacity too small (n_nodes holds the size)");
    return rc;
  } catch (const std::exception& e) {
    trg::set_error(e.what());
    return TRG_ERUNTIME;
  }
}

int trg_save_tree(trg_ctx* ctx, const trg_tree_dev* tree, const char* path) {
  const int J = trg_tree_size(tree);
  if (J <= 0) {
    trg::set_error("save_tree: empty model");
    return TRG_EINVAL;
  }
  std::vector<double> w(J), mean(3 * (size_t)J), cov(9 * (size_t)J), lam(3 * (size_t)J),
      axes(9 * (size_t)J), ln(J);
  std::vector<int> parent(J), first(J), count(J), level(J);
  trg_tree h{};
  h.capacity = J;
  h.weight = w.data();
  h.mean = mean.data();
  h.cov = cov.data();
  h.lambdas = lam.data();
  h.axes = axes.data();
  h.log_norm = ln.data();
  h.parent = parent.data();
  h.first_child = first.data();
  h.child_count = count.data();
  h.level = level.data();
  const int rc = trg_tree_download(ctx, tree, &h);
  if (rc != TRG_OK) return rc;
  return trg_save_tree_host(&h, path);
}

int trg_load_tree(trg_ctx* ctx, const char* path, trg_tree_dev** out) {
  trg_tree h{};
  int rc = trg_load_tree_host(path, &h);  // capacity 0: sizes only
  if (rc != TRG_ERANGE) return rc == TRG_OK ? TRG_EINVAL : rc;
  const int J = h.n_nodes;
  std::vector<double> w(J), mean(3 * (size_t)J), cov(9 * (size_t)J);
  std::vector<int> parent(J), first(J), count(J), level(J);
  h.capacity = J;
  h.weight = w.data();
  h.mean = mean.data();
  h.cov = cov.data();
  h.parent = parent.data();
  h.first_child = first.data();
  h.child_count = count.data();
  h.level = level.data();
  if ((rc = trg_load_tree_host(path, &h)) != TRG_OK) return rc;
  rc = trg_tree_upload_refresh(ctx, &h, out);
  if (rc == TRG_EDOMAIN)  // load_tree's runtime_error for a non-PD covariance
    trg::set_error(std::string("bad model file ") + path + ": a node covariance is not positive definite");
  return rc == TRG_EDOMAIN ? TRG_ERUNTIME : rc;
}

}  // extern "C"
