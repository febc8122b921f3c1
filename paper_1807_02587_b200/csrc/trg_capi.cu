// C-ABI entry points (include/treereg_b200.h): context, workspace, tree
// upload/download and the E-step.  Host code here only validates, stages
// and launches; all arithmetic on the hot path runs in the kernels.
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <string>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "trg_internal.cuh"
#include "trg_assoc.cuh"
#include "trg_gmm.cuh"

namespace {
thread_local std::string g_last_error;
}

namespace trg {

void set_error(const std::string& msg) { g_last_error = msg; }

int ws_get(trg_ctx* ctx, int slot, size_t bytes, void** out) {
  if (bytes == 0) bytes = 16;
  if (ctx->slot_size[slot] < bytes) {
    if (ctx->slot_ptr[slot]) {
      TRG_CU(cudaStreamSynchronize(ctx->stream));
      TRG_CU(cudaFree(ctx->slot_ptr[slot]));
      ctx->slot_ptr[slot] = nullptr;
      ctx->slot_size[slot] = 0;
    }
    const size_t sz = bytes + bytes / 4;
    TRG_CU(cudaMalloc(&ctx->slot_ptr[slot], sz));
    ctx->slot_size[slot] = sz;
    if (slot == kSlotStamps) TRG_CU(cudaMemset(ctx->slot_ptr[slot], 0, sz));
  }
  *out = ctx->slot_ptr[slot];
  return TRG_OK;
}

int host_ws_get(trg_ctx* ctx, int slot, size_t bytes, void** out) {
  if (bytes == 0) bytes = 16;
  if (ctx->host_slot_size[slot] < bytes) {
    if (ctx->host_slot_ptr[slot]) {
      TRG_CU(cudaStreamSynchronize(ctx->stream));
      TRG_CU(cudaFreeHost(ctx->host_slot_ptr[slot]));
    }
    const size_t sz = bytes + bytes / 4;
    TRG_CU(cudaMallocHost(&ctx->host_slot_ptr[slot], sz));
    ctx->host_slot_size[slot] = sz;
  }
  *out = ctx->host_slot_ptr[slot];
  return TRG_OK;
}

static bool is_pinned(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

cudaError_t trg_memcpy(trg_ctx* ctx, void* dst, const void* src, size_t bytes, cudaMemcpyKind kind) {
  if (bytes == 0) return cudaSuccess;
  if (kind == cudaMemcpyHostToDevice) ctx->bytes_h2d += bytes;
  if (kind == cudaMemcpyDeviceToHost) ctx->bytes_d2h += bytes;
  const bool h2d = kind == cudaMemcpyHostToDevice, d2h = kind == cudaMemcpyDeviceToHost;
  if ((!h2d && !d2h) || is_pinned(h2d ? src : dst))
    return cudaMemcpyAsync(dst, src, bytes, kind, ctx->stream);
  void* stage = nullptr;
  if (host_ws_get(ctx, kSlotHostStage, bytes, &stage) != TRG_OK) return cudaErrorMemoryAllocation;
  cudaError_t e;
  if (h2d) {
    // the staging buffer may still feed an earlier copy on this stream
    if ((e = cudaStreamSynchronize(ctx->stream)) != cudaSuccess) return e;
    std::memcpy(stage, src, bytes);
    return cudaMemcpyAsync(dst, stage, bytes, kind, ctx->stream);
  }
  if ((e = cudaMemcpyAsync(stage, src, bytes, kind, ctx->stream)) != cudaSuccess) return e;
  if ((e = cudaStreamSynchronize(ctx->stream)) != cudaSuccess) return e;
  std::memcpy(dst, stage, bytes);
  return cudaSuccess;
}

int check_status(trg_ctx* ctx, const char* where) { return check_status_at(ctx, ctx->status, where); }

int check_status_at(trg_ctx* ctx, int* dev_status, const char* where) {
  int st = 0;
  TRG_CU(trg_memcpy(ctx, &st, dev_status, sizeof(int), cudaMemcpyDeviceToHost));
  TRG_CU(cudaStreamSynchronize(ctx->stream));
  return status_result(ctx, st, dev_status, where);
}

int status_result(trg_ctx* ctx, int st, int* dev_status, const char* where) {
  if (st != 0) {
    TRG_CU(cudaMemsetAsync(dev_status, 0, sizeof(int), ctx->stream));
    const char* what = st == kEDomain   ? "covariance is not positive definite / no positive trace"
                       : st == kEInval  ? "invalid argument"
                       : st == kERuntime ? "no responsibility mass"
                                         : "device error";
    set_error(std::string(where) + ": " + what);
    return st;
  }
  return TRG_OK;
}

int timeline_reset(trg_ctx* ctx) {
  TRG_CU(cudaMemsetAsync(ctx->dev_timeline, 0, sizeof(int), ctx->stream));
  return TRG_OK;
}

// Stream-ordered copy into a pinned buffer; parsed only when asked for
// (trg_debug_build_timeline), so the hot path never waits on it.
int timeline_fetch(trg_ctx* ctx) {
  void* h = nullptr;
  TRG_TRY(host_ws_get(ctx, kSlotTimelineHost, sizeof(Timeline), &h));
  TRG_CU(cudaMemcpyAsync(h, ctx->dev_timeline, sizeof(Timeline), cudaMemcpyDeviceToHost, ctx->stream));
  ctx->timeline_pending = true;
  return TRG_OK;
}

// Occupancy and the dynamic-smem attribute are per kernel and configuration,
// not per call: both are cached (process-wide, thread-safe) so a
// registration issues no driver queries on its way to the first launch.
static std::mutex g_attr_mu;
static std::map<std::tuple<const void*, int, size_t>, int> g_occ;
static std::map<const void*, size_t> g_smem_attr;

int persistent_grid(trg_ctx* ctx, const void* kernel, int block, size_t smem) {
  int per_sm = 0;
  {
    std::lock_guard<std::mutex> lk(g_attr_mu);
    auto it = g_occ.find({kernel, block, smem});
    if (it != g_occ.end()) per_sm = it->second;
  }
  if (per_sm == 0) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, smem);
    if (per_sm < 1) per_sm = 1;
    std::lock_guard<std::mutex> lk(g_attr_mu);
    g_occ[{kernel, block, smem}] = per_sm;
  }
  return ctx->sms * per_sm;
}

cudaError_t set_dynamic_smem(const void* kernel, size_t bytes) {
  {
    std::lock_guard<std::mutex> lk(g_attr_mu);
    auto it = g_smem_attr.find(kernel);
    if (it != g_smem_attr.end() && it->second >= bytes) return cudaSuccess;
  }
  const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) {
    std::lock_guard<std::mutex> lk(g_attr_mu);
    size_t& v = g_smem_attr[kernel];
    v = std::max(v, bytes);
  }
  return e;
}

// Whole-device contexts launch cooperatively: the driver guarantees every
// CTA is resident, which the grid barriers and role handovers need.
// SM-budgeted worker contexts (trg_register_batch) launch plainly so several
// run at once; their budgets sum to at most the device's SMs, which makes
// co-residency LIKELY but not guaranteed (the block scheduler may place a
// grid's CTAs unevenly).  Every spin-wait therefore carries a 10 s guard
// (spin_guard, trg_internal.cuh): a grid that cannot become resident traps
// and the call returns TRG_ECUDA instead of hanging the device.
cudaError_t launch_persistent(trg_ctx* ctx, const void* kernel, int G, int block, void** args,
                              size_t smem) {
  if (ctx->sms < ctx->device_sms)
    return cudaLaunchKernel(kernel, dim3(G), dim3(block), args, smem, ctx->stream);
  return cudaLaunchCooperativeKernel(kernel, dim3(G), dim3(block), args, smem, ctx->stream);
}

int tree_alloc(trg_ctx* ctx, int capacity, trg_tree_dev** out) {
  if (ctx->build_into_scratch) {
    // register_clouds' internal model: reuse the context's tree so repeated
    // registrations never call cudaMalloc/cudaFree (both synchronise the
    // device and would serialise concurrent contexts)
    if (ctx->scratch_tree && ctx->scratch_tree->capacity >= capacity) {
      *out = ctx->scratch_tree;
      return TRG_OK;
    }
    if (ctx->scratch_tree) {
      TRG_CU(cudaStreamSynchronize(ctx->stream));
      ctx->scratch_tree->ctx_scratch = false;
      trg_tree_free(ctx, ctx->scratch_tree);
      ctx->scratch_tree = nullptr;
    }
  }
  auto* t = new trg_tree_dev;
  t->capacity = capacity;
  if (cudaMalloc(&t->nodes, sizeof(DNode) * capacity) != cudaSuccess ||
      cudaMalloc(&t->cov, sizeof(double) * 9 * capacity) != cudaSuccess) {
    cudaFree(t->nodes);
    cudaFree(t->cov);
    delete t;
    set_error("tree_alloc: cudaMalloc failed");
    return TRG_ECUDA;
  }
  if (ctx->build_into_scratch) {
    t->ctx_scratch = true;
    ctx->scratch_tree = t;
  }
  *out = t;
  return TRG_OK;
}

// Stage N*3 points on the device (no-op when already there).
int stage_points_public(trg_ctx* ctx, const double* xyz, size_t n, int on_device, int slot,
                        const double** dev) {
  if (on_device) {
    *dev = xyz;
    return TRG_OK;
  }
  void* p = nullptr;
  TRG_TRY(ws_get(ctx, slot, sizeof(double) * 3 * n, &p));
  TRG_CU(trg_memcpy(ctx, p, xyz, sizeof(double) * 3 * n, cudaMemcpyHostToDevice));
  *dev = static_cast<const double*>(p);
  return TRG_OK;
}

int stage_points_side(trg_ctx* ctx, const double* xyz, size_t n, int on_device, int slot,
                      const double** dev, bool* deferred) {
  *deferred = false;
  if (on_device || !is_pinned(xyz)) return stage_points_public(ctx, xyz, n, on_device, slot, dev);
  if (!ctx->side) {
    TRG_CU(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
    TRG_CU(cudaEventCreateWithFlags(&ctx->side_done, cudaEventDisableTiming));
  }
  void* p = nullptr;
  TRG_TRY(ws_get(ctx, slot, sizeof(double) * 3 * n, &p));
  // the slot's previous reader (an earlier call on the main stream) is done:
  // every call collects before returning
  TRG_CU(cudaMemcpyAsync(p, xyz, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, ctx->side));
  TRG_CU(cudaEventRecord(ctx->side_done, ctx->side));
  ctx->bytes_h2d += sizeof(double) * 3 * n;
  *dev = static_cast<const double*>(p);
  *deferred = true;
  return TRG_OK;
}

int stage_wait(trg_ctx* ctx) {
  TRG_CU(cudaStreamWaitEvent(ctx->stream, ctx->side_done, 0));
  return TRG_OK;
}

}  // namespace trg

using namespace trg;

extern "C" {

const char* trg_last_error(void) { return g_last_error.c_str(); }

int trg_ctx_create(int device, trg_ctx** out) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    set_error("trg_ctx_create: no CUDA device (there is no CPU fallback)");
    return TRG_ECUDA;
  }
  if (device < 0 || device >= n) {
    set_error("trg_ctx_create: bad device index");
    return TRG_EINVAL;
  }
  TRG_CU(cudaSetDevice(device));
  auto* c = new trg_ctx;
  c->device = device;
  cudaDeviceProp prop;
  TRG_CU(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) {
    set_error("trg_ctx_create: this build targets sm_100a (B200) only");
    delete c;
    return TRG_ECUDA;
  }
  c->sms = prop.multiProcessorCount;
  c->device_sms = c->sms;
  TRG_CU(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  TRG_CU(cudaMalloc(&c->status, 2 * sizeof(int)));
  TRG_CU(cudaMemset(c->status, 0, 2 * sizeof(int)));
  c->status2 = c->status + 1;
  TRG_CU(cudaMalloc(&c->dev_timeline, sizeof(Timeline)));
  TRG_CU(cudaMemset(c->dev_timeline, 0, sizeof(Timeline)));
  *out = c;
  return TRG_OK;
}

int trg_ctx_destroy(trg_ctx* ctx) {
  if (!ctx) return TRG_OK;
  for (trg_ctx* w : ctx->workers) trg_ctx_destroy(w);
  ctx->workers.clear();
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (int i = 0; i < trg_ctx::kSlots; ++i) {
    if (ctx->slot_ptr[i]) cudaFree(ctx->slot_ptr[i]);
    if (ctx->host_slot_ptr[i]) cudaFreeHost(ctx->host_slot_ptr[i]);
  }
  if (ctx->scratch_tree) {
    ctx->scratch_tree->ctx_scratch = false;
    trg_tree_free(ctx, ctx->scratch_tree);
  }
  cudaFree(ctx->status);
  cudaFree(ctx->dev_timeline);
  if (ctx->side) {
    cudaStreamSynchronize(ctx->side);
    cudaEventDestroy(ctx->side_done);
    cudaStreamDestroy(ctx->side);
  }
  if (ctx->ext_ready) cudaEventDestroy(ctx->ext_ready);
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
  return TRG_OK;
}

int trg_device_sms(trg_ctx* ctx) { return ctx->sms; }
int trg_ctx_set_sm_budget(trg_ctx* ctx, int sms) {
  if (!ctx || sms < 0) {
    set_error("trg_ctx_set_sm_budget: bad argument");
    return TRG_EINVAL;
  }
  ctx->sms = (sms == 0 || sms > ctx->device_sms) ? ctx->device_sms : sms;
  return TRG_OK;
}
int trg_debug_build_timeline(trg_ctx* ctx, uint64_t* t_ns, int* labels, int cap) {
  if (ctx->timeline_pending) {
    TRG_CU(cudaStreamSynchronize(ctx->stream));
    const Timeline* h = (const Timeline*)ctx->host_slot_ptr[kSlotTimelineHost];
    const int m = std::min(h->n, 1024);
    ctx->timeline.assign(h->t, h->t + m);
    ctx->timeline_lab.assign(h->lab, h->lab + m);
    ctx->timeline_pending = false;
  }
  const int n = (int)ctx->timeline.size();
  for (int i = 0; i < n && i < cap; ++i) {
    t_ns[i] = ctx->timeline[i];
    labels[i] = ctx->timeline_lab[i];
  }
  return n;
}
void trg_ctx_transfer_bytes(trg_ctx* ctx, uint64_t* h2d, uint64_t* d2h) {
  *h2d = ctx->bytes_h2d;
  *d2h = ctx->bytes_d2h;
}
uint64_t trg_kernel_launches(trg_ctx* ctx) { return ctx->launches; }
void* trg_ctx_stream(trg_ctx* ctx) { return (void*)ctx->stream; }
int trg_ctx_wait_stream(trg_ctx* ctx, void* stream) {
  if (!ctx) {
    set_error("ctx_wait_stream: null context");
    return TRG_EINVAL;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (s == ctx->stream) return TRG_OK;
  TRG_CU(cudaSetDevice(ctx->device));
  if (!ctx->ext_ready) TRG_CU(cudaEventCreateWithFlags(&ctx->ext_ready, cudaEventDisableTiming));
  TRG_CU(cudaEventRecord(ctx->ext_ready, s));
  TRG_CU(cudaStreamWaitEvent(ctx->stream, ctx->ext_ready, 0));
  return TRG_OK;
}

int trg_tree_capacity(int max_level) {
  int cap = 0, p = 1;
  for (int l = 0; l < max_level; ++l) {
    p *= 8;
    cap += p;
  }
  return cap;
}

int trg_tree_size(const trg_tree_dev* tree) { return tree ? tree->n_nodes : 0; }

// Host tree -> packed device records.
// refresh_eig (gmm.cpp:31-35) of every node of an uploaded model, as
// load_tree does (gmm.cpp:889-894); the lowest failing node's error wins
// (key = node * 4 + code), like the reference's in-order loop.
__global__ void k_refresh_nodes(DNode* nodes, const double* cov, int J, int* first_bad) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= J) return;
  int code = 0;
  if (refresh_node(nodes[j], cov + 9 * (size_t)j)) code = 1;  // eig_sym3 rejected it
  else if (!(nodes[j].lam[2] > 0.0)) code = 2;                 // not positive definite
  if (code) atomicMin(first_bad, j * 4 + code);
}

static int tree_upload(trg_ctx* ctx, const trg_tree* h, bool refresh, trg_tree_dev** out);

int trg_tree_upload(trg_ctx* ctx, const trg_tree* h, trg_tree_dev** out) {
  trg::NvtxRange nvtx_range_("trg_tree_upload");
  return tree_upload(ctx, h, false, out);
}

int trg_tree_upload_refresh(trg_ctx* ctx, const trg_tree* h, trg_tree_dev** out) {
  return tree_upload(ctx, h, true, out);
}

static int tree_upload(trg_ctx* ctx, const trg_tree* h, bool refresh, trg_tree_dev** out) {
  if (!h || h->n_nodes <= 0 || h->max_level < 1) {
    set_error("trg_tree_upload: empty model");
    return TRG_EINVAL;
  }
  TRG_CU(cudaSetDevice(ctx->device));
  const int J = h->n_nodes;
  std::vector<DNode> nodes(J);
  int root_count = 0;
  while (root_count < J && h->level[root_count] == 0) ++root_count;
  for (int i = 0; i < J; ++i) {
    DNode& d = nodes[i];
    for (int r = 0; r < 3; ++r) {
      d.mean[r] = h->mean[3 * i + r];
      d.lam[r] = refresh ? 1.0 : h->lambdas[3 * i + r];  // (refresh: computed on the device)
      for (int k = 0; k < 3; ++k) d.axT[3 * r + k] = refresh ? (r == k) : h->axes[9 * i + 3 * k + r];
    }
    for (int r = 0; r < 3; ++r) d.il[r] = 1.0 / d.lam[r];
    set_prec(d.axT, d.il, d.prec);
    d.pad = 0.0;
    d.log_norm = refresh ? 0.0 : h->log_norm[i];
    d.weight = h->weight[i];
    const double tr = (d.lam[0] + d.lam[1]) + d.lam[2];
    d.cplx = tr > 0.0 ? d.lam[2] / tr : -1.0;
    d.first_child = h->first_child[i];
    d.child_count = h->child_count[i];
    d.level = h->level[i];
    d.parent = h->parent[i];
  }
  trg_tree_dev* t = nullptr;
  TRG_TRY(tree_alloc(ctx, std::max(J, trg_tree_capacity(h->max_level)), &t));
  t->n_nodes = J;
  t->max_level = h->max_level;
  t->root_count = root_count;
  {
    int up = 0;  // BFS prefix above the deepest level
    while (up < J && h->level[up] < h->max_level - 1) ++up;
    t->n_upper = up;
  }
  TRG_CU(trg_memcpy(ctx, t->nodes, nodes.data(), sizeof(DNode) * J, cudaMemcpyHostToDevice));
  TRG_CU(trg_memcpy(ctx, t->cov, h->cov, sizeof(double) * 9 * J, cudaMemcpyHostToDevice));
  if (refresh) {
    int* bad = nullptr;
    const int none = INT_MAX;
    TRG_CU(cudaMallocAsync((void**)&bad, sizeof(int), ctx->stream));
    TRG_CU(cudaMemcpyAsync(bad, &none, sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
    k_refresh_nodes<<<(J + 127) / 128, 128, 0, ctx->stream>>>(t->nodes, t->cov, J, bad);
    ctx->launches += 1;
    int key = none;
    TRG_CU(cudaMemcpyAsync(&key, bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    TRG_CU(cudaFreeAsync(bad, ctx->stream));
    TRG_CU(cudaStreamSynchronize(ctx->stream));
    if (key != none) {
      trg_tree_free(ctx, t);
      const int node = key / 4;
      if (key % 4 == 1) {
        set_error("eig_sym3: non-finite, non-symmetric or corrupted covariance (node " +
                  std::to_string(node) + ")");
        return TRG_EINVAL;
      }
      set_error("a node covariance is not positive definite");
      return TRG_EDOMAIN;
    }
  } else {
    TRG_CU(cudaStreamSynchronize(ctx->stream));
  }
  *out = t;
  return TRG_OK;
}

int trg_tree_download(trg_ctx* ctx, const trg_tree_dev* t, trg_tree* h) {
  trg::NvtxRange nvtx_range_("trg_tree_download");
  if (!t || !h) {
    set_error("trg_tree_download: null argument");
    return TRG_EINVAL;
  }
  if (h->capacity < t->n_nodes) {
    set_error("trg_tree_download: host capacity too small");
    return TRG_EINVAL;
  }
  TRG_CU(cudaSetDevice(ctx->device));
  const int J = t->n_nodes;
  std::vector<DNode> nodes(J);
  TRG_CU(trg_memcpy(ctx, nodes.data(), t->nodes, sizeof(DNode) * J, cudaMemcpyDeviceToHost));
  TRG_CU(trg_memcpy(ctx, h->cov, t->cov, sizeof(double) * 9 * J, cudaMemcpyDeviceToHost));
  TRG_CU(cudaStreamSynchronize(ctx->stream));
  h->n_nodes = J;
  h->max_level = t->max_level;
  for (int i = 0; i < J; ++i) {
    const DNode& d = nodes[i];
    for (int r = 0; r < 3; ++r) {
      h->mean[3 * i + r] = d.mean[r];
      h->lambdas[3 * i + r] = d.lam[r];
      for (int k = 0; k < 3; ++k) h->axes[9 * i + 3 * k + r] = d.axT[3 * r + k];
    }
    h->log_norm[i] = d.log_norm;
    h->weight[i] = d.weight;
    h->first_child[i] = d.first_child;
    h->child_count[i] = d.child_count;
    h->level[i] = d.level;
    h->parent[i] = d.parent;
  }
  return TRG_OK;
}

int trg_tree_free(trg_ctx* ctx, trg_tree_dev* t) {
  if (!t || t->ctx_scratch) return TRG_OK;
  if (ctx) cudaSetDevice(ctx->device);
  cudaFree(t->nodes);
  cudaFree(t->cov);
  delete t;
  return TRG_OK;
}


int trg_associate(trg_ctx* ctx, const trg_tree_dev* tree, const double* xyz, size_t n,
                  int xyz_on_device, const double R[9], const double t[3],
                  const trg_assoc_config* cfg, trg_moments* out, int* point_node,
                  double* point_weight) {
  trg::NvtxRange nvtx_range_("trg_associate");
  // association.cpp:43-50 validate_inputs, :95-102
  if (n == 0) {
    set_error("association: empty point cloud");
    return TRG_EINVAL;
  }
  if (!tree || tree->n_nodes == 0) {
    set_error("association: empty model");
    return TRG_EINVAL;
  }
  if (!(cfg->lambda_c >= 0.0 && cfg->lambda_c <= 1.0 / 3.0)) {
    set_error("association: lambda_c outside [0, 1/3]");
    return TRG_EINVAL;
  }
  const int depth = cfg->max_level == 0 ? tree->max_level : cfg->max_level;
  if (depth < 1 || depth > tree->max_level) {
    set_error("association: search depth exceeds tree depth");
    return TRG_EINVAL;
  }
  TRG_CU(cudaSetDevice(ctx->device));
  const int nm = out->m2 ? 10 : 4;
  const int J = tree->n_nodes;
  const int G = assoc_grid(ctx, nm);
  AssocParams p{};
  p.nodes = tree->nodes;
  p.n_nodes = J;
  p.root_count = tree->root_count;
  p.n_snodes = std::min(tree->n_upper, kStageNodes);
  p.depth = depth;
  p.lambda_c = cfg->lambda_c;
  p.outlier_floor = cfg->outlier_floor;
  p.n = n;
  p.status = ctx->status;
  TRG_TRY(stage_points_public(ctx, xyz, n, xyz_on_device, kSlotPoints, &p.pts));
  void *accv, *mom, *cnt, *rt;
  const size_t acc_bytes = sizeof(long long) * 3 * nm * (size_t)J;
  TRG_TRY(ws_get(ctx, kSlotPartials, acc_bytes, &accv));
  TRG_TRY(ws_get(ctx, kSlotMoments, sizeof(double) * nm * (size_t)J, &mom));
  TRG_TRY(ws_get(ctx, kSlotCounters, 64 + 12 * sizeof(double) + 64, &cnt));
  rt = static_cast<char*>(cnt) + 64;
  unsigned long long* pmax = reinterpret_cast<unsigned long long*>(static_cast<char*>(cnt) + 64 + 12 * sizeof(double));
  p.acc = static_cast<long long*>(accv);
  p.acc_stride = (size_t)J;
  p.pmax = reinterpret_cast<const double*>(pmax);
  p.counters = static_cast<unsigned long long*>(cnt);
  double hrt[12];
  for (int k = 0; k < 9; ++k) hrt[k] = R[k];
  for (int k = 0; k < 3; ++k) hrt[9 + k] = t[k];
  TRG_CU(trg_memcpy(ctx, rt, hrt, sizeof hrt, cudaMemcpyHostToDevice));
  p.Rt = static_cast<const double*>(rt);
  TRG_CU(cudaMemsetAsync(cnt, 0, 64, ctx->stream));
  TRG_CU(cudaMemsetAsync(pmax, 0, 8, ctx->stream));
  TRG_CU(cudaMemsetAsync(accv, 0, acc_bytes, ctx->stream));
  TRG_TRY(launch_absmax(ctx, p.pts, n, pmax, nullptr));
  if (point_node) {
    void *pn, *pw;
    TRG_TRY(ws_get(ctx, kSlotPointNode, sizeof(int) * n, &pn));
    TRG_TRY(ws_get(ctx, kSlotPointW, sizeof(double) * n, &pw));
    p.point_node = static_cast<int*>(pn);
    p.point_w = static_cast<double*>(pw);
  }
  TRG_TRY(launch_associate(ctx, p, nm, static_cast<double*>(mom), G));
  std::vector<double> hm((size_t)nm * J);
  unsigned long long hc[2];
  TRG_CU(trg_memcpy(ctx, hm.data(), mom, sizeof(double) * nm * J, cudaMemcpyDeviceToHost));
  TRG_CU(trg_memcpy(ctx, hc, cnt, sizeof hc, cudaMemcpyDeviceToHost));
  if (point_node) {
    TRG_CU(trg_memcpy(ctx, point_node, p.point_node, sizeof(int) * n, cudaMemcpyDeviceToHost));
    TRG_CU(trg_memcpy(ctx, point_weight, p.point_w, sizeof(double) * n, cudaMemcpyDeviceToHost));
  }
  TRG_TRY(check_status(ctx, "associate_adaptive"));
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

}  // extern "C"
