// Internal declarations shared by the CUDA translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/treereg_b200.h"
#include "trg_math.cuh"
#include "trg_fx.cuh"

#include <nvtx3/nvToolsExt.h>  // header-only; ranges cost nothing without a tool attached

namespace trg {
// NVTX range over one C-ABI call (visible in Nsight Systems / ncu --nvtx).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
}  // namespace trg

namespace trg {

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);
#define TRG_CU(expr)                                                              \
  do {                                                                            \
    cudaError_t e_ = (expr);                                                      \
    if (e_ != cudaSuccess) {                                                      \
      ::trg::set_error(std::string(#expr) + ": " + cudaGetErrorString(e_));       \
      return TRG_ECUDA;                                                           \
    }                                                                             \
  } while (0)
#define TRG_TRY(expr)            \
  do {                           \
    int rc_ = (expr);            \
    if (rc_ != TRG_OK) return rc_; \
  } while (0)

// ------------------------------------------------------- device records
// Packed per-node record used by every scoring loop (association, EM).
// axT[3*l + k] = axes(k, l): row l is the unit axis of lam[l].
struct __align__(16) DNode {
  double mean[3];
  double axT[9];
  double lam[3];
  double il[3];  // 1 / lam (scoring loops multiply instead of divide)
  double log_norm;
  double weight;
  double cplx;  // node_complexity (gmm.cpp:53-59); -1 when trace <= 0
  double pad;
  int first_child, child_count;
  int level, parent;
  double prec[6];  // precision matrix for fast_q (set_prec): P00, 2P01, 2P02, P11, 2P12, P22
};
static_assert(sizeof(DNode) == 240, "DNode layout");

// Hot-loop Gaussian: log N(x) = log_norm - q/2 with q = sum_l (n_l.d)^2 / lam_l
// (gmm.cpp:41-46) evaluated as the quadratic form d^T P d of the precision
// matrix P = sum_l a_l a_l^T / lam_l (set_prec, once per covariance update):
// 12 FP64 operations per density instead of the 18 of the axis projections.
// The value agrees with the reference's to ~eps x cond(cov) relative
// (covariances are floored at 1e-4 of their trace: <= ~1e-11), far inside
// the documented near-tie band (1e-6 in log-score) of the association parity
// and the 1e-4 parameter tolerance of the build; all eigen/solve math stays
// in the reference's order.
__device__ __forceinline__ double fast_q(const double* mean, const double* P, double x0, double x1,
                                         double x2) {
  const double d0 = x0 - mean[0], d1 = x1 - mean[1], d2 = x2 - mean[2];
  const double u0 = __fma_rn(P[2], d2, __fma_rn(P[1], d1, __dmul_rn(P[0], d0)));
  const double u1 = __fma_rn(P[4], d2, __dmul_rn(P[3], d1));
  return __fma_rn(d0, u0, __fma_rn(d1, u1, __dmul_rn(__dmul_rn(P[5], d2), d2)));
}

}  // namespace trg

struct trg_tree_dev {
  int n_nodes = 0, max_level = 0, capacity = 0, root_count = 0;
  int n_upper = 0;  // nodes above the deepest level (BFS prefix; staged in smem by the descent)
  trg::DNode* nodes = nullptr;  // [capacity]
  double* cov = nullptr;        // [capacity*9] row-major
  int* owner_ctx_device = nullptr;
  bool ctx_scratch = false;  // owned by a context (register_clouds' model); free is a no-op
};

namespace trg {
// Device timeline written by the persistent kernels (globaltimer ns per mark;
// label conventions in include/treereg_b200.h, trg_debug_build_timeline).
struct Timeline {
  int n;
  int lab[1024];
  unsigned long long t[1024];
};
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Spin-wait guard: a wait that exceeds 10 s can only be a grid whose CTAs
// are not all resident (e.g. SM-budgeted batch workers sharing the device):
// trap (the launch fails with an error the host reports) instead of hanging.
__device__ __forceinline__ void spin_guard(unsigned long long t0) {
  if (gtimer() - t0 > 10000000000ull) __trap();
}
// The same, reading the clock only every 64th poll (the polls stay cheap:
// a polling thread shares its SM's issue slots with working CTAs).
__device__ __forceinline__ void spin_guard_every(unsigned long long t0, unsigned& polls) {
  if ((++polls & 63u) == 0u) spin_guard(t0);
}
// Max of non-negative doubles over the block (result in thread 0; exact, so
// any order); block size a multiple of 32, at most 1024.
__device__ __forceinline__ double block_max_nonneg(double v) {
  __shared__ double wm[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    v = threadIdx.x < (blockDim.x >> 5) ? wm[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  }
  return v;
}
__device__ __forceinline__ void tl_mark_any(Timeline* tl, int label) {
  const int i = atomicAdd(&tl->n, 1);
  if (i < 1024) {
    tl->lab[i] = label;
    tl->t[i] = gtimer();
  }
}
__device__ __forceinline__ void tl_mark(Timeline* tl, int label) {
  if (blockIdx.x == 0 && threadIdx.x == 0) tl_mark_any(tl, label);
}
}  // namespace trg

struct trg_ctx {
  int device = 0;
  uint64_t bytes_h2d = 0, bytes_d2h = 0;
  double build_growth = 0.0;  // largest E_max / N a build on this context needed
  int sms = 0;         // SMs this context's persistent grids may use (trg_ctx_set_sm_budget)
  int device_sms = 0;
  cudaStream_t stream = nullptr;
  uint64_t launches = 0;
  uint32_t epoch = 1;
  trg_tree_dev* scratch_tree = nullptr;  // reused by register_clouds (no cudaMalloc/cudaFree per call)
  bool build_into_scratch = false;
  bool timeline_pending = false;
  std::vector<trg_ctx*> workers;  // trg_register_batch: SM-budgeted sub-contexts
  bool own_stream = true;         // false: a shard context on its parent's stream
  cudaStream_t side = nullptr;    // copy stream: a pinned source cloud's H2D under the build
  cudaEvent_t side_done = nullptr;
  cudaEvent_t ext_ready = nullptr;  // trg_ctx_wait_stream
  static constexpr int kSlots = 32;
  void* slot_ptr[kSlots] = {};
  size_t slot_size[kSlots] = {};
  void* host_slot_ptr[kSlots] = {};
  size_t host_slot_size[kSlots] = {};
  int* status = nullptr;  // device status word
  int* status2 = nullptr;  // second word: the EM of an asynchronous register_clouds
  trg::Timeline* dev_timeline = nullptr;      // device buffer (reset per call)
  std::vector<unsigned long long> timeline;  // last call: globaltimer ns per mark
  std::vector<int> timeline_lab;
};

// Point-sharded execution (trg_comm_*).  NCCL mode: one shard
// per process, `world` processes (one per GPU).  Local mode: `world` shards
// driven by this process on one device (each on its own shard context that
// shares the parent's stream), exchanged by a device reduction in fixed
// shard order — the same segmented algorithm, runnable on one GPU.
struct trg_comm {
  trg_ctx* ctx = nullptr;
  int rank = 0, world = 1;
  int local = 1;                       // shards this process drives
  std::vector<trg_ctx*> shard_ctx;     // [local]; shard_ctx[0] == ctx
  void* nccl = nullptr;                // ncclComm_t (NCCL mode)
  double* dscratch = nullptr;          // device scratch for host-value reductions
};

namespace trg {

// Workspace slots (device memory, grown on demand, never shrunk).
enum Slot : int {
  kSlotPoints = 0,
  kSlotPartials,
  kSlotStamps,
  kSlotMoments,
  kSlotCounters,
  kSlotPointNode,
  kSlotPointW,
  kSlotSolve,
  kSlotEm,
  kSlotEmTrace,
  kSlotBuild0,
  kSlotBuild1,
  kSlotBuild2,
  kSlotBuild3,
  kSlotBuild4,
  kSlotBuild5,
  kSlotBuild6,
  kSlotBuild7,
  kSlotBuild8,
  kSlotBuild9,
  kSlotBuild10,
  kSlotBuild11,
  kSlotPoints2,
  kSlotDense,         // dense association: per-point score sums
  kSlotHostStage,     // host slots only: pinned staging for pageable copies
  kSlotTimelineHost,  // host slots only: last device timeline
  kSlotHostEmInit,    // host slots only: pinned EmState initialiser (no staging sync)
  kSlotHostBuildInit, // host slots only: pinned BuildState initialiser
  kSlotHostCollect,   // host slots only: a call's results, fetched with one synchronisation
  kSlotRender,        // frame renderer (trg_render.cu): poses, noise draws, direction tables
};

int ws_get(trg_ctx* ctx, int slot, size_t bytes, void** out);
// trg_sort.cu: a Morton-ordered copy of a cloud for the association passes
// (locality of the descents and of the deposit runs).  Large clouds (the
// sort pays at any order) and small ones (the sort is a few microseconds of
// fixed cost; C1's unordered 10k points: +6 %) are sorted; the mid-size
// organised scans in between (C2 / C3: raster / sweep order, already
// coherent) are used as they are (sorting C2: -3 %).
constexpr size_t kSortMinPoints = 262144, kSortMaxSmall = 32768;
int morton_sorted_copy(trg_ctx* ctx, const double* pts, size_t n, const double* pmax, int slot_pts,
                       int slot_tmp, const double** out);

// Every host<->device copy of the library goes through here (byte counters
// back the e2e h2d/d2h figures of bench.py).  Pinned host buffers are copied
// asynchronously on the context's stream; pageable ones are staged through
// the context's pinned buffer (a pageable cudaMemcpyAsync holds driver locks
// that serialise every other context's launches), which makes those copies
// complete before the call returns.
cudaError_t trg_memcpy(trg_ctx* ctx, void* dst, const void* src, size_t bytes, cudaMemcpyKind kind);
int host_ws_get(trg_ctx* ctx, int slot, size_t bytes, void** out);
// Collectives over a trg_comm, stream-ordered on comm->ctx->stream.  bufs /
// src / dst hold one device pointer per local shard.
int comm_allreduce_sum(trg_comm* c, double* const* bufs, size_t n);
int comm_allgather(trg_comm* c, double* const* src, double* const* dst, size_t n);
// vals: [local][n] host values (one row per local shard); on return row 0
// (and every row) holds the reduction over all shards.  op: 0 sum, 1 max, 2 min.
int comm_host_reduce(trg_comm* c, double* vals, int n, int op);
int check_model_config(const trg_model_config* cfg);  // validate_config gmm.cpp:465-477
int check_finite_dev(trg_ctx* ctx, const double* dev, size_t n, const char* msg);
// Device pointer to N x 3 points: the caller's (on_device) or a staged copy.
int stage_points_public(trg_ctx* ctx, const double* xyz, size_t n, int on_device, int slot,
                        const double** dev);
// As stage_points_public, but a pinned host cloud is copied on the context's
// side stream (overlapping whatever the main stream runs meanwhile); *deferred
// tells the caller to stage_wait() before the main stream reads it.
int stage_points_side(trg_ctx* ctx, const double* xyz, size_t n, int on_device, int slot,
                      const double** dev, bool* deferred);
int stage_wait(trg_ctx* ctx);
// register_icp_pt2pt (registration.cpp:211-298) over device clouds.
int register_icp_dev(trg_ctx* ctx, const double* tgt, size_t nt, const double* src, size_t ns,
                     const trg_reg_config* cfg, double diag, trg_reg_result* out);
// build_flat_gmm (gmm.cpp:659-736) over a device cloud -> J-root mixture.
int flat_build(trg_ctx* ctx, const double* dev, size_t n, size_t J, const trg_model_config* cfg,
               trg_tree_dev** out, trg_build_diag* diag);
// Sharded build over device-resident shard clouds (trg_build.cu).
int build_sharded_dev(trg_comm* c, const double* const* dev, const size_t* n,
                      const trg_model_config* cfg, trg_tree_dev** trees, trg_build_diag* diag);
int check_status(trg_ctx* ctx, const char* where);
int check_status_at(trg_ctx* ctx, int* dev_status, const char* where);
// A status word already fetched (value st): clears the device word and sets
// the error like check_status_at.
int status_result(trg_ctx* ctx, int st, int* dev_status, const char* where);
// What k_calibrate publishes about the finished tree for work queued behind
// it without a host round trip (ok = 0: the build failed or overflowed).
struct TreeMeta {
  int ok, J, root_count, n_upper;
};
// Asynchronous build (register_clouds): launch the build, queue work behind
// it, then collect.  finish() sets *retry when the entry buffers overflowed
// (the queued work saw meta->ok == 0 and did nothing); start() again reuses
// the grown allocation.
struct AsyncBuild;
int build_async_start(trg_ctx* ctx, const double* dev, size_t n, const trg_model_config* cfg,
                      AsyncBuild** h, trg_tree_dev** tree, const TreeMeta** meta, bool launch = true);
int build_batch_launch(trg_ctx* ctx, AsyncBuild* const* hs, int m);
// trg_register_batch of tree-variant pairs: waves of `inflight` pairs, each
// wave's builds and EMs as single launches (trg_em.cu)
constexpr int kBatchInflightDefault = 24, kBatchInflightMax = 24;
int register_batch_fused(trg_ctx* ctx, int n_pairs, const double* const* targets,
                         const size_t* n_targets, const double* const* sources,
                         const size_t* n_sources, int on_device, const trg_reg_config* cfg,
                         int inflight, trg_reg_result* out);
int build_async_finish(trg_ctx* ctx, AsyncBuild* h, trg_tree_dev** out, bool* retry);
void build_async_free(AsyncBuild* h);
int timeline_reset(trg_ctx* ctx);
int timeline_fetch(trg_ctx* ctx);
int tree_alloc(trg_ctx* ctx, int capacity, trg_tree_dev** out);

// Grid size for persistent kernels: SMs x resident CTAs.
int persistent_grid(trg_ctx* ctx, const void* kernel, int block, size_t smem);
// cudaFuncAttributeMaxDynamicSharedMemorySize, set once per kernel (cached).
cudaError_t set_dynamic_smem(const void* kernel, size_t bytes);
// Launches a persistent (grid-barrier) kernel of G = persistent_grid() CTAs.
// Whole-device contexts use a cooperative launch (co-residency checked by
// the driver).  SM-budgeted contexts (trg_ctx_set_sm_budget) use a plain
// launch so several contexts' persistent kernels run concurrently: their
// budgets sum to at most the device's SMs, which makes co-residency likely
// but not guaranteed -- every spin-wait is guarded (spin_guard).
cudaError_t launch_persistent(trg_ctx* ctx, const void* kernel, int G, int block, void** args,
                              size_t smem = 0);

// ---- association (trg_assoc.cu)
struct AssocParams {
  const DNode* nodes;
  int n_nodes, root_count, depth;
  double lambda_c, outlier_floor;
  const double* pts;  // N*3 AoS
  size_t n;
  const double* Rt;  // device: R[9], t[3] (nullable => identity)
  // tree path: exact fixed-point accumulators acc[J][NM][3] (trg_fx.cuh)
  long long* acc;
  size_t acc_stride;   // node stride of the planar limbs (>= n_nodes)
  const double* pmax;  // device: max |coordinate| of pts (the accumulators' scale)
  // dense path (flat mixture): per-(component, chunk) rows, stamped
  double* partials;  // [J][G][NM]
  uint32_t* stamps;  // [J][G]
  uint32_t epoch;
  unsigned long long* counters;  // outliers, evals (atomic adds of integers)
  int* point_node;               // nullable
  double* point_w;               // nullable
  int* status;
  // nodes [0, n_snodes) read from a shared-memory copy (the calling kernel
  // stages them): the tree's upper levels, visited by every point
  const trg::DNode* snodes;
  int n_snodes;
  Timeline* tl;  // probes only (TRG_ASSOC_PROBE)
};
int launch_associate(trg_ctx* ctx, const AssocParams& p, int nm, double* moments /*[J][nm]*/,
                     int grid);
// max |coordinate| of a device cloud into *pmax_bits (bits of a double >= 0;
// the caller zeroes it first); also flags non-finite coordinates (status).
int launch_absmax(trg_ctx* ctx, const double* pts, size_t n, unsigned long long* pmax_bits,
                  int* status);
int assoc_grid(trg_ctx* ctx, int nm);
// Per-node fixed-order combine of epoch-stamped partial rows -> out[J][nm].
int launch_combine(trg_ctx* ctx, const double* partials, const uint32_t* stamps, uint32_t epoch,
                   int G, int J, int nm, double* out);

}  // namespace trg
