// Point-sharded execution (north_star "large clouds shard by
// point, per-node moment vectors all-reduced over NVLink"): communicators and
// the collectives the sharded build / calibration / EM segments exchange
// between launches.
//
// NCCL is bound at run time (dlopen of libnccl.so.2: the copy torch already
// loaded when there is one) so the library has no link-time NCCL dependency;
// nccl.h supplies only the types.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <string>
#include <vector>

#include "trg_internal.cuh"

namespace {

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
};

NcclApi* nccl_api() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api.h ? &api : nullptr;
  tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
  if (!h) return nullptr;
  api.getUniqueId = (decltype(api.getUniqueId))dlsym(h, "ncclGetUniqueId");
  api.commInitRank = (decltype(api.commInitRank))dlsym(h, "ncclCommInitRank");
  api.commDestroy = (decltype(api.commDestroy))dlsym(h, "ncclCommDestroy");
  api.allReduce = (decltype(api.allReduce))dlsym(h, "ncclAllReduce");
  api.allGather = (decltype(api.allGather))dlsym(h, "ncclAllGather");
  api.getErrorString = (decltype(api.getErrorString))dlsym(h, "ncclGetErrorString");
  if (!api.getUniqueId || !api.commInitRank || !api.commDestroy || !api.allReduce ||
      !api.allGather || !api.getErrorString)
    return nullptr;
  api.h = h;
  return &api;
}

int nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return TRG_OK;
  NcclApi* a = nccl_api();
  trg::set_error(std::string(what) + ": " + (a ? a->getErrorString(r) : "nccl error"));
  return TRG_ENCCL;
}

constexpr int kMaxLocalShards = 16;
struct ShardPtrs {
  double* p[kMaxLocalShards];
};

// Sum over the local shards in shard order, written back to every shard.
__global__ void k_shard_sum(ShardPtrs b, int shards, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    double s = b.p[0][i];
    for (int k = 1; k < shards; ++k) s += b.p[k][i];
    for (int k = 0; k < shards; ++k) b.p[k][i] = s;
  }
}

}  // namespace

namespace trg {

int comm_allreduce_sum(trg_comm* c, double* const* bufs, size_t n) {
  if (n == 0) return TRG_OK;
  cudaStream_t st = c->ctx->stream;
  if (c->nccl) {
    return nccl_check(nccl_api()->allReduce(bufs[0], bufs[0], n, ncclFloat64, ncclSum,
                                            (ncclComm_t)c->nccl, st),
                      "ncclAllReduce");
  }
  if (c->local == 1) return TRG_OK;
  ShardPtrs b{};
  for (int k = 0; k < c->local; ++k) b.p[k] = bufs[k];
  const int blocks = (int)std::min<size_t>(4 * (size_t)c->ctx->device_sms, (n + 255) / 256);
  k_shard_sum<<<blocks, 256, 0, st>>>(b, c->local, n);
  c->ctx->launches += 1;
  TRG_CU(cudaGetLastError());
  return TRG_OK;
}

int comm_allgather(trg_comm* c, double* const* src, double* const* dst, size_t n) {
  if (n == 0) return TRG_OK;
  cudaStream_t st = c->ctx->stream;
  if (c->nccl) {
    return nccl_check(nccl_api()->allGather(src[0], dst[0], n, ncclFloat64, (ncclComm_t)c->nccl,
                                            st),
                      "ncclAllGather");
  }
  for (int j = 0; j < c->local; ++j)
    for (int k = 0; k < c->local; ++k)
      TRG_CU(cudaMemcpyAsync(dst[j] + (size_t)k * n, src[k], sizeof(double) * n,
                             cudaMemcpyDeviceToDevice, st));
  return TRG_OK;
}

int comm_host_reduce(trg_comm* c, double* vals, int n, int op) {
  auto fold = [&](double a, double b) {
    return op == 0 ? a + b : op == 1 ? (a < b ? b : a) : (b < a ? b : a);
  };
  for (int k = 1; k < c->local; ++k)
    for (int i = 0; i < n; ++i) vals[i] = fold(vals[i], vals[(size_t)k * n + i]);
  if (c->nccl) {
    cudaStream_t st = c->ctx->stream;
    TRG_CU(cudaMemcpyAsync(c->dscratch, vals, sizeof(double) * n, cudaMemcpyHostToDevice, st));
    const ncclRedOp_t ro = op == 0 ? ncclSum : op == 1 ? ncclMax : ncclMin;
    TRG_TRY(nccl_check(nccl_api()->allReduce(c->dscratch, c->dscratch, n, ncclFloat64, ro,
                                             (ncclComm_t)c->nccl, st),
                       "ncclAllReduce"));
    TRG_CU(cudaMemcpyAsync(vals, c->dscratch, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    TRG_CU(cudaStreamSynchronize(st));
  }
  for (int k = 1; k < c->local; ++k)
    for (int i = 0; i < n; ++i) vals[(size_t)k * n + i] = vals[i];
  return TRG_OK;
}

}  // namespace trg

using namespace trg;

extern "C" {

int trg_comm_unique_id(unsigned char id[128]) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId");
  NcclApi* a = nccl_api();
  if (!a) {
    set_error("trg_comm_unique_id: libnccl.so.2 not found");
    return TRG_ENCCL;
  }
  ncclUniqueId u;
  TRG_TRY(nccl_check(a->getUniqueId(&u), "ncclGetUniqueId"));
  std::memcpy(id, &u, 128);
  return TRG_OK;
}

static int comm_alloc(trg_ctx* ctx, trg_comm** out) {
  auto* c = new trg_comm;
  c->ctx = ctx;
  if (cudaMalloc(&c->dscratch, 4096) != cudaSuccess) {
    cudaGetLastError();
    delete c;
    set_error("trg_comm: cudaMalloc failed");
    return TRG_ECUDA;
  }
  c->shard_ctx.push_back(ctx);
  *out = c;
  return TRG_OK;
}

int trg_comm_create_nccl(trg_ctx* ctx, const unsigned char id[128], int rank, int world,
                         trg_comm** out) {
  if (!ctx || !id || !out || world < 1 || rank < 0 || rank >= world) {
    set_error("trg_comm_create_nccl: bad argument");
    return TRG_EINVAL;
  }
  NcclApi* a = nccl_api();
  if (!a) {
    set_error("trg_comm_create_nccl: libnccl.so.2 not found");
    return TRG_ENCCL;
  }
  TRG_CU(cudaSetDevice(ctx->device));
  trg_comm* c = nullptr;
  TRG_TRY(comm_alloc(ctx, &c));
  ncclUniqueId u;
  std::memcpy(&u, id, 128);
  ncclComm_t nc = nullptr;
  const int rc = nccl_check(a->commInitRank(&nc, world, u, rank), "ncclCommInitRank");
  if (rc != TRG_OK) {
    cudaFree(c->dscratch);
    delete c;
    return rc;
  }
  c->nccl = nc;
  c->rank = rank;
  c->world = world;
  c->local = 1;
  *out = c;
  return TRG_OK;
}

int trg_comm_create_local(trg_ctx* ctx, int shards, trg_comm** out) {
  if (!ctx || !out || shards < 1 || shards > kMaxLocalShards) {
    set_error("trg_comm_create_local: shards must be in 1..16");
    return TRG_EINVAL;
  }
  TRG_CU(cudaSetDevice(ctx->device));
  trg_comm* c = nullptr;
  TRG_TRY(comm_alloc(ctx, &c));
  c->world = shards;
  c->local = shards;
  for (int k = 1; k < shards; ++k) {
    trg_ctx* s = nullptr;
    const int rc = trg_ctx_create(ctx->device, &s);
    if (rc != TRG_OK) {
      trg_comm_destroy(c);
      return rc;
    }
    cudaStreamDestroy(s->stream);  // shards run in order on the parent's stream
    s->stream = ctx->stream;
    s->own_stream = false;
    c->shard_ctx.push_back(s);
  }
  *out = c;
  return TRG_OK;
}

int trg_comm_destroy(trg_comm* c) {
  if (!c) return TRG_OK;
  if (c->ctx) cudaSetDevice(c->ctx->device);
  if (c->ctx) cudaStreamSynchronize(c->ctx->stream);
  if (c->nccl && nccl_api()) nccl_api()->commDestroy((ncclComm_t)c->nccl);
  for (size_t k = 1; k < c->shard_ctx.size(); ++k) trg_ctx_destroy(c->shard_ctx[k]);
  cudaFree(c->dscratch);
  delete c;
  return TRG_OK;
}

int trg_comm_rank(trg_comm* c) { return c ? c->rank : -1; }
int trg_comm_world(trg_comm* c) { return c ? c->world : 0; }
int trg_comm_local_shards(trg_comm* c) { return c ? c->local : 0; }

}  // extern "C"
