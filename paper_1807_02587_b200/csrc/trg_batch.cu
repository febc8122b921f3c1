// trg_register_batch: independent frame pairs (BASELINE config C5).
// Tree variants (adaptive / tree): waves of pairs whose builds and EMs run
// as single cooperative launches, one CTA group per pair
// (register_batch_fused, trg_em.cu).  Flat / ICP variants run as concurrent
// registrations: each worker owns an SM-budgeted sub-context
// (own stream, workspace and scratch tree; persistent grids sized to
// device_sms / streams SMs: the budgets sum to the device, so the grids are
// normally co-resident -- not guaranteed for plain launches, hence the spin
// guards of trg_internal.cuh, which fail a call instead of hanging) and pulls
// pair indices from a shared counter.  Host work per pair is launch/staging
// only; the GPU overlaps one pair's latency-bound phases (grid barriers,
// eigen-solves, calibration climbs) with the others' E-step tiles.
#include <atomic>
#include <string>
#include <thread>
#include <vector>

#include "trg_internal.cuh"

using namespace trg;

extern "C" int trg_register_batch(trg_ctx* ctx, int n_pairs, const double* const* targets,
                                  const size_t* n_targets, const double* const* sources,
                                  const size_t* n_sources, int on_device,
                                  const trg_reg_config* cfg, int streams, trg_reg_result* out) {
  trg::NvtxRange nvtx_range_("trg_register_batch");
  if (!ctx || n_pairs < 0 || (n_pairs > 0 && (!targets || !n_targets || !sources || !n_sources ||
                                               !cfg || !out))) {
    set_error("register_batch: bad argument");
    return TRG_EINVAL;
  }
  const bool fused =
      cfg && (cfg->variant_kind == TRG_VARIANT_ADAPTIVE || cfg->variant_kind == TRG_VARIANT_TREE);
  if (streams == 0) streams = fused ? kBatchInflightDefault : 4;
  if (streams < 1 || streams > (fused ? kBatchInflightMax : 16)) {
    set_error(fused ? "register_batch: pairs in flight must be in 1..24"
                    : "register_batch: streams must be in 1..16");
    return TRG_EINVAL;
  }
  if (n_pairs == 0) return TRG_OK;
  if (fused) {
    TRG_CU(cudaSetDevice(ctx->device));
    return register_batch_fused(ctx, n_pairs, targets, n_targets, sources, n_sources, on_device,
                                cfg, streams, out);
  }
  streams = std::min(streams, n_pairs);
  const int budget = std::max(1, ctx->device_sms / streams);
  while ((int)ctx->workers.size() < streams) {
    trg_ctx* w = nullptr;
    TRG_TRY(trg_ctx_create(ctx->device, &w));
    ctx->workers.push_back(w);
  }
  for (int k = 0; k < streams; ++k) TRG_TRY(trg_ctx_set_sm_budget(ctx->workers[k], budget));
  // inputs the caller produced on its own stream must be complete
  TRG_CU(cudaStreamSynchronize(ctx->stream));
  std::vector<int> rc(n_pairs, TRG_OK);
  std::vector<std::string> msg(n_pairs);
  std::atomic<int> next{0};
  std::vector<uint64_t> l0(streams), h0(streams), d0(streams);
  for (int k = 0; k < streams; ++k) {
    l0[k] = ctx->workers[k]->launches;
    h0[k] = ctx->workers[k]->bytes_h2d;
    d0[k] = ctx->workers[k]->bytes_d2h;
  }
  auto work = [&](int k) {
    trg_ctx* w = ctx->workers[k];
    cudaSetDevice(w->device);
    for (;;) {
      const int i = next.fetch_add(1);
      if (i >= n_pairs) break;
      rc[i] = trg_register_clouds(w, targets[i], n_targets[i], sources[i], n_sources[i], on_device,
                                  cfg, &out[i]);
      if (rc[i] != TRG_OK) msg[i] = trg_last_error();
    }
  };
  std::vector<std::thread> th;
  for (int k = 1; k < streams; ++k) th.emplace_back(work, k);
  work(0);
  for (auto& t : th) t.join();
  for (int k = 0; k < streams; ++k) {
    ctx->launches += ctx->workers[k]->launches - l0[k];
    ctx->bytes_h2d += ctx->workers[k]->bytes_h2d - h0[k];
    ctx->bytes_d2h += ctx->workers[k]->bytes_d2h - d0[k];
  }
  for (int i = 0; i < n_pairs; ++i)
    if (rc[i] != TRG_OK) {
      set_error("register_batch: pair " + std::to_string(i) + ": " + msg[i]);
      return rc[i];
    }
  return TRG_OK;
}
