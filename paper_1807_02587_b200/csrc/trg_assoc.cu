// K7 associate_descend: standalone E-step kernels (trg_associate C-ABI).
// The same device code (trg_assoc.cuh) runs inside the fused registration
// and calibration kernels.
#include "trg_assoc.cuh"

namespace trg {

template <int NM>
__global__ void __launch_bounds__(kAssocBlock) k_assoc(AssocParams p) {
  __shared__ AssocSmem<NM> sm;
  __shared__ double rt[12];
  extern __shared__ __align__(16) unsigned char k_assoc_stage[];  // p.n_snodes DNodes
  if (p.Rt && threadIdx.x < 12) rt[threadIdx.x] = p.Rt[threadIdx.x];
  DNode* sn = reinterpret_cast<DNode*>(k_assoc_stage);
  stage_nodes(sn, p.nodes, p.n_snodes);
  p.snodes = sn;
  assoc_pass<NM>(sm, p, p.Rt ? rt : nullptr, gridDim.x, blockIdx.x);
}

template <int NM>
__global__ void __launch_bounds__(256) k_combine(const double* __restrict__ partials,
                                                 const uint32_t* __restrict__ stamps,
                                                 uint32_t epoch, int G, int J,
                                                 double* __restrict__ out) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (warp >= J) return;
  double acc[NM];
  combine_node<NM>(partials, stamps, epoch, G, warp, acc);
  if ((threadIdx.x & 31) == 0)
#pragma unroll
    for (int m = 0; m < NM; ++m) out[(size_t)warp * NM + m] = acc[m];
}

int assoc_grid(trg_ctx* ctx, int nm) {
  int per_sm = 1;
  const size_t stage = sizeof(DNode) * kStageNodes;
  cudaFuncSetAttribute(k_assoc<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)stage);
  cudaFuncSetAttribute(k_assoc<10>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)stage);
  if (nm == 4)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_assoc<4>, kAssocBlock, stage);
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_assoc<10>, kAssocBlock, stage);
  if (per_sm < 1) per_sm = 1;
  return ctx->sms * per_sm;
}

int launch_associate(trg_ctx* ctx, const AssocParams& p, int nm, double* moments, int grid) {
  const int cblocks = (p.n_nodes * 32 + 255) / 256;
  const size_t stage = sizeof(DNode) * (size_t)p.n_snodes;
  if (nm == 4) {
    k_assoc<4><<<grid, kAssocBlock, stage, ctx->stream>>>(p);
    k_combine<4><<<cblocks, 256, 0, ctx->stream>>>(p.partials, p.stamps, p.epoch, grid,
                                                   p.n_nodes, moments);
  } else {
    k_assoc<10><<<grid, kAssocBlock, stage, ctx->stream>>>(p);
    k_combine<10><<<cblocks, 256, 0, ctx->stream>>>(p.partials, p.stamps, p.epoch, grid,
                                                    p.n_nodes, moments);
  }
  ctx->launches += 2;
  TRG_CU(cudaGetLastError());
  return TRG_OK;
}

int launch_combine(trg_ctx* ctx, const double* partials, const uint32_t* stamps, uint32_t epoch,
                   int G, int J, int nm, double* out) {
  const int cblocks = (J * 32 + 255) / 256;
  if (nm == 4)
    k_combine<4><<<cblocks, 256, 0, ctx->stream>>>(partials, stamps, epoch, G, J, out);
  else
    k_combine<10><<<cblocks, 256, 0, ctx->stream>>>(partials, stamps, epoch, G, J, out);
  ctx->launches += 1;
  TRG_CU(cudaGetLastError());
  return TRG_OK;
}

}  // namespace trg
