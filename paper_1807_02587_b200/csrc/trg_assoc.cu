// K7 associate_descend: standalone E-step kernels (trg_associate C-ABI).
// The same device code (trg_assoc.cuh) runs inside the fused registration
// and calibration kernels.
#include "trg_dense.cuh"

namespace trg {

template <int NM>
__global__ void __launch_bounds__(kAssocBlock) k_assoc(AssocParams p) {
  __shared__ double rt[12];
  __shared__ FxScale sc[3];
  __shared__ __align__(8) uint64_t bar;
  extern __shared__ __align__(128) unsigned char k_assoc_stage[];  // p.n_snodes DNodes
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
  }
  if (p.Rt && threadIdx.x < 12) rt[threadIdx.x] = p.Rt[threadIdx.x];
  __syncthreads();
  if (threadIdx.x == 0) assoc_scales(p.pmax, p.Rt ? rt : nullptr, sc);
  DNode* sn = reinterpret_cast<DNode*>(k_assoc_stage);
  unsigned phase = 0;
  stage_nodes_bulk(sn, p.nodes, p.n_snodes, &bar, phase);
  __syncthreads();
  p.snodes = sn;
  const int wpb = kAssocBlock / 32;
  assoc_fx_pass<NM>(p, p.Rt ? rt : nullptr, sc, gridDim.x * wpb, (threadIdx.x >> 5) * gridDim.x + blockIdx.x);
}

// acc[J][NM][3] -> out[J][NM] (doubles), one thread per value.
template <int NM>
__global__ void __launch_bounds__(256) k_fx_out(const long long* __restrict__ acc,
                                                const double* pmax, const double* Rt, int J,
                                                double* __restrict__ out) {
  __shared__ FxScale sc[3];
  __shared__ double rt[12];
  if (Rt && threadIdx.x < 12) rt[threadIdx.x] = Rt[threadIdx.x];
  __syncthreads();
  if (threadIdx.x == 0) assoc_scales(pmax, Rt ? rt : nullptr, sc);
  __syncthreads();
  constexpr int kOrd[10] = {0, 1, 1, 1, 2, 2, 2, 2, 2, 2};
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= J * NM) return;
  const int j = i / NM, m = i % NM;
  out[i] = fx_load(acc, (size_t)J, j, m, sc[kOrd[m]].down);
}

__global__ void k_absmax(const double* __restrict__ p, size_t n3, unsigned long long* bits,
                         int* status) {
  double m = 0.0;
  bool bad = false;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n3;
       i += (size_t)gridDim.x * blockDim.x) {
    const double v = p[i];
    bad |= !isfinite(v);
    m = fmax(m, fabs(v));
  }
  m = block_max_nonneg(m);  // one atomic per block (per-warp atomics serialised on one word)
  if (threadIdx.x == 0 && m > 0.0) atomicMax(bits, (unsigned long long)__double_as_longlong(m));
  if (bad && status) atomicCAS(status, 0, kEInval);
}

int launch_absmax(trg_ctx* ctx, const double* pts, size_t n, unsigned long long* pmax_bits,
                  int* status) {
  if (n == 0) return TRG_OK;
  const int blocks = (int)std::min<size_t>(128, (3 * n + 255) / 256);
  k_absmax<<<blocks, 256, 0, ctx->stream>>>(pts, 3 * n, pmax_bits, status);
  ctx->launches += 1;
  TRG_CU(cudaGetLastError());
  return TRG_OK;
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

// p.acc must be zeroed (J * nm * 3 limbs) and *p.pmax set before the launch.
int launch_associate(trg_ctx* ctx, const AssocParams& p, int nm, double* moments, int grid) {
  const size_t stage = sizeof(DNode) * (size_t)p.n_snodes;
  const int ob = (p.n_nodes * nm + 255) / 256;
  if (nm == 4) {
    k_assoc<4><<<grid, kAssocBlock, stage, ctx->stream>>>(p);
    k_fx_out<4><<<ob, 256, 0, ctx->stream>>>(p.acc, p.pmax, p.Rt, p.n_nodes, moments);
  } else {
    k_assoc<10><<<grid, kAssocBlock, stage, ctx->stream>>>(p);
    k_fx_out<10><<<ob, 256, 0, ctx->stream>>>(p.acc, p.pmax, p.Rt, p.n_nodes, moments);
  }
  ctx->launches += 2;
  TRG_CU(cudaGetLastError());
  return TRG_OK;
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
