// Spatially sorted copy of a cloud for the association passes (calibration
// and EM E-steps).  Their deposits are exact fixed-point sums of per-window
// run sums (trg_fx.cuh), so the order of the points changes the results only
// by the rounding of those short FP64 run sums (the sorted order is itself
// deterministic, so grid invariance and run-to-run reproducibility hold).
// The copy makes each 32-point window's descents share nodes (L1 hits) and
// their stop nodes form long runs, so a window deposits a few run sums
// instead of up to 32 x (3 limbs x NM values) integer reductions.  Clouds
// generated in scan order (C2, C3) already have this locality; a large
// cloud in arbitrary order (C4, synthetic_scene) did not: its calibration
// association took 411 us per pass (190 us sorted), its EM 18.7 ms (6.9 ms).
#include <cub/device/device_radix_sort.cuh>

#include "trg_internal.cuh"

namespace trg {

// 30-bit Morton code of a point quantised to 10 bits per axis over
// [-pmax, pmax]^3.
__device__ __forceinline__ unsigned spread10(unsigned v) {
  v &= 0x3ffu;
  v = (v | (v << 16)) & 0x030000ffu;
  v = (v | (v << 8)) & 0x0300f00fu;
  v = (v | (v << 4)) & 0x030c30c3u;
  v = (v | (v << 2)) & 0x09249249u;
  return v;
}

__global__ void k_morton_keys(const double* __restrict__ pts, size_t n, const double* pmax,
                              unsigned* keys, unsigned* idx) {
  const double m = __ldcg(pmax);
  const double s = m > 0.0 ? 1023.0 / (2.0 * m) : 0.0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    unsigned q[3];
    for (int k = 0; k < 3; ++k) {
      const double v = (pts[3 * i + k] + m) * s;
      q[k] = (unsigned)fmin(fmax(v, 0.0), 1023.0);
    }
    keys[i] = spread10(q[0]) | (spread10(q[1]) << 1) | (spread10(q[2]) << 2);
    idx[i] = (unsigned)i;
  }
}

__global__ void k_gather_points(const double* __restrict__ pts, const unsigned* __restrict__ idx,
                                size_t n, double* out) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const size_t j = idx[i];
    out[3 * i] = pts[3 * j];
    out[3 * i + 1] = pts[3 * j + 1];
    out[3 * i + 2] = pts[3 * j + 2];
  }
}

// A Morton-ordered copy of pts (n points) in workspace slot `slot_pts`
// (scratch: `slot_tmp`), queued on the context's stream; *out points to it.
// pmax: the cloud's max |coordinate| on the device (already computed on the
// stream).  Clouds in (kSortMaxSmall, kSortMinPoints) are used as they are.
int morton_sorted_copy(trg_ctx* ctx, const double* pts, size_t n, const double* pmax, int slot_pts,
                       int slot_tmp, const double** out) {
  *out = pts;
  if ((n > kSortMaxSmall && n < kSortMinPoints) || n < 64 || n > 0xffffffffull) return TRG_OK;
  size_t temp = 0;
  unsigned* null = nullptr;
  TRG_CU(cub::DeviceRadixSort::SortPairs(nullptr, temp, null, null, null, null, (int)n, 0, 30,
                                         ctx->stream));
  const size_t kb = (sizeof(unsigned) * n + 255) & ~size_t(255);
  void* tmp = nullptr;
  TRG_TRY(ws_get(ctx, slot_tmp, 4 * kb + temp, &tmp));
  char* T = static_cast<char*>(tmp);
  unsigned *k0 = (unsigned*)T, *k1 = (unsigned*)(T + kb), *i0 = (unsigned*)(T + 2 * kb),
           *i1 = (unsigned*)(T + 3 * kb);
  void* sorted = nullptr;
  TRG_TRY(ws_get(ctx, slot_pts, sizeof(double) * 3 * n, &sorted));
  const int blocks = 4 * ctx->device_sms;
  k_morton_keys<<<blocks, 256, 0, ctx->stream>>>(pts, n, pmax, k0, i0);
  TRG_CU(cub::DeviceRadixSort::SortPairs(T + 4 * kb, temp, k0, k1, i0, i1, (int)n, 0, 30,
                                         ctx->stream));
  k_gather_points<<<blocks, 256, 0, ctx->stream>>>(pts, i1, n, static_cast<double*>(sorted));
  ctx->launches += 3;
  TRG_CU(cudaGetLastError());
  *out = static_cast<const double*>(sorted);
  return TRG_OK;
}

}  // namespace trg
