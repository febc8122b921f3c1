// Device frame renderer of the synthetic Kinect / LiDAR inputs (SURVEY.md
// 8f rank 3, configs C2 / C3 / C5): one thread per pixel / beam ray-casts
// the scene of trg_raycast.h -- the same source the host generator
// (trg_synth.cpp) runs, compiled here with -fmad=false, so given the poses,
// noise draws and beam directions of trg_synth_*_pair_plan (libtrg_host.so)
// a frame is bit-identical to the host generator's.  The sequential parts
// (the mt19937_64 / normal_distribution draws, libm trigonometry) stay on
// the host; the per-ray work (a few hundred FP64 operations per point, 3.7
// MB of points per pair) moves to the GPU and never crosses PCIe.
#include <algorithm>
#include <cstring>
#include <vector>

#include "trg_internal.cuh"
#include "trg_raycast.h"

namespace {

constexpr int kKinectPixels = 320 * 240;
constexpr int kLidarBeams = 2250 * 32;

// poses: [frames][12] = R (9, sensor -> world) then t (3)
__global__ void k_render_kinect(int frames, const double* __restrict__ poses,
                                const double* __restrict__ noise, double noise_scale,
                                double* __restrict__ out) {
  const size_t n = (size_t)frames * kKinectPixels;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const int f = (int)(i / kKinectPixels), pix = (int)(i % kKinectPixels);
    const double* P = poses + 12 * (size_t)f;
    double o[3];
    trg_rc::kinect_pixel(P, P + 9, pix % 320, pix / 320, noise ? noise[i] : 0.0, noise_scale, o);
    out[3 * i] = o[0];
    out[3 * i + 1] = o[1];
    out[3 * i + 2] = o[2];
  }
}

// tab: [cos az 2250 | sin az 2250 | cos el 32 | sin el 32]
__global__ void k_render_lidar(int frames, const double* __restrict__ poses,
                               const double* __restrict__ noise, const double* __restrict__ tab,
                               double* __restrict__ out) {
  const size_t n = (size_t)frames * kLidarBeams;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const int f = (int)(i / kLidarBeams), beam = (int)(i % kLidarBeams);
    const int a = beam / 32, b = beam % 32;
    const double* P = poses + 12 * (size_t)f;
    const trg_rc::V3 ds{tab[4500 + b] * tab[a], tab[4500 + b] * tab[2250 + a], tab[4532 + b]};
    double o[3];
    trg_rc::lidar_beam(P, P + 9, ds, noise ? noise[i] : 0.0, o);
    out[3 * i] = o[0];
    out[3 * i + 1] = o[1];
    out[3 * i + 2] = o[2];
  }
}

// Poses, noise draws and tables into one device buffer (one staged copy).
int stage_render_inputs(trg_ctx* ctx, int frames, const double* R, const double* t,
                        const double* noise, size_t per_frame, const double* tab, size_t ntab,
                        double** poses_d, double** noise_d, double** tab_d) {
  const size_t np = 12 * (size_t)frames, nn = noise ? per_frame * frames : 0;
  std::vector<double> h(np + nn + ntab);
  for (int f = 0; f < frames; ++f) {
    for (int k = 0; k < 9; ++k) h[12 * (size_t)f + k] = R[9 * (size_t)f + k];
    for (int k = 0; k < 3; ++k) h[12 * (size_t)f + 9 + k] = t[3 * (size_t)f + k];
  }
  if (nn) std::memcpy(h.data() + np, noise, sizeof(double) * nn);
  if (ntab) std::memcpy(h.data() + np + nn, tab, sizeof(double) * ntab);
  void* d = nullptr;
  TRG_TRY(ws_get(ctx, trg::kSlotRender, sizeof(double) * h.size(), &d));
  TRG_CU(trg::trg_memcpy(ctx, d, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice));
  double* base = static_cast<double*>(d);
  *poses_d = base;
  *noise_d = nn ? base + np : nullptr;
  *tab_d = ntab ? base + np + nn : nullptr;
  return TRG_OK;
}

}  // namespace

using namespace trg;

extern "C" {

int trg_render_kinect_frames(trg_ctx* ctx, int frames, const double* Rwc, const double* twc,
                             const double* noise, double noise_scale, double* out) {
  trg::NvtxRange nvtx_range_("trg_render_kinect_frames");
  if (!ctx || frames < 1 || !Rwc || !twc || !out) {
    set_error("render_kinect_frames: bad argument");
    return TRG_EINVAL;
  }
  TRG_CU(cudaSetDevice(ctx->device));
  double *pd = nullptr, *nd = nullptr, *td = nullptr;
  TRG_TRY(stage_render_inputs(ctx, frames, Rwc, twc, noise, kKinectPixels, nullptr, 0, &pd, &nd, &td));
  const size_t n = (size_t)frames * kKinectPixels;
  k_render_kinect<<<(unsigned)std::min<size_t>((n + 255) / 256, 8u * ctx->device_sms), 256, 0,
                    ctx->stream>>>(frames, pd, nd, noise_scale, out);
  ctx->launches += 1;
  TRG_CU(cudaGetLastError());
  return TRG_OK;
}

int trg_render_lidar_frames(trg_ctx* ctx, int frames, const double* Rws, const double* tws,
                            const double* noise, const double* dir_tables, double* out) {
  trg::NvtxRange nvtx_range_("trg_render_lidar_frames");
  if (!ctx || frames < 1 || !Rws || !tws || !dir_tables || !out) {
    set_error("render_lidar_frames: bad argument");
    return TRG_EINVAL;
  }
  TRG_CU(cudaSetDevice(ctx->device));
  double *pd = nullptr, *nd = nullptr, *td = nullptr;
  TRG_TRY(stage_render_inputs(ctx, frames, Rws, tws, noise, kLidarBeams, dir_tables, 4564, &pd, &nd,
                              &td));
  const size_t n = (size_t)frames * kLidarBeams;
  k_render_lidar<<<(unsigned)std::min<size_t>((n + 255) / 256, 8u * ctx->device_sms), 256, 0,
                   ctx->stream>>>(frames, pd, nd, td, out);
  ctx->launches += 1;
  TRG_CU(cudaGetLastError());
  return TRG_OK;
}

}  // extern "C"
