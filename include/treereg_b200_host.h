/* libtrg_host.so -- host-only companion of libtrg_cuda.so.
 *
 * Cloud ingest (the reference's cloud_io: read_cloud, subsample) and the
 * synthetic inputs (the reference's generators restated + the new Kinect /
 * LiDAR frame-pair generators of SURVEY.md 8d).  Byte-serial parsing and
 * sequential RNG streams: host code by design.  Kept out of the
 * product library, so a CPU-only caller (bench.py's reference arm) can make
 * the inputs without loading any device code.  Errors: the same status codes;
 * messages through trg_host_last_error(). */
#ifndef TREEREG_B200_HOST_H
#define TREEREG_B200_HOST_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* trg_host_last_error(void);

/* ---- ingest (host code) ---------------------------
 * treereg::read_cloud (cloud_io.hpp, cloud_io.cpp:401-427): format 0 = by
 * content ("ply" magic, else XYZ text), 1 = PLY ascii, 2 = PLY
 * binary_little_endian, 3 = XYZ text.  *xyz is malloc'd (N x 3, free with
 * trg_free_cloud); parse errors return TRG_ERUNTIME (ParseError). */
int trg_read_cloud(const char* path, int format, double** xyz, size_t* n);
void trg_free_cloud(double* xyz);
/* treereg::subsample (cloud_io.cpp:477-498): selection sampling of m of n
 * points in index order, std::mt19937_64(seed) -- identical picks. */
int trg_subsample(const double* xyz, size_t n, size_t m, uint64_t seed, double* out);

/* ---- host-side data (synthetic inputs; the reference's generators,
 *      synthetic.cpp / cloud_io.cpp, restated + the new Kinect / LiDAR
 *      frame-pair generators of SURVEY.md §8d) -------------------------- */
int trg_synthetic(const char* kind, size_t n, uint64_t seed, double* out);
int trg_unit_normalize(double* xyz, size_t n);
double trg_bbox_diagonal(const double* xyz, size_t n);
int trg_random_rigid_transform(double rot_range_deg, double trans_range, uint64_t seed, int trial,
                               double R[9], double t[3]);
/* 320x240 Kinect-style depth-frame pair (76,800 points each).  R_gt, t_gt map
 * the source frame into the target frame. */
int trg_synth_kinect_pair(uint64_t seed, double* target, double* source, double R_gt[9],
                          double t_gt[3]);
/* Same with explicit axial-noise scale and camera-motion ranges. */
int trg_synth_kinect_pair_ex(uint64_t seed, double noise_scale, double rot_range_deg,
                             double trans_range, double* target, double* source, double R_gt[9],
                             double t_gt[3]);
/* A Kinect-style frame sequence (frames x 76,800 points): camera k is
 * camera k-1 moved by random_rigid_transform({step_rot_deg, step_trans},
 * trial k) in its own frame; R_gt/t_gt [frames][9]/[3] map frame k into
 * frame 0 (the trajectory a sequence registration recovers). */
int trg_synth_kinect_sequence(uint64_t seed, int frames, double step_rot_deg, double step_trans,
                              double* out, double* R_gt, double* t_gt);
/* HDL-32-style sweep pair (72,000 points each). */
int trg_synth_lidar_pair(uint64_t seed, double* target, double* source, double R_gt[9],
                         double t_gt[3]);
/* The sequential parts of the two pair generators, for the device renderer
 * (trg_render_kinect_frames / trg_render_lidar_frames, libtrg_cuda.so): the
 * sensor poses of both frames (R[f]: 9 doubles sensor -> world, t[f]: 3),
 * the noise draws of both frames in pixel / beam order (noise: 2 x 76,800
 * resp. 2 x 72,000 doubles), the LiDAR beam direction tables (dir_tables:
 * 4,564 doubles: cos / sin of the 2,250 azimuths, cos / sin of the 32
 * elevations) and the ground truth.  Rendering from them reproduces
 * trg_synth_kinect_pair_ex(seed, noise_scale, rot, trans, ...) /
 * trg_synth_lidar_pair(seed, ...) bit for bit. */
int trg_synth_kinect_pair_plan(uint64_t seed, double rot_range_deg, double trans_range,
                               double R[18], double t[6], double* noise, double R_gt[9],
                               double t_gt[3]);
int trg_synth_lidar_pair_plan(uint64_t seed, double R[18], double t[6], double* noise,
                              double* dir_tables, double R_gt[9], double t_gt[3]);

#ifdef __cplusplus
}
#endif
#endif
