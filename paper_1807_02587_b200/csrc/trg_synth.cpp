// Host-side synthetic inputs (the data formats either side of the hot path).
//
// * trg_synthetic / trg_unit_normalize / trg_random_rigid_transform restate
//   the reference generators (synthetic.cpp:46-165, cloud_io.cpp:14-57,
//   511-532) with the same libstdc++ engines and distributions, so they
//   reproduce the reference's clouds bit-for-bit (checked against the
//   reference build in tests/test_synth.py).  The reference builds vectors
//   with unsequenced function-call arguments; g++ evaluates those right to
//   left, which is the draw order reproduced below.
// * trg_synth_kinect_pair / trg_synth_lidar_pair are the NEW frame-pair
//   generators of SURVEY.md §8d (configs C2 / C3): analytic ray casting of a
//   closed room through a 320x240 pinhole camera, and of an HDL-32-style
//   spinning sensor over a street scene.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <random>
#include <string>
#include <vector>

#include "../../include/treereg_b200.h"  // status codes
#include "../../include/treereg_b200_host.h"
#include "trg_raycast.h"

namespace {

using Rng = std::mt19937_64;

struct V3 {
  double x, y, z;
};
inline V3 add(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V3 mul(double s, V3 a) { return {s * a.x, s * a.y, s * a.z}; }
inline double dot(V3 a, V3 b) {
  double s = a.x * b.x;
  s += a.y * b.y;
  s += a.z * b.z;
  return s;
}
inline double norm(V3 a) { return std::sqrt(dot(a, a)); }

// synthetic.cpp:14-17: a fresh N(0, sigma) per call, x then y then z.
V3 noise(Rng& rng, double sigma) {
  std::normal_distribution<double> g(0.0, sigma);
  const double x = g(rng);
  const double y = g(rng);
  const double z = g(rng);
  return {x, y, z};
}

// synthetic.cpp:19-27 add_rect (right-to-left operand evaluation)
void add_rect(std::vector<V3>& pts, Rng& rng, V3 corner, V3 eu, V3 ev, std::size_t count,
              double sigma) {
  std::uniform_real_distribution<double> u(0.0, 1.0);
  for (std::size_t i = 0; i < count; ++i) {
    const V3 nz = noise(rng, sigma);
    const double b = u(rng);
    const double a = u(rng);
    pts.push_back(add(add(add(corner, mul(a, eu)), mul(b, ev)), nz));
  }
}

// Vec3(g(rng), g(rng), g(rng)) with right-to-left argument evaluation.
V3 gauss3(std::normal_distribution<double>& g, Rng& rng) {
  const double z = g(rng);
  const double y = g(rng);
  const double x = g(rng);
  return {x, y, z};
}

// synthetic.cpp:29-42 add_sphere
void add_sphere(std::vector<V3>& pts, Rng& rng, V3 center, double radius, std::size_t count,
                double sigma) {
  std::normal_distribution<double> g(0.0, 1.0);
  for (std::size_t i = 0; i < count; ++i) {
    V3 dir = gauss3(g, rng);
    const double n = norm(dir);
    if (n < 1e-12) {
      dir = {1, 0, 0};
    } else {
      dir = {dir.x / n, dir.y / n, dir.z / n};
    }
    const V3 nz = noise(rng, sigma);
    pts.push_back(add(add(center, mul(radius, dir)), nz));
  }
}

std::vector<V3> blobs(std::size_t n, double sigma, std::uint64_t seed) {  // :46-62
  std::vector<V3> pts;
  pts.reserve(n);
  Rng rng(seed);
  for (int corner = 0; corner < 8; ++corner) {
    const V3 c{static_cast<double>(corner & 1), static_cast<double>((corner >> 1) & 1),
               static_cast<double>((corner >> 2) & 1)};
    const std::size_t count = n / 8 + (static_cast<std::size_t>(corner) < n % 8);
    for (std::size_t i = 0; i < count; ++i) pts.push_back(add(c, noise(rng, sigma)));
  }
  return pts;
}

std::vector<V3> plane(std::size_t n, std::uint64_t seed) {  // :64-74
  std::vector<V3> pts;
  Rng rng(seed);
  std::uniform_real_distribution<double> u(0.0, 1.0);
  for (std::size_t i = 0; i < n; ++i) {
    const double b = u(rng);
    const double a = u(rng);
    pts.push_back({a, b, 0.0});
  }
  return pts;
}

std::vector<V3> sphere(std::size_t n, std::uint64_t seed) {  // :76-82
  std::vector<V3> pts;
  Rng rng(seed);
  add_sphere(pts, rng, {0, 0, 0}, 1.0, n, 0.0);
  return pts;
}

std::vector<V3> scene(std::size_t n, std::uint64_t seed) {  // :84-132
  std::vector<V3> pts;
  pts.reserve(n);
  Rng rng(seed);
  const double kNoise = 0.002;
  const std::size_t n_wall_z = n * 18 / 100;
  const std::size_t n_wall_x = n * 14 / 100;
  const std::size_t n_box = n * 16 / 100;
  const std::size_t n_ball = n * 12 / 100;
  const std::size_t n_ramp = n * 12 / 100;
  const std::size_t n_floor = n - n_wall_z - n_wall_x - n_box - n_ball - n_ramp;
  add_rect(pts, rng, {0, 0, 0}, {2, 0, 0}, {0, 0, 1.5}, n_floor, kNoise);
  add_rect(pts, rng, {0, 0, 0}, {2, 0, 0}, {0, 1, 0}, n_wall_z, kNoise);
  add_rect(pts, rng, {0, 0, 0}, {0, 0, 1.5}, {0, 1, 0}, n_wall_x, kNoise);
  {
    const V3 lo{1.2, 0.0, 0.9};
    const V3 dx{0.4, 0, 0}, dy{0, 0.35, 0}, dz{0, 0, 0.4};
    const double a_top = 0.4 * 0.4;
    const double a_x = 0.35 * 0.4;
    const double a_z = 0.4 * 0.35;
    const double total = a_top + 2 * a_x + 2 * a_z;
    const auto share = [&](double a) {
      return static_cast<std::size_t>(static_cast<double>(n_box) * a / total);
    };
    const std::size_t nx = share(a_x), nz = share(a_z);
    const std::size_t ntop = n_box - 2 * nx - 2 * nz;
    add_rect(pts, rng, add(lo, dy), dx, dz, ntop, kNoise);
    add_rect(pts, rng, lo, dy, dz, nx, kNoise);
    add_rect(pts, rng, add(lo, dx), dy, dz, nx, kNoise);
    add_rect(pts, rng, lo, dx, dy, nz, kNoise);
    add_rect(pts, rng, add(lo, dz), dx, dy, nz, kNoise);
  }
  add_sphere(pts, rng, {0.55, 0.3, 0.5}, 0.22, n_ball, kNoise);
  add_rect(pts, rng, {0.9, 0.0, 0.1}, {0.5, 0.0, 0.15}, {0.0, 0.4, 0.3}, n_ramp, kNoise);
  return pts;
}

std::vector<V3> lumpy(std::size_t n, std::uint64_t seed) {  // :134-157
  std::vector<V3> pts;
  pts.reserve(n);
  Rng rng(seed);
  std::normal_distribution<double> g(0.0, 1.0);
  while (pts.size() < n) {
    V3 dir = gauss3(g, rng);
    const double nr = norm(dir);
    if (nr < 1e-12) continue;
    dir = {dir.x / nr, dir.y / nr, dir.z / nr};
    const double theta = std::acos(std::clamp(dir.z, -1.0, 1.0));
    const double phi = std::atan2(dir.y, dir.x);
    const double radius =
        0.5 * (1.0 + 0.22 * std::sin(3.0 * theta) * std::sin(2.0 * phi) +
               0.18 * std::cos(2.0 * theta) * std::cos(3.0 * phi) +
               0.12 * std::sin(5.0 * phi) * std::sin(theta) + 0.08 * std::cos(4.0 * theta));
    const V3 nz = noise(rng, 0.002);
    pts.push_back(add(mul(radius, dir), nz));
  }
  return pts;
}

void store(const std::vector<V3>& pts, double* out) {
  for (std::size_t i = 0; i < pts.size(); ++i) {
    out[3 * i] = pts[i].x;
    out[3 * i + 1] = pts[i].y;
    out[3 * i + 2] = pts[i].z;
  }
}

std::uint64_t splitmix64(std::uint64_t x) {  // cloud_io.cpp:500-505
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

void matmul(const double a[9], const double b[9], double c[9]) {
  double t[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double s = a[3 * i] * b[j];
      s += a[3 * i + 1] * b[3 + j];
      s += a[3 * i + 2] * b[6 + j];
      t[3 * i + j] = s;
    }
  std::memcpy(c, t, sizeof t);
}

// geometry.cpp:120-129 rotation_from_euler_xyz = Rx * Ry * Rz
void euler_xyz(double a, double b, double c, double R[9]) {
  const double ca = std::cos(a), sa = std::sin(a);
  const double cb = std::cos(b), sb = std::sin(b);
  const double cc = std::cos(c), sc = std::sin(c);
  const double rx[9] = {1, 0, 0, 0, ca, -sa, 0, sa, ca};
  const double ry[9] = {cb, 0, sb, 0, 1, 0, -sb, 0, cb};
  const double rz[9] = {cc, -sc, 0, sc, cc, 0, 0, 0, 1};
  double t[9];
  matmul(rx, ry, t);
  matmul(t, rz, R);
}

void rigid(double rot_deg, double trans, std::uint64_t seed, int trial, double R[9],
           double t[3]) {
  Rng rng(splitmix64(seed ^ splitmix64(static_cast<std::uint64_t>(trial) + 1)));
  constexpr double kDegToRad = 0.017453292519943295;
  const double r = rot_deg * kDegToRad;
  std::uniform_real_distribution<double> rot(-r, r);
  std::uniform_real_distribution<double> tr(-trans, trans);
  for (int k = 0; k < 9; ++k) R[k] = (k % 4 == 0) ? 1.0 : 0.0;
  t[0] = t[1] = t[2] = 0.0;
  if (rot_deg > 0.0) {
    const double c = rot(rng);
    const double b = rot(rng);
    const double a = rot(rng);
    euler_xyz(a, b, c, R);
  }
  if (trans > 0.0) {
    const double z = tr(rng);
    const double y = tr(rng);
    const double x = tr(rng);
    t[0] = x;
    t[1] = y;
    t[2] = z;
  }
}

// p -> R p + t
V3 apply(const double R[9], const double t[3], V3 p) {
  double s0 = R[0] * p.x;
  s0 += R[1] * p.y;
  s0 += R[2] * p.z;
  double s1 = R[3] * p.x;
  s1 += R[4] * p.y;
  s1 += R[5] * p.z;
  double s2 = R[6] * p.x;
  s2 += R[7] * p.y;
  s2 += R[8] * p.z;
  return {s0 + t[0], s1 + t[1], s2 + t[2]};
}

// ------------------------------------------------------- ray casting (new)
// The scenes and the per-pixel / per-beam casts live in trg_raycast.h, shared
// with the device renderer (trg_render.cu): the same operations in the same
// order on both sides.

// Camera-to-world pose for a Kinect frame: looks from (3.4,1.5,2.6) at the
// room corner area.  Camera axes: x right, y down, z forward.
void look_at(V3 eye, V3 target, double R[9], double t[3]) {
  V3 f = sub(target, eye);
  f = mul(1.0 / norm(f), f);
  const V3 up{0, 1, 0};
  V3 xr{f.y * up.z - f.z * up.y, f.z * up.x - f.x * up.z, f.x * up.y - f.y * up.x};
  xr = mul(1.0 / norm(xr), xr);
  const V3 yd{f.y * xr.z - f.z * xr.y, f.z * xr.x - f.x * xr.z, f.x * xr.y - f.y * xr.x};
  // columns of R = camera axes in world coordinates
  R[0] = xr.x; R[1] = yd.x; R[2] = f.x;
  R[3] = xr.y; R[4] = yd.y; R[5] = f.y;
  R[6] = xr.z; R[7] = yd.z; R[8] = f.z;
  t[0] = eye.x; t[1] = eye.y; t[2] = eye.z;
}

// The axial-noise draws of one frame: one N(0, 1) per pixel in pixel order
// (a fresh distribution per frame, as render_kinect draws them).
void frame_normals(Rng& rng, std::size_t n, double* out) {
  std::normal_distribution<double> g(0.0, 1.0);
  for (std::size_t i = 0; i < n; ++i) out[i] = g(rng);
}

// Renders one 320x240 frame from camera pose (Rwc, twc); points in camera
// coordinates, axial noise sigma_z = 0.0012 + 0.0019 (z - 0.4)^2.
void render_kinect(const double Rwc[9], const double twc[3], Rng& rng, double* out,
                   double noise_scale) {
  std::normal_distribution<double> g(0.0, 1.0);
  std::size_t k = 0;
  for (int v = 0; v < 240; ++v)
    for (int u = 0; u < 320; ++u, k += 3) trg_rc::kinect_pixel(Rwc, twc, u, v, g(rng), noise_scale, out + k);
}

// HDL-32 beam directions: azimuth a (2250 steps of 0.16 deg), elevation b
// (32 beams from -30.67 deg by 1.3333 deg); cos / sin tables [cos 2250 | sin
// 2250 | cos 32 | sin 32] (libm on the host; the device renderer takes them)
void lidar_tables(double* tab) {
  constexpr double kDeg = 0.017453292519943295;
  for (int a = 0; a < 2250; ++a) {
    const double az = a * 0.16 * kDeg;
    tab[a] = std::cos(az);
    tab[2250 + a] = std::sin(az);
  }
  for (int b = 0; b < 32; ++b) {
    const double el = (-30.67 + 1.3333 * b) * kDeg;
    tab[4500 + b] = std::cos(el);
    tab[4532 + b] = std::sin(el);
  }
}

void render_lidar(const double Rws[9], const double tws[3], Rng& rng, double* out) {
  std::normal_distribution<double> g(0.0, 1.0);
  double tab[4564];
  lidar_tables(tab);
  std::size_t k = 0;
  for (int a = 0; a < 2250; ++a)
    for (int b = 0; b < 32; ++b, k += 3) {
      const trg_rc::V3 ds{tab[4500 + b] * tab[a], tab[4500 + b] * tab[2250 + a], tab[4532 + b]};
      trg_rc::lidar_beam(Rws, tws, ds, g(rng), out + k);
    }
}

// Relative pose: source frame -> target frame, given both sensor->world poses.
void relative(const double R1[9], const double t1[3], const double R2[9], const double t2[3],
              double R[9], double t[3]) {
  // T = T1^-1 * T2 : R = R1^T R2, t = R1^T (t2 - t1)
  double r1t[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r1t[3 * i + j] = R1[3 * j + i];
  matmul(r1t, R2, R);
  const double d[3] = {t2[0] - t1[0], t2[1] - t1[1], t2[2] - t1[2]};
  for (int i = 0; i < 3; ++i) t[i] = r1t[3 * i] * d[0] + r1t[3 * i + 1] * d[1] + r1t[3 * i + 2] * d[2];
}

}  // namespace

extern "C" {

int trg_synthetic(const char* kind, size_t n, uint64_t seed, double* out) {
  const std::string k(kind ? kind : "");
  std::vector<V3> pts;
  if (k == "blobs") {
    if (n < 8) return TRG_EINVAL;
    pts = blobs(n, 0.01, seed);
  } else if (k == "plane") {
    if (n == 0) return TRG_EINVAL;
    pts = plane(n, seed);
  } else if (k == "sphere") {
    if (n == 0) return TRG_EINVAL;
    pts = sphere(n, seed);
  } else if (k == "scene") {
    if (n < 20) return TRG_EINVAL;
    pts = scene(n, seed);
  } else if (k == "lumpy") {
    if (n == 0) return TRG_EINVAL;
    pts = lumpy(n, seed);
  } else {
    return TRG_EINVAL;
  }
  store(pts, out);
  return TRG_OK;
}

double trg_bbox_diagonal(const double* p, size_t n) {  // cloud_io.cpp:21-33
  if (n == 0) return 0.0;
  double lo[3] = {p[0], p[1], p[2]}, hi[3] = {p[0], p[1], p[2]};
  for (size_t i = 0; i < n; ++i)
    for (int k = 0; k < 3; ++k) {
      const double v = p[3 * i + k];
      lo[k] = (v < lo[k]) ? v : lo[k];
      hi[k] = (hi[k] < v) ? v : hi[k];
    }
  const V3 d{hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]};
  return norm(d);
}

int trg_unit_normalize(double* p, size_t n) {  // cloud_io.cpp:48-57
  if (n == 0) return TRG_OK;
  double c[3] = {0, 0, 0};
  for (size_t i = 0; i < n; ++i)
    for (int k = 0; k < 3; ++k) c[k] = c[k] + p[3 * i + k];
  for (int k = 0; k < 3; ++k) c[k] = c[k] / static_cast<double>(n);
  const double diag = trg_bbox_diagonal(p, n);
  const double s = diag > 0.0 ? 1.0 / diag : 1.0;
  for (size_t i = 0; i < n; ++i)
    for (int k = 0; k < 3; ++k) p[3 * i + k] = (p[3 * i + k] - c[k]) * s;
  return TRG_OK;
}

int trg_random_rigid_transform(double rot_deg, double trans, uint64_t seed, int trial, double R[9],
                               double t[3]) {
  if (trial < 0) return TRG_EINVAL;
  rigid(rot_deg, trans, seed, trial, R, t);
  return TRG_OK;
}

}  // extern "C"

namespace {
// Camera poses of a Kinect pair: camera 2 = camera 1 moved by
// random_rigid_transform({rot_deg, trans}, trial 0) in its own frame.
void kinect_pair_poses(uint64_t seed, double rot_deg, double trans, double R1[9], double t1[3],
                       double R2[9], double t2[3]) {
  look_at({3.4, 1.5, 2.6}, {1.2, 0.7, 0.9}, R1, t1);
  double dR[9], dt[3];
  rigid(rot_deg, trans, seed, 0, dR, dt);
  matmul(R1, dR, R2);
  for (int i = 0; i < 3; ++i)
    t2[i] = t1[i] + R1[3 * i] * dt[0] + R1[3 * i + 1] * dt[1] + R1[3 * i + 2] * dt[2];
}

// Sensor poses of a LiDAR pair: 1 m forward + 2 deg yaw, then a small
// random perturbation.
void lidar_pair_poses(uint64_t seed, double R1[9], double t1[3], double R2[9], double t2[3]) {
  constexpr double kDeg = 0.017453292519943295;
  for (int k = 0; k < 9; ++k) R1[k] = (k % 4 == 0) ? 1.0 : 0.0;
  t1[0] = 0.0;
  t1[1] = 0.0;
  t1[2] = 1.8;
  const double c = std::cos(2.0 * kDeg), s = std::sin(2.0 * kDeg);
  const double Rego[9] = {c, -s, 0, s, c, 0, 0, 0, 1};
  double dR[9], dt[3];
  rigid(1.0, 0.05, seed, 0, dR, dt);
  matmul(Rego, dR, R2);
  t2[0] = 1.0 + dt[0];
  t2[1] = dt[1];
  t2[2] = 1.8 + dt[2];
}
}  // namespace

extern "C" {

int trg_synth_kinect_pair_ex(uint64_t seed, double noise_scale, double rot_deg, double trans,
                             double* target, double* source, double R_gt[9], double t_gt[3]) {
  double R1[9], t1[3], R2[9], t2[3];
  kinect_pair_poses(seed, rot_deg, trans, R1, t1, R2, t2);
  Rng rng(splitmix64(seed + 0x4b696e656374ull));
  render_kinect(R1, t1, rng, target, noise_scale);
  render_kinect(R2, t2, rng, source, noise_scale);
  relative(R1, t1, R2, t2, R_gt, t_gt);
  return TRG_OK;
}

int trg_synth_kinect_pair_plan(uint64_t seed, double rot_deg, double trans, double Rwc[18],
                               double twc[6], double* noise, double R_gt[9], double t_gt[3]) {
  if (!Rwc || !twc || !noise || !R_gt || !t_gt) return TRG_EINVAL;
  kinect_pair_poses(seed, rot_deg, trans, Rwc, twc, Rwc + 9, twc + 3);
  Rng rng(splitmix64(seed + 0x4b696e656374ull));
  frame_normals(rng, 76800, noise);
  frame_normals(rng, 76800, noise + 76800);
  relative(Rwc, twc, Rwc + 9, twc + 3, R_gt, t_gt);
  return TRG_OK;
}

int trg_synth_lidar_pair_plan(uint64_t seed, double Rws[18], double tws[6], double* noise,
                              double* dir_tables, double R_gt[9], double t_gt[3]) {
  if (!Rws || !tws || !noise || !dir_tables || !R_gt || !t_gt) return TRG_EINVAL;
  lidar_pair_poses(seed, Rws, tws, Rws + 9, tws + 3);
  Rng rng(splitmix64(seed + 0x4c69444152ull));
  frame_normals(rng, 72000, noise);
  frame_normals(rng, 72000, noise + 72000);
  lidar_tables(dir_tables);
  relative(Rws, tws, Rws + 9, tws + 3, R_gt, t_gt);
  return TRG_OK;
}

int trg_synth_kinect_sequence(uint64_t seed, int frames, double step_rot_deg, double step_trans,
                              double* out, double* R_gt, double* t_gt) {
  if (frames < 1 || !out || !R_gt || !t_gt) return TRG_EINVAL;
  double R0[9], t0[3];
  look_at({3.4, 1.5, 2.6}, {1.2, 0.7, 0.9}, R0, t0);
  double Rk[9], tk[3];
  for (int i = 0; i < 9; ++i) Rk[i] = R0[i];
  for (int i = 0; i < 3; ++i) tk[i] = t0[i];
  Rng rng(splitmix64(seed + 0x53657175656e6365ull));
  for (int k = 0; k < frames; ++k) {
    if (k > 0) {  // camera k = camera k-1 moved by a random step in its own frame
      double dR[9], dt[3], Rn[9], tn[3];
      rigid(step_rot_deg, step_trans, seed, k, dR, dt);
      matmul(Rk, dR, Rn);
      for (int i = 0; i < 3; ++i)
        tn[i] = tk[i] + Rk[3 * i] * dt[0] + Rk[3 * i + 1] * dt[1] + Rk[3 * i + 2] * dt[2];
      for (int i = 0; i < 9; ++i) Rk[i] = Rn[i];
      for (int i = 0; i < 3; ++i) tk[i] = tn[i];
    }
    render_kinect(Rk, tk, rng, out + (size_t)k * 76800 * 3, 1.0);
    relative(R0, t0, Rk, tk, R_gt + 9 * (size_t)k, t_gt + 3 * (size_t)k);  // frame k -> frame 0
  }
  return TRG_OK;
}

int trg_synth_kinect_pair(uint64_t seed, double* target, double* source, double R_gt[9],
                          double t_gt[3]) {
  return trg_synth_kinect_pair_ex(seed, 1.0, 5.0, 0.05, target, source, R_gt, t_gt);
}

int trg_synth_lidar_pair(uint64_t seed, double* target, double* source, double R_gt[9],
                         double t_gt[3]) {
  double R1[9], t1[3], R2[9], t2[3];
  lidar_pair_poses(seed, R1, t1, R2, t2);
  Rng rng(splitmix64(seed + 0x4c69444152ull));
  render_lidar(R1, t1, rng, target);
  render_lidar(R2, t2, rng, source);
  relative(R1, t1, R2, t2, R_gt, t_gt);
  return TRG_OK;
}

}  // extern "C"
