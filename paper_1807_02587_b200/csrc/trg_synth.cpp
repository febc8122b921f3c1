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
constexpr double kInf = std::numeric_limits<double>::infinity();

struct Ray {
  V3 o, d;
};

// Axis-aligned box, inside (room: ray starts inside) or outside hit.
double hit_box_outside(const Ray& r, V3 lo, V3 hi) {
  double t0 = 0.0, t1 = kInf;
  const double o[3] = {r.o.x, r.o.y, r.o.z}, d[3] = {r.d.x, r.d.y, r.d.z};
  const double l[3] = {lo.x, lo.y, lo.z}, h[3] = {hi.x, hi.y, hi.z};
  for (int k = 0; k < 3; ++k) {
    if (std::fabs(d[k]) < 1e-15) {
      if (o[k] < l[k] || o[k] > h[k]) return kInf;
      continue;
    }
    double a = (l[k] - o[k]) / d[k], b = (h[k] - o[k]) / d[k];
    if (a > b) std::swap(a, b);
    t0 = std::max(t0, a);
    t1 = std::min(t1, b);
    if (t0 > t1) return kInf;
  }
  return t0 > 1e-9 ? t0 : kInf;
}

double hit_box_inside(const Ray& r, V3 lo, V3 hi) {
  double t = kInf;
  const double o[3] = {r.o.x, r.o.y, r.o.z}, d[3] = {r.d.x, r.d.y, r.d.z};
  const double l[3] = {lo.x, lo.y, lo.z}, h[3] = {hi.x, hi.y, hi.z};
  for (int k = 0; k < 3; ++k) {
    if (d[k] > 0) t = std::min(t, (h[k] - o[k]) / d[k]);
    if (d[k] < 0) t = std::min(t, (l[k] - o[k]) / d[k]);
  }
  return t;
}

double hit_sphere(const Ray& r, V3 c, double rad) {
  const V3 oc = sub(r.o, c);
  const double a = dot(r.d, r.d);  // ray directions are not unit length
  const double b = dot(oc, r.d), cc = dot(oc, oc) - rad * rad;
  const double disc = b * b - a * cc;
  if (disc < 0) return kInf;
  const double t = (-b - std::sqrt(disc)) / a;
  return t > 1e-9 ? t : kInf;
}

// Parallelogram corner + a*eu + b*ev, a,b in [0,1].
double hit_panel(const Ray& r, V3 corner, V3 eu, V3 ev) {
  const V3 n{eu.y * ev.z - eu.z * ev.y, eu.z * ev.x - eu.x * ev.z, eu.x * ev.y - eu.y * ev.x};
  const double dn = dot(r.d, n);
  if (std::fabs(dn) < 1e-15) return kInf;
  const double t = dot(sub(corner, r.o), n) / dn;
  if (!(t > 1e-9)) return kInf;
  const V3 p = sub(add(r.o, mul(t, r.d)), corner);
  const double uu = dot(eu, eu), vv = dot(ev, ev), uv = dot(eu, ev);
  const double pu = dot(p, eu), pv = dot(p, ev);
  const double det = uu * vv - uv * uv;
  const double a = (pu * vv - pv * uv) / det, b = (pv * uu - pu * uv) / det;
  return (a >= 0 && a <= 1 && b >= 0 && b <= 1) ? t : kInf;
}

// Closed room: synthetic_scene's layout scaled x2 (metres), y up.
double cast_room(const Ray& r) {
  double t = hit_box_inside(r, {0, 0, 0}, {4, 2.4, 3});
  t = std::min(t, hit_box_outside(r, {2.4, 0.0, 1.8}, {3.2, 0.7, 2.6}));
  t = std::min(t, hit_sphere(r, {1.1, 0.6, 1.0}, 0.44));
  t = std::min(t, hit_panel(r, {1.8, 0.0, 0.2}, {1.0, 0.0, 0.3}, {0.0, 0.8, 0.6}));
  return t;
}

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

// Renders one 320x240 frame from camera pose (Rwc, twc); points in camera
// coordinates, axial noise sigma_z = 0.0012 + 0.0019 (z - 0.4)^2.
void render_kinect(const double Rwc[9], const double twc[3], Rng& rng, double* out,
                   double noise_scale) {
  const double fx = 262.5, fy = 262.5, cx = 159.5, cy = 119.5;
  std::normal_distribution<double> g(0.0, 1.0);
  std::size_t k = 0;
  for (int v = 0; v < 240; ++v)
    for (int u = 0; u < 320; ++u) {
      const V3 dc{(u - cx) / fx, (v - cy) / fy, 1.0};
      const V3 dw{Rwc[0] * dc.x + Rwc[1] * dc.y + Rwc[2] * dc.z,
                  Rwc[3] * dc.x + Rwc[4] * dc.y + Rwc[5] * dc.z,
                  Rwc[6] * dc.x + Rwc[7] * dc.y + Rwc[8] * dc.z};
      const Ray r{{twc[0], twc[1], twc[2]}, dw};
      const double t = cast_room(r);  // z = t since dc.z == 1
      const double z = std::isfinite(t) ? t : 6.0;
      const double sz = 0.0012 + 0.0019 * (z - 0.4) * (z - 0.4);
      const double zn = z + noise_scale * sz * g(rng);
      out[k++] = dc.x * zn;
      out[k++] = dc.y * zn;
      out[k++] = zn;
    }
}

// HDL-32 street: ground z = 0, building boxes, poles, enclosing cylinder.
double cast_street(const Ray& r) {
  double t = kInf;
  if (r.d.z < 0) t = -r.o.z / r.d.z;
  static const double boxes[][6] = {
      {8, -20, 0, 20, -9, 9},  {-25, -22, 0, -10, -8, 14}, {-6, 10, 0, 12, 24, 7},
      {25, 6, 0, 40, 18, 11},  {-40, 12, 0, -28, 30, 16},  {-18, -45, 0, 5, -34, 10},
      {30, -30, 0, 44, -16, 8}, {3, -6, 0, 5, -4, 1.2}};
  for (const auto& b : boxes)
    t = std::min(t, hit_box_outside(r, {b[0], b[1], b[2]}, {b[3], b[4], b[5]}));
  static const double poles[][3] = {{6, 4, 0.15}, {-5, 5, 0.2}, {14, -3, 0.15},
                                    {-12, -4, 0.25}, {2, 12, 0.15}, {-3, -14, 0.2}};
  for (const auto& p : poles) {  // vertical cylinders of height 6 m
    const double ox = r.o.x - p[0], oy = r.o.y - p[1];
    const double a = r.d.x * r.d.x + r.d.y * r.d.y;
    if (a < 1e-15) continue;
    const double b = ox * r.d.x + oy * r.d.y, c = ox * ox + oy * oy - p[2] * p[2];
    const double disc = b * b - a * c;
    if (disc < 0) continue;
    const double tc = (-b - std::sqrt(disc)) / a;
    if (tc > 1e-9 && r.o.z + tc * r.d.z <= 6.0) t = std::min(t, tc);
  }
  {  // enclosing cylinder r = 60 (every ray returns)
    const double a = r.d.x * r.d.x + r.d.y * r.d.y;
    const double b = r.o.x * r.d.x + r.o.y * r.d.y, c = r.o.x * r.o.x + r.o.y * r.o.y - 3600.0;
    const double tc = (-b + std::sqrt(b * b - a * c)) / a;
    t = std::min(t, tc);
  }
  return t;
}

void render_lidar(const double Rws[9], const double tws[3], Rng& rng, double* out) {
  std::normal_distribution<double> g(0.0, 1.0);
  constexpr double kDeg = 0.017453292519943295;
  std::size_t k = 0;
  for (int a = 0; a < 2250; ++a) {
    const double az = a * 0.16 * kDeg;
    for (int b = 0; b < 32; ++b) {
      const double el = (-30.67 + 1.3333 * b) * kDeg;
      const V3 ds{std::cos(el) * std::cos(az), std::cos(el) * std::sin(az), std::sin(el)};
      const V3 dw{Rws[0] * ds.x + Rws[1] * ds.y + Rws[2] * ds.z,
                  Rws[3] * ds.x + Rws[4] * ds.y + Rws[5] * ds.z,
                  Rws[6] * ds.x + Rws[7] * ds.y + Rws[8] * ds.z};
      const Ray r{{tws[0], tws[1], tws[2]}, dw};
      const double range = cast_street(r) + 0.02 * g(rng);
      out[k++] = ds.x * range;
      out[k++] = ds.y * range;
      out[k++] = ds.z * range;
    }
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

int trg_synth_kinect_pair_ex(uint64_t seed, double noise_scale, double rot_deg, double trans,
                             double* target, double* source, double R_gt[9], double t_gt[3]) {
  double R1[9], t1[3];
  look_at({3.4, 1.5, 2.6}, {1.2, 0.7, 0.9}, R1, t1);
  double dR[9], dt[3];
  rigid(rot_deg, trans, seed, 0, dR, dt);
  double R2[9], t2[3];  // camera 2 = camera 1 moved by (dR, dt) in its own frame
  matmul(R1, dR, R2);
  for (int i = 0; i < 3; ++i)
    t2[i] = t1[i] + R1[3 * i] * dt[0] + R1[3 * i + 1] * dt[1] + R1[3 * i + 2] * dt[2];
  Rng rng(splitmix64(seed + 0x4b696e656374ull));
  render_kinect(R1, t1, rng, target, noise_scale);
  render_kinect(R2, t2, rng, source, noise_scale);
  relative(R1, t1, R2, t2, R_gt, t_gt);
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
  constexpr double kDeg = 0.017453292519943295;
  double R1[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
  const double t1[3] = {0.0, 0.0, 1.8};
  // ego motion: 1 m forward + 2 deg yaw, then a small random perturbation
  const double c = std::cos(2.0 * kDeg), s = std::sin(2.0 * kDeg);
  const double Rego[9] = {c, -s, 0, s, c, 0, 0, 0, 1};
  double dR[9], dt[3];
  rigid(1.0, 0.05, seed, 0, dR, dt);
  double R2[9], t2[3];
  matmul(Rego, dR, R2);
  t2[0] = 1.0 + dt[0];
  t2[1] = dt[1];
  t2[2] = 1.8 + dt[2];
  Rng rng(splitmix64(seed + 0x4c69444152ull));
  render_lidar(R1, t1, rng, target);
  render_lidar(R2, t2, rng, source);
  relative(R1, t1, R2, t2, R_gt, t_gt);
  return TRG_OK;
}

}  // extern "C"
