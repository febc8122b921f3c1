// Ray casting of the Kinect / LiDAR frame-pair scenes (SURVEY.md 8d configs
// C2 / C3), shared by the host generators (trg_synth.cpp, g++ with
// -ffp-contract=off) and the device renderer (trg_render.cu, nvcc with
// -fmad=false): one source, IEEE operations in the same order on both sides,
// so a frame rendered on the GPU is bit-identical to the host frame given
// the same poses and noise draws.  (The transcendental parts -- the pose
// trigonometry, the LiDAR beam directions, the normal draws -- stay on the
// host: libm and libdevice round them differently.)
#pragma once
#include <cmath>

#ifdef __CUDACC__
#define RC_HD __host__ __device__ __forceinline__
#define RC_SQRT(x) sqrt(x)
#define RC_FABS(x) fabs(x)
#define RC_ISFINITE(x) isfinite(x)
#else
#define RC_HD inline
#define RC_SQRT(x) std::sqrt(x)
#define RC_FABS(x) std::fabs(x)
#define RC_ISFINITE(x) std::isfinite(x)
#endif

namespace trg_rc {

struct V3 {
  double x, y, z;
};
RC_HD V3 add(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
RC_HD V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
RC_HD V3 mul(double s, V3 a) { return {s * a.x, s * a.y, s * a.z}; }
RC_HD double dot(V3 a, V3 b) {
  double s = a.x * b.x;
  s += a.y * b.y;
  s += a.z * b.z;
  return s;
}
// std::min / std::max semantics (first argument on ties)
RC_HD double rmin(double a, double b) { return (b < a) ? b : a; }
RC_HD double rmax(double a, double b) { return (a < b) ? b : a; }

struct Ray {
  V3 o, d;
};
constexpr double kInf = __builtin_huge_val();

// Axis-aligned box, hit from outside.
RC_HD double hit_box_outside(const Ray& r, V3 lo, V3 hi) {
  double t0 = 0.0, t1 = kInf;
  const double o[3] = {r.o.x, r.o.y, r.o.z}, d[3] = {r.d.x, r.d.y, r.d.z};
  const double l[3] = {lo.x, lo.y, lo.z}, h[3] = {hi.x, hi.y, hi.z};
  for (int k = 0; k < 3; ++k) {
    if (RC_FABS(d[k]) < 1e-15) {
      if (o[k] < l[k] || o[k] > h[k]) return kInf;
      continue;
    }
    double a = (l[k] - o[k]) / d[k], b = (h[k] - o[k]) / d[k];
    if (a > b) {
      const double s = a;
      a = b;
      b = s;
    }
    t0 = rmax(t0, a);
    t1 = rmin(t1, b);
    if (t0 > t1) return kInf;
  }
  return t0 > 1e-9 ? t0 : kInf;
}

// Axis-aligned box, the ray starts inside (the room).
RC_HD double hit_box_inside(const Ray& r, V3 lo, V3 hi) {
  double t = kInf;
  const double o[3] = {r.o.x, r.o.y, r.o.z}, d[3] = {r.d.x, r.d.y, r.d.z};
  const double l[3] = {lo.x, lo.y, lo.z}, h[3] = {hi.x, hi.y, hi.z};
  for (int k = 0; k < 3; ++k) {
    if (d[k] > 0) t = rmin(t, (h[k] - o[k]) / d[k]);
    if (d[k] < 0) t = rmin(t, (l[k] - o[k]) / d[k]);
  }
  return t;
}

RC_HD double hit_sphere(const Ray& r, V3 c, double rad) {
  const V3 oc = sub(r.o, c);
  const double a = dot(r.d, r.d);  // ray directions are not unit length
  const double b = dot(oc, r.d), cc = dot(oc, oc) - rad * rad;
  const double disc = b * b - a * cc;
  if (disc < 0) return kInf;
  const double t = (-b - RC_SQRT(disc)) / a;
  return t > 1e-9 ? t : kInf;
}

// Parallelogram corner + a*eu + b*ev, a,b in [0,1].
RC_HD double hit_panel(const Ray& r, V3 corner, V3 eu, V3 ev) {
  const V3 n{eu.y * ev.z - eu.z * ev.y, eu.z * ev.x - eu.x * ev.z, eu.x * ev.y - eu.y * ev.x};
  const double dn = dot(r.d, n);
  if (RC_FABS(dn) < 1e-15) return kInf;
  const double t = dot(sub(corner, r.o), n) / dn;
  if (!(t > 1e-9)) return kInf;
  const V3 p = sub(add(r.o, mul(t, r.d)), corner);
  const double uu = dot(eu, eu), vv = dot(ev, ev), uv = dot(eu, ev);
  const double pu = dot(p, eu), pv = dot(p, ev);
  const double det = uu * vv - uv * uv;
  const double a = (pu * vv - pv * uv) / det, b = (pv * uu - pu * uv) / det;
  return (a >= 0 && a <= 1 && b >= 0 && b <= 1) ? t : kInf;
}

// Closed room (metres, y up): walls, a box, a ball, a slanted panel.
RC_HD double cast_room(const Ray& r) {
  double t = hit_box_inside(r, {0, 0, 0}, {4, 2.4, 3});
  t = rmin(t, hit_box_outside(r, {2.4, 0.0, 1.8}, {3.2, 0.7, 2.6}));
  t = rmin(t, hit_sphere(r, {1.1, 0.6, 1.0}, 0.44));
  t = rmin(t, hit_panel(r, {1.8, 0.0, 0.2}, {1.0, 0.0, 0.3}, {0.0, 0.8, 0.6}));
  return t;
}

// HDL-32 street: ground z = 0, building boxes, poles, enclosing cylinder.
RC_HD double cast_street(const Ray& r) {
  double t = kInf;
  if (r.d.z < 0) t = -r.o.z / r.d.z;
  const double boxes[8][6] = {
      {8, -20, 0, 20, -9, 9},  {-25, -22, 0, -10, -8, 14}, {-6, 10, 0, 12, 24, 7},
      {25, 6, 0, 40, 18, 11},  {-40, 12, 0, -28, 30, 16},  {-18, -45, 0, 5, -34, 10},
      {30, -30, 0, 44, -16, 8}, {3, -6, 0, 5, -4, 1.2}};
  for (int i = 0; i < 8; ++i) {
    const double* b = boxes[i];
    t = rmin(t, hit_box_outside(r, {b[0], b[1], b[2]}, {b[3], b[4], b[5]}));
  }
  const double poles[6][3] = {{6, 4, 0.15}, {-5, 5, 0.2}, {14, -3, 0.15},
                              {-12, -4, 0.25}, {2, 12, 0.15}, {-3, -14, 0.2}};
  for (int i = 0; i < 6; ++i) {  // vertical cylinders of height 6 m
    const double* p = poles[i];
    const double ox = r.o.x - p[0], oy = r.o.y - p[1];
    const double a = r.d.x * r.d.x + r.d.y * r.d.y;
    if (a < 1e-15) continue;
    const double b = ox * r.d.x + oy * r.d.y, c = ox * ox + oy * oy - p[2] * p[2];
    const double disc = b * b - a * c;
    if (disc < 0) continue;
    const double tc = (-b - RC_SQRT(disc)) / a;
    if (tc > 1e-9 && r.o.z + tc * r.d.z <= 6.0) t = rmin(t, tc);
  }
  {  // enclosing cylinder r = 60 (every ray returns)
    const double a = r.d.x * r.d.x + r.d.y * r.d.y;
    const double b = r.o.x * r.d.x + r.o.y * r.d.y, c = r.o.x * r.o.x + r.o.y * r.o.y - 3600.0;
    const double tc = (-b + RC_SQRT(b * b - a * c)) / a;
    t = rmin(t, tc);
  }
  return t;
}

// Kinect pixel (u, v) of a 320x240 frame from camera pose (Rwc, twc): the
// point in camera coordinates, axial noise sigma_z = 0.0012 + 0.0019 (z -
// 0.4)^2 times noise_scale times the pixel's normal draw g.
RC_HD void kinect_pixel(const double* Rwc, const double* twc, int u, int v, double g,
                        double noise_scale, double out[3]) {
  const double fx = 262.5, fy = 262.5, cx = 159.5, cy = 119.5;
  const V3 dc{(u - cx) / fx, (v - cy) / fy, 1.0};
  const V3 dw{Rwc[0] * dc.x + Rwc[1] * dc.y + Rwc[2] * dc.z,
              Rwc[3] * dc.x + Rwc[4] * dc.y + Rwc[5] * dc.z,
              Rwc[6] * dc.x + Rwc[7] * dc.y + Rwc[8] * dc.z};
  const Ray r{{twc[0], twc[1], twc[2]}, dw};
  const double t = cast_room(r);  // z = t since dc.z == 1
  const double z = RC_ISFINITE(t) ? t : 6.0;
  const double sz = 0.0012 + 0.0019 * (z - 0.4) * (z - 0.4);
  const double zn = z + noise_scale * sz * g;
  out[0] = dc.x * zn;
  out[1] = dc.y * zn;
  out[2] = zn;
}

// LiDAR beam with sensor-frame direction ds from pose (Rws, tws): the point
// in sensor coordinates, range noise 0.02 g.
RC_HD void lidar_beam(const double* Rws, const double* tws, V3 ds, double g, double out[3]) {
  const V3 dw{Rws[0] * ds.x + Rws[1] * ds.y + Rws[2] * ds.z,
              Rws[3] * ds.x + Rws[4] * ds.y + Rws[5] * ds.z,
              Rws[6] * ds.x + Rws[7] * ds.y + Rws[8] * ds.z};
  const Ray r{{tws[0], tws[1], tws[2]}, dw};
  const double range = cast_street(r) + 0.02 * g;
  out[0] = ds.x * range;
  out[1] = ds.y * range;
  out[2] = ds.z * range;
}

}  // namespace trg_rc
