// host_scene.cpp — host-side workload and camera plumbing of the C-ABI.
//
//   psm_default_config      RasterConfig defaults (proj/include/psimap/raster.hpp:42-54)
//   psm_camera_make         Camera::make        (proj/src/core_types.cpp:18-38)
//   psm_camera_look_at      Camera::look_at     (proj/src/core_types.cpp:40-60)
//   psm_make_street_scene   make_street_scene   (proj/src/synthetic.cpp:236-312) with
//                           quat_from_axes (synthetic.cpp:21-27), quat_from_rotation
//                           (math_util.cpp:73-92) and Rng (math_util.hpp:27-63)
//
// The generator keeps the reference's RNG draw order. Where the reference's
// order is compiler-defined (C++ leaves the evaluation order of operands of `+`
// and of constructor arguments unspecified) we follow GCC 13, the toolchain of
// this image, which evaluates them right to left: the centre draws the normal
// jitter, then the e2 coefficient, then the e1 coefficient
// (synthetic.cpp:278-279), and Vec3(u, u, u) draws blue, green, red
// (synthetic.cpp:289). The only addition is `scale_mult` (applied to s1 right
// after it is drawn; SURVEY.md §8d density normalisation).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "../../include/psm.h"

namespace {

struct V3 {
  double x, y, z;
};
inline V3 add(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V3 scale(double s, V3 a) { return {s * a.x, s * a.y, s * a.z}; }
inline double sqnorm(V3 a) { return (a.x * a.x + a.y * a.y) + a.z * a.z; }
inline double norm(V3 a) { return std::sqrt(sqnorm(a)); }
inline V3 normalized(V3 a) {  // Eigen MatrixBase::normalized: n / sqrt(squaredNorm) if > 0
  const double z = sqnorm(a);
  if (z > 0) {
    const double s = std::sqrt(z);
    return {a.x / s, a.y / s, a.z / s};
  }
  return a;
}
inline V3 cross(V3 a, V3 b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}

struct Rng {  // math_util.hpp:27-63
  uint64_t state;
  explicit Rng(uint64_t seed) : state(seed) {}
  uint64_t next() {
    uint64_t z = (state += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  double normal() {
    double u1 = uniform();
    double u2 = uniform();
    if (u1 < 1e-300) u1 = 1e-300;
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
  }
};

// quat_from_rotation (math_util.cpp:73-92); r is row-indexed r[row][col]
void quat_from_rotation(const double r[3][3], double q[4]) {
  const double tr = (r[0][0] + r[1][1]) + r[2][2];
  if (tr > 0) {
    const double s = std::sqrt(tr + 1.0) * 2;
    q[0] = 0.25 * s; q[1] = (r[2][1] - r[1][2]) / s; q[2] = (r[0][2] - r[2][0]) / s; q[3] = (r[1][0] - r[0][1]) / s;
  } else if (r[0][0] > r[1][1] && r[0][0] > r[2][2]) {
    const double s = std::sqrt(1.0 + r[0][0] - r[1][1] - r[2][2]) * 2;
    q[0] = (r[2][1] - r[1][2]) / s; q[1] = 0.25 * s; q[2] = (r[0][1] + r[1][0]) / s; q[3] = (r[0][2] + r[2][0]) / s;
  } else if (r[1][1] > r[2][2]) {
    const double s = std::sqrt(1.0 + r[1][1] - r[0][0] - r[2][2]) * 2;
    q[0] = (r[0][2] - r[2][0]) / s; q[1] = (r[0][1] + r[1][0]) / s; q[2] = 0.25 * s; q[3] = (r[1][2] + r[2][1]) / s;
  } else {
    const double s = std::sqrt(1.0 + r[2][2] - r[0][0] - r[1][1]) * 2;
    q[0] = (r[1][0] - r[0][1]) / s; q[1] = (r[0][2] + r[2][0]) / s; q[2] = (r[1][2] + r[2][1]) / s; q[3] = 0.25 * s;
  }
  if (q[0] < 0) for (int i = 0; i < 4; ++i) q[i] = -q[i];
  const double n = std::sqrt((q[0] * q[0] + q[2] * q[2]) + (q[1] * q[1] + q[3] * q[3]));
  for (int i = 0; i < 4; ++i) q[i] = q[i] / n;
}

// quat_from_axes (synthetic.cpp:21-27)
void quat_from_axes(V3 t_u, V3 t_v, double q[4]) {
  const V3 c0 = normalized(t_u);
  const V3 c2 = normalized(cross(t_u, t_v));
  const V3 c1 = cross(c2, c0);
  const double r[3][3] = {{c0.x, c1.x, c2.x}, {c0.y, c1.y, c2.y}, {c0.z, c1.z, c2.z}};
  quat_from_rotation(r, q);
}

bool finite_all(const double* v, int n) {
  for (int i = 0; i < n; ++i)
    if (!std::isfinite(v[i])) return false;
  return true;
}

}  // namespace

extern "C" {

void psm_default_config(psm_raster_config* cfg) {
  std::memset(cfg, 0, sizeof *cfg);
  cfg->tile_size = 16;
  cfg->chi2 = 9.0;
  cfg->alpha_min = 1.0 / 255.0;
  cfg->t_min = 1e-4;
  cfg->support_cutoff = 1;
  cfg->binning = PSM_BIN_AABB;
  cfg->blending = PSM_BLEND_FULL;
  cfg->top_k = 16;
  cfg->render_depth_normal = 1;
  cfg->threads = 0;
}

int psm_camera_make(const double r_cw[9], const double t_cw[3], double fx, double fy, double cx, double cy,
                    int32_t width, int32_t height, double near_clip, double far_clip, psm_camera* out) {
  if (!out || !r_cw || !t_cw) return PSM_EINVAL;
  if (!(fx > 0) || !(fy > 0)) return PSM_EINVAL;
  if (width <= 0 || height <= 0) return PSM_EINVAL;
  if (!(near_clip > 0) || !(near_clip < far_clip)) return PSM_EINVAL;
  if (!finite_all(r_cw, 9) || !finite_all(t_cw, 3)) return PSM_EINVAL;
  std::memcpy(out->r_cw, r_cw, sizeof out->r_cw);
  std::memcpy(out->t_cw, t_cw, sizeof out->t_cw);
  out->fx = fx; out->fy = fy; out->cx = cx; out->cy = cy;
  out->width = width; out->height = height;
  out->near_clip = near_clip; out->far_clip = far_clip;
  return PSM_OK;
}

int psm_camera_look_at(const double eye_[3], const double target_[3], const double up_[3], double fx, double fy,
                       int32_t width, int32_t height, double near_clip, double far_clip, psm_camera* out) {
  const V3 eye{eye_[0], eye_[1], eye_[2]}, target{target_[0], target_[1], target_[2]}, up{up_[0], up_[1], up_[2]};
  V3 fwd = sub(target, eye);
  if (norm(fwd) < 1e-12) return PSM_EINVAL;
  fwd = normalized(fwd);
  V3 right = cross(fwd, up);
  if (norm(right) < 1e-9) {
    right = cross(fwd, V3{1, 0, 0});
    if (norm(right) < 1e-9) right = cross(fwd, V3{0, 1, 0});
  }
  right = normalized(right);
  const V3 down = cross(fwd, right);
  // r_wc columns (right, down, fwd); r_cw = r_wc^T, stored column-major
  double r_cw[9];
  const V3 rows[3] = {right, down, fwd};
  for (int row = 0; row < 3; ++row) {
    r_cw[0 * 3 + row] = rows[row].x;
    r_cw[1 * 3 + row] = rows[row].y;
    r_cw[2 * 3 + row] = rows[row].z;
  }
  // t = -r_cw * eye  ((-R) * eye, 3-term sums left to right)
  double t[3];
  for (int row = 0; row < 3; ++row) {
    t[row] = ((-r_cw[0 * 3 + row]) * eye.x + (-r_cw[1 * 3 + row]) * eye.y) + (-r_cw[2 * 3 + row]) * eye.z;
  }
  return psm_camera_make(r_cw, t, fx, fy, 0.5 * width, 0.5 * height, width, height, near_clip, far_clip, out);
}

static int street_scene(const psm_street_spec* spec, int64_t* n_out, double* surfels13, double* f_sem,
                        double* labels, double* f_ins, psm_camera* cam) {
  if (!spec || !n_out) return PSM_EINVAL;
  if (spec->n_surfels < 0 || spec->c_sem < 0 || spec->n_instances < 1) return PSM_EINVAL;
  struct Group {
    V3 origin, e1, e2;
    int instance;
    double share;
  };
  std::vector<Group> groups;
  groups.push_back({{-4, 1.5, 1.5}, {8, 0, 0}, {0, 0, 38}, 0, 0.10});
  groups.push_back({{-4.0, 1.5, 1.5}, {0.9, -4.0, 0}, {0, 0, 38}, 1, 0.06});
  groups.push_back({{4.0, 1.5, 1.5}, {-0.9, -4.0, 0}, {0, 0, 38}, 2, 0.06});
  const int n_layers = 18;
  const int n_inst = spec->n_instances;
  const int bands = std::max(1, (n_inst - 3) / n_layers + 1);
  for (int l = 0; l < n_layers; ++l) {
    const double z = 3.2 + 2.0 * l;
    const double band_w = 7.2 / bands;
    for (int b = 0; b < bands; ++b) {
      groups.push_back({{-3.6 + b * band_w, -2.6, z}, {band_w, 0, 0}, {0, 5.2, 0},
                        3 + (b % std::max(1, n_inst - 3)), 0.78 / (n_layers * bands)});
    }
  }
  int64_t total = 0;
  for (const Group& g : groups) total += static_cast<int64_t>(std::round(g.share * spec->n_surfels));
  *n_out = total;
  if (cam) {
    const double eye[3] = {0, 0, 0}, target[3] = {0, 0, 20}, up[3] = {0, -1, 0};
    const int st = psm_camera_look_at(eye, target, up, 0.8 * spec->image_w, 0.8 * spec->image_w, spec->image_w,
                                      spec->image_h, 0.1, 200.0, cam);
    if (st != PSM_OK) return st;
  }
  if (!surfels13) return PSM_OK;  // size query

  Rng rng(spec->seed);
  const int c_ins = 8;
  const double smult = spec->scale_mult > 0 ? spec->scale_mult : 1.0;
  int64_t at = 0;
  for (const Group& g : groups) {
    const int n = static_cast<int>(std::round(g.share * spec->n_surfels));
    const V3 u1 = normalized(g.e1);
    const V3 u2 = normalized(g.e2);
    const V3 g_normal = normalized(cross(u1, u2));
    for (int i = 0; i < n; ++i, ++at) {
      double* s = surfels13 + 13 * at;
      // centre: GCC evaluates the three draws right to left (see header)
      const double dj = rng.uniform(-0.03, 0.03);
      const double db = rng.uniform();
      const double da = rng.uniform();
      const V3 c = add(add(add(g.origin, scale(da, g.e1)), scale(db, g.e2)), scale(dj, g_normal));
      s[0] = c.x; s[1] = c.y; s[2] = c.z;
      const double phi = rng.uniform(0, M_PI);
      const double cphi = std::cos(phi), sphi = std::sin(phi);
      const V3 t_u = add(scale(cphi, u1), scale(sphi, u2));
      const V3 t_v_raw = add(scale(-sphi, u1), scale(cphi, u2));
      quat_from_axes(t_u, t_v_raw, s + 3);
      double s1 = rng.uniform(0.45, 1.1);
      s1 = s1 * smult;
      const double aspect = rng.uniform(spec->min_aspect, 2.0 * spec->min_aspect);
      s[7] = s1;
      s[8] = s1 / aspect;
      s[9] = rng.uniform(0.30, 0.70);
      const double cb = rng.uniform(0.2, 0.9);  // Vec3(u, u, u): right to left
      const double cg = rng.uniform(0.2, 0.9);
      const double cr = rng.uniform(0.2, 0.9);
      s[10] = cr; s[11] = cg; s[12] = cb;
      for (int c = 0; c < spec->c_sem; ++c) {
        const double v = rng.normal();
        if (f_sem) f_sem[at * spec->c_sem + c] = v;
      }
      for (int c = 0; c < c_ins; ++c) {  // f_ins: unused by render (drawn for the RNG order); assign_labels
        const double v = 0.3 * rng.normal();
        if (f_ins) f_ins[at * c_ins + c] = v;
      }
    }
  }
  if (labels) {  // near one-hot per structural instance (synthetic.cpp:298-309)
    int64_t a = 0;
    for (const Group& g : groups) {
      const int n = static_cast<int>(std::round(g.share * spec->n_surfels));
      for (int i = 0; i < n; ++i, ++a) {
        double* col = labels + a * n_inst;
        for (int q = 0; q < n_inst; ++q) col[q] = q == g.instance ? 0.92 : 0.08 / (n_inst - 1);
      }
    }
  }
  return PSM_OK;
}

int psm_make_street_scene(const psm_street_spec* spec, int64_t* n_out, double* surfels13, double* f_sem,
                          double* labels, psm_camera* cam) {
  return street_scene(spec, n_out, surfels13, f_sem, labels, nullptr, cam);
}

int psm_make_street_scene_ins(const psm_street_spec* spec, int64_t* n_out, double* f_ins) {
  int64_t n = 0;
  int st = street_scene(spec, &n, nullptr, nullptr, nullptr, nullptr, nullptr);
  if (st != PSM_OK) return st;
  if (n_out) *n_out = n;
  if (!f_ins) return PSM_OK;
  std::vector<double> tmp(static_cast<size_t>(n > 0 ? n : 1) * 13);
  return street_scene(spec, &n, tmp.data(), nullptr, nullptr, f_ins, nullptr);
}

}  // extern "C"
