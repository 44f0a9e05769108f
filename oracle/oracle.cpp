// oracle.cpp — CPU restatement of the reference render path. TEST INFRASTRUCTURE ONLY.
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference legs may load this library, and only as the checker or the timed
// CPU baseline. The product (paper_2604_10982_b200/) never links or calls it.
//
// What it restates (all paths under /root/reference/proj):
//   src/raster.cpp:17-49     footprint_cov, max_eigenvalue2, circle_box, aabb_box
//   src/raster.cpp:51-90     bin_boxes (bin_circle / bin_aabb, raster.cpp:144-152)
//   src/raster.cpp:94-142    project_surfel
//   src/raster.cpp:154-177   sample_surfel_alpha, evaluate_alpha
//   src/raster.cpp:225-251   topk_select
//   src/raster.cpp:273-511   render_into (hot-SoA build 321-353, tile loop 355-504)
//   src/raster.cpp:513-573   bench_render
//   src/math_util.cpp:16-23,46-52   rotation_unit, rotation_from_quat
//   src/math_util.cpp:135-162       worker_count, parallel_chunks
//   include/psimap/core_types.hpp:51-52  Camera::to_camera, center_world
//   src/panoptic.cpp:36-91   assign_labels (math in psm_panoptic.h, shared with the GPU)
//   src/metrics.cpp:339-369  render_panoptic epilogue (oracle/pyoracle.py, over render's fp64 planes)
//   src/pipeline.cpp:347-460 blending backward, raster.cpp:179-203 project_surfel_backward
//                            (oracle_render_backward; geometry chain in psm_backward.h)
//
// Why a restatement: the reference needs Eigen3, which is not in this image
// (proj/CMakeLists.txt:13-15 `find_path(EIGEN3_INCLUDE_DIR ... REQUIRED)`), so
// it cannot be compiled here. Eigen's fixed-size
// evaluation order is restated explicitly below (3-term sums left to right,
// Vector4d::norm as (q0^2+q2^2)+(q1^2+q3^2) from SSE2 packet reduction,
// Matrix3d::determinant and ::inverse by cofactors). PARITY PIN: this oracle is
// pinned to the reference through every known-answer test the reference's
// own suites hold for this path (proj/tests/test_raster.cpp, acceptance
// criteria 1-3), ported in tests/test_oracle_kat.py; those pins are
// tolerance-level (1e-8..1e-12), so bit-level agreement with an Eigen build of
// the reference is unpinned. glibc `exp` is replaced by psm_exp (see
// paper_2604_10982_b200/csrc/psm_exp.h); building with -DORACLE_LIBM_EXP
// restores std::exp, and tests/test_oracle_kat.py measures the divergence.
//
// Build: oracle/Makefile (-O3 -ffp-contract=off -mfma; no fast-math).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <numeric>
#include <thread>
#include <vector>
#include <chrono>

#include "../include/psm.h"
#include "../paper_2604_10982_b200/csrc/psm_ellipse.h"
#include "../paper_2604_10982_b200/csrc/psm_exp.h"
#include "../paper_2604_10982_b200/csrc/psm_panoptic.h"
#include "../paper_2604_10982_b200/csrc/psm_backward.h"

namespace {

#ifdef ORACLE_LIBM_EXP
inline double oexp(double x) { return std::exp(x); }
#else
inline double oexp(double x) { return psm_exp(x); }
#endif

// ---------------------------------------------------------------- tiny linear algebra
// Column-major like Eigen: m[c*N + r].
struct V2 { double v[2]; };
struct V3 { double v[3]; };
struct M2 { double m[4]; double& at(int r, int c) { return m[c * 2 + r]; } double at(int r, int c) const { return m[c * 2 + r]; } };
struct M3 { double m[9]; double& at(int r, int c) { return m[c * 3 + r]; } double at(int r, int c) const { return m[c * 3 + r]; } };

// Eigen 3-term reductions: evaluated left to right, (x0 + x1) + x2.
inline double sum3(double a, double b, double c) { return (a + b) + c; }
inline V3 matvec(const M3& a, const V3& x) {
  V3 r;
  for (int i = 0; i < 3; ++i) r.v[i] = sum3(a.at(i, 0) * x.v[0], a.at(i, 1) * x.v[1], a.at(i, 2) * x.v[2]);
  return r;
}
inline V3 matTvec(const M3& a, const V3& x) {  // a^T x
  V3 r;
  for (int i = 0; i < 3; ++i) r.v[i] = sum3(a.at(0, i) * x.v[0], a.at(1, i) * x.v[1], a.at(2, i) * x.v[2]);
  return r;
}
inline double dot3(const V3& a, const V3& b) { return sum3(a.v[0] * b.v[0], a.v[1] * b.v[1], a.v[2] * b.v[2]); }
inline double norm3(const V3& a) { return std::sqrt(dot3(a, a)); }

// Matrix3d::determinant (Eigen Determinant.h, bruteforce_det3_helper)
inline double det3_helper(const M3& m, int a, int b, int c) {
  return m.at(0, a) * (m.at(1, b) * m.at(2, c) - m.at(1, c) * m.at(2, b));
}
inline double det3(const M3& m) {
  return det3_helper(m, 0, 1, 2) - det3_helper(m, 1, 0, 2) + det3_helper(m, 2, 0, 1);
}
// Matrix3d::inverse (Eigen InverseImpl.h, cofactor_3x3 + compute_inverse_size3_helper)
inline double cof3(const M3& m, int i, int j) {
  const int i1 = (i + 1) % 3, i2 = (i + 2) % 3, j1 = (j + 1) % 3, j2 = (j + 2) % 3;
  return m.at(i1, j1) * m.at(i2, j2) - m.at(i1, j2) * m.at(i2, j1);
}
inline M3 inverse3(const M3& m) {
  const double c00 = cof3(m, 0, 0), c10 = cof3(m, 1, 0), c20 = cof3(m, 2, 0);
  const double det = sum3(c00 * m.at(0, 0), c10 * m.at(1, 0), c20 * m.at(2, 0));
  const double invdet = 1.0 / det;
  M3 r;
  r.at(0, 1) = c10 * invdet;  // row 0 = cofactor column 0 * invdet
  r.at(0, 0) = c00 * invdet;
  r.at(0, 2) = c20 * invdet;
  r.at(1, 0) = cof3(m, 0, 1) * invdet;
  r.at(1, 1) = cof3(m, 1, 1) * invdet;
  r.at(2, 0) = cof3(m, 0, 2) * invdet;
  r.at(1, 2) = cof3(m, 2, 1) * invdet;
  r.at(2, 1) = cof3(m, 1, 2) * invdet;
  r.at(2, 2) = cof3(m, 2, 2) * invdet;
  return r;
}

// ---------------------------------------------------------------- L0 (math_util.cpp)
// rotation_unit, math_util.cpp:16-23
M3 rotation_unit(double w, double x, double y, double z) {
  M3 r;
  r.at(0, 0) = 1 - 2 * (y * y + z * z); r.at(0, 1) = 2 * (x * y - w * z); r.at(0, 2) = 2 * (x * z + w * y);
  r.at(1, 0) = 2 * (x * y + w * z); r.at(1, 1) = 1 - 2 * (x * x + z * z); r.at(1, 2) = 2 * (y * z - w * x);
  r.at(2, 0) = 2 * (x * z - w * y); r.at(2, 1) = 2 * (y * z + w * x); r.at(2, 2) = 1 - 2 * (x * x + y * y);
  return r;
}
// rotation_from_quat, math_util.cpp:46-52. Returns false where the reference throws.
bool rotation_from_quat(const double q[4], M3& out) {
  const double norm = std::sqrt((q[0] * q[0] + q[2] * q[2]) + (q[1] * q[1] + q[3] * q[3]));
  const bool finite = std::isfinite(q[0]) && std::isfinite(q[1]) && std::isfinite(q[2]) && std::isfinite(q[3]);
  if (!(norm > 1e-12) || !finite) return false;
  out = rotation_unit(q[0] / norm, q[1] / norm, q[2] / norm, q[3] / norm);
  return true;
}

int worker_count() {  // math_util.cpp:135-142
  if (const char* env = std::getenv("PSIMAP_THREADS")) {
    const int n = std::atoi(env);
    if (n > 0) return n;
  }
  const unsigned hw = std::thread::hardware_concurrency();
  return hw == 0 ? 1 : static_cast<int>(hw);
}

void parallel_chunks(int64_t n, int threads, const std::function<void(int64_t, int64_t)>& fn) {  // :144-162
  if (threads <= 0) threads = worker_count();
  if (n <= 0) return;
  const int used = static_cast<int>(std::min<int64_t>(threads, n));
  if (used <= 1) { fn(0, n); return; }
  std::vector<std::thread> pool;
  pool.reserve(used);
  const int64_t chunk = (n + used - 1) / used;
  for (int t = 0; t < used; ++t) {
    const int64_t begin = t * chunk;
    const int64_t end = std::min<int64_t>(begin + chunk, n);
    if (begin >= end) break;
    pool.emplace_back([&fn, begin, end] { fn(begin, end); });
  }
  for (auto& th : pool) th.join();
}

// ---------------------------------------------------------------- L1 raster
struct Projected {  // ProjectedSurfel, raster.hpp:21-30
  int source = -1;
  double center[2];
  M2 sigma;
  double sort_depth;
  M3 h, h_inv;
  M2 finv;
  double normal_vis[3];
};

struct Cam {
  M3 r;
  V3 t;
  double fx, fy, cx, cy;
  int w, h;
  double near_clip, far_clip;
};
Cam cam_from(const psm_camera* c) {
  Cam o;
  std::memcpy(o.r.m, c->r_cw, sizeof o.r.m);
  for (int i = 0; i < 3; ++i) o.t.v[i] = c->t_cw[i];
  o.fx = c->fx; o.fy = c->fy; o.cx = c->cx; o.cy = c->cy;
  o.w = c->width; o.h = c->height;
  o.near_clip = c->near_clip; o.far_clip = c->far_clip;
  return o;
}

constexpr double kFootprintDilation = 0.3;  // raster.cpp:17
M2 footprint_cov(const M2& s) {             // raster.cpp:19-24
  M2 f = s;
  f.at(0, 0) += kFootprintDilation;
  f.at(1, 1) += kFootprintDilation;
  return f;
}
double max_eigenvalue2(const M2& m) {       // raster.cpp:26-31
  const double half_tr = 0.5 * (m.at(0, 0) + m.at(1, 1));
  const double det = m.at(0, 0) * m.at(1, 1) - m.at(0, 1) * m.at(1, 0);
  const double disc = std::sqrt(std::max(half_tr * half_tr - det, 0.0));
  return half_tr + disc;
}
struct Box { double x0, x1, y0, y1; };
Box circle_box(const Projected& p, double chi2) {  // raster.cpp:37-41
  const double r = std::sqrt(chi2 * max_eigenvalue2(footprint_cov(p.sigma)));
  return {p.center[0] - r, p.center[0] + r, p.center[1] - r, p.center[1] + r};
}
Box aabb_box(const Projected& p, double chi2) {    // raster.cpp:43-49
  const M2 f = footprint_cov(p.sigma);
  const double dx = std::sqrt(chi2 * f.at(0, 0));
  const double dy = std::sqrt(chi2 * f.at(1, 1));
  return {p.center[0] - dx, p.center[0] + dx, p.center[1] - dy, p.center[1] + dy};
}

// project_surfel, raster.cpp:94-142. Returns 1 = projected, 0 = culled, -1 = degenerate quaternion.
int project_surfel(const double* s13, const Cam& cam, double chi2, Projected& out) {
  const V3 mu{{s13[0], s13[1], s13[2]}};
  const V3 pr = matvec(cam.r, mu);
  const V3 p_cam{{pr.v[0] + cam.t.v[0], pr.v[1] + cam.t.v[1], pr.v[2] + cam.t.v[2]}};  // to_camera
  if (!(p_cam.v[2] > cam.near_clip) || !(p_cam.v[2] < cam.far_clip)) return 0;

  M3 r_s;
  if (!rotation_from_quat(s13 + 3, r_s)) return -1;
  const V3 sa{{s13[7] * r_s.at(0, 0), s13[7] * r_s.at(1, 0), s13[7] * r_s.at(2, 0)}};
  const V3 sb{{s13[8] * r_s.at(0, 1), s13[8] * r_s.at(1, 1), s13[8] * r_s.at(2, 1)}};
  const V3 a = matvec(cam.r, sa);
  const V3 b = matvec(cam.r, sb);

  for (int i = 0; i < 3; ++i) {
    out.h.at(i, 0) = a.v[i];
    out.h.at(i, 1) = b.v[i];
    out.h.at(i, 2) = p_cam.v[i];
  }
  const double det = det3(out.h);
  const double det_scale = norm3(a) * norm3(b) * norm3(p_cam);
  if (std::abs(det) <= 1e-12 * std::max(det_scale, 1e-30)) return 0;  // grazing
  out.h_inv = inverse3(out.h);

  const double z = p_cam.v[2];
  out.sort_depth = z;
  out.center[0] = cam.fx * p_cam.v[0] / z + cam.cx;
  out.center[1] = cam.fy * p_cam.v[1] / z + cam.cy;

  // jac (2x3) and bb = [jac*a, jac*b]; sigma = bb bb^T  (raster.cpp:119-125)
  const double j00 = cam.fx / z, j01 = 0, j02 = -cam.fx * p_cam.v[0] / (z * z);
  const double j10 = 0, j11 = cam.fy / z, j12 = -cam.fy * p_cam.v[1] / (z * z);
  const double bb00 = sum3(j00 * a.v[0], j01 * a.v[1], j02 * a.v[2]);
  const double bb10 = sum3(j10 * a.v[0], j11 * a.v[1], j12 * a.v[2]);
  const double bb01 = sum3(j00 * b.v[0], j01 * b.v[1], j02 * b.v[2]);
  const double bb11 = sum3(j10 * b.v[0], j11 * b.v[1], j12 * b.v[2]);
  out.sigma.at(0, 0) = bb00 * bb00 + bb01 * bb01;
  out.sigma.at(0, 1) = bb00 * bb10 + bb01 * bb11;
  out.sigma.at(1, 0) = bb10 * bb00 + bb11 * bb01;
  out.sigma.at(1, 1) = bb10 * bb10 + bb11 * bb11;

  const Box bounds = circle_box(out, chi2);
  if (bounds.x1 < 0 || bounds.x0 > cam.w || bounds.y1 < 0 || bounds.y0 > cam.h) return 0;

  const M2 f = footprint_cov(out.sigma);
  const double fdet = f.at(0, 0) * f.at(1, 1) - f.at(0, 1) * f.at(1, 0);
  out.finv.at(0, 0) = f.at(1, 1) / fdet;
  out.finv.at(1, 0) = -f.at(1, 0) / fdet;  // comma-init is row-major: (f11, -f01; -f10, f00)
  out.finv.at(0, 1) = -f.at(0, 1) / fdet;
  out.finv.at(1, 1) = f.at(0, 0) / fdet;

  const V3 n_world{{r_s.at(0, 2), r_s.at(1, 2), r_s.at(2, 2)}};
  const V3 rt = matTvec(cam.r, cam.t);
  const V3 cw{{-rt.v[0], -rt.v[1], -rt.v[2]}};  // center_world = -R^T t
  const V3 d{{cw.v[0] - mu.v[0], cw.v[1] - mu.v[1], cw.v[2] - mu.v[2]}};
  const bool front = dot3(d, n_world) >= 0;
  for (int i = 0; i < 3; ++i) out.normal_vis[i] = front ? n_world.v[i] : -n_world.v[i];
  out.source = -1;
  return 1;
}

struct Grid {
  int tiles_x = 0, tiles_y = 0;
  std::vector<std::vector<int>> tiles;  // projected indices, ascending (depth, source)
  uint64_t rn_total = 0;
  double rn_per_tile = 0;
  int64_t nonempty = 0;
};

// bin_boxes, raster.cpp:51-90, with binning 0 circle / 1 aabb / 2 ellipse (extension)
Grid bin(const std::vector<Projected>& projected, const Cam& cam, int ts, double chi2, int binning) {
  Grid g;
  g.tiles_x = (cam.w + ts - 1) / ts;
  g.tiles_y = (cam.h + ts - 1) / ts;
  g.tiles.assign(static_cast<size_t>(g.tiles_x) * g.tiles_y, {});
  const double tsd = ts;
  for (size_t i = 0; i < projected.size(); ++i) {
    const Projected& p = projected[i];
    const Box b = binning == 0 ? circle_box(p, chi2) : aabb_box(p, chi2);
    int tx0 = static_cast<int>(std::floor(b.x0 / tsd));
    int tx1 = static_cast<int>(std::floor(b.x1 / tsd));
    int ty0 = static_cast<int>(std::floor(b.y0 / tsd));
    int ty1 = static_cast<int>(std::floor(b.y1 / tsd));
    tx0 = std::max(tx0, 0);
    ty0 = std::max(ty0, 0);
    tx1 = std::min(tx1, g.tiles_x - 1);
    ty1 = std::min(ty1, g.tiles_y - 1);
    const M2 f = footprint_cov(p.sigma);
    PsmEllipse e{};
    if (binning == 2) e = psm_ellipse_prep(p.center[0], p.center[1], f.at(0, 0), f.at(0, 1), f.at(1, 1), chi2);
    for (int ty = ty0; ty <= ty1; ++ty) {
      int lo = tx0, hi = tx1;
      if (binning == 2 && !psm_ellipse_row(e, ty, ts, cam.h, tx0, tx1, &lo, &hi)) continue;
      for (int tx = lo; tx <= hi; ++tx) g.tiles[static_cast<size_t>(ty) * g.tiles_x + tx].push_back(static_cast<int>(i));
    }
  }
  uint64_t total = 0;
  int64_t nonempty = 0;
  for (auto& tile : g.tiles) {
    std::sort(tile.begin(), tile.end(), [&](int a, int b) {
      if (projected[a].sort_depth != projected[b].sort_depth) return projected[a].sort_depth < projected[b].sort_depth;
      return projected[a].source < projected[b].source;
    });
    total += tile.size();
    if (!tile.empty()) ++nonempty;
  }
  g.rn_total = total;
  g.nonempty = nonempty;
  g.rn_per_tile = nonempty > 0 ? static_cast<double>(total) / nonempty : 0.0;
  return g;
}

struct WeightKey { double weight; int proj; int index; };

// topk_select, raster.cpp:225-251
void topk_select(const WeightKey* keys, int m, int k, std::vector<WeightKey>& best, std::vector<char>& selected) {
  selected.assign(m, 0);
  if (k >= m) {
    for (int i = 0; i < m; ++i) selected[i] = 1;
    return;
  }
  auto before = [](const WeightKey& a, const WeightKey& b) {
    if (a.weight != b.weight) return a.weight > b.weight;
    return a.proj < b.proj;
  };
  best.clear();
  best.reserve(k);
  for (int i = 0; i < m; ++i) {
    const WeightKey& cand = keys[i];
    const int filled = static_cast<int>(best.size());
    if (filled == k && !before(cand, best.back())) continue;
    int pos = filled == k ? k - 1 : filled;
    if (filled < k) best.push_back(cand);
    while (pos > 0 && before(cand, best[pos - 1])) {
      best[pos] = best[pos - 1];
      --pos;
    }
    best[pos] = cand;
  }
  for (const WeightKey& wk : best) selected[wk.index] = 1;
}

struct Scratch {
  struct Entry { int proj; double alpha, u, v, weight, depth; };
  std::vector<Entry> entries, selected_entries;
  std::vector<WeightKey> keys, best;
  std::vector<char> selected;
  std::vector<double> accum;
};

struct Outputs {
  double *color, *depth, *normal, *sem_feat, *ins_dist, *alpha_acc;
  int32_t *ins_argmax, *blend_count;
};


// ---------------------------------------------------------------- workload (synthetic.cpp)
// make_street_scene (synthetic.cpp:236-312) with Camera::look_at (core_types.cpp:40-60),
// quat_from_axes (synthetic.cpp:21-27), quat_from_rotation (math_util.cpp:73-92) and Rng
// (math_util.hpp:27-63), plus the scale_mult density knob of SURVEY.md §8d (s1 *= k right
// after its draw). Operand draws follow the order GCC gives the reference's expressions
// (right to left; pinned against oracle/_ref by tests/test_ref_pin.py).
struct SplitMix {
  uint64_t state;
  uint64_t next() {
    uint64_t z = (state += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  double u01() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  double uni(double lo, double hi) { return lo + (hi - lo) * u01(); }
  double gauss() {
    double a = u01();
    const double b = u01();
    if (a < 1e-300) a = 1e-300;
    return std::sqrt(-2.0 * std::log(a)) * std::cos(2.0 * M_PI * b);
  }
};
inline V3 v3(double x, double y, double z) { return V3{{x, y, z}}; }
inline V3 vadd(const V3& a, const V3& b) { return v3(a.v[0] + b.v[0], a.v[1] + b.v[1], a.v[2] + b.v[2]); }
inline V3 vmul(double s, const V3& a) { return v3(s * a.v[0], s * a.v[1], s * a.v[2]); }
inline V3 vcross(const V3& a, const V3& b) {
  return v3(a.v[1] * b.v[2] - a.v[2] * b.v[1], a.v[2] * b.v[0] - a.v[0] * b.v[2], a.v[0] * b.v[1] - a.v[1] * b.v[0]);
}
inline V3 vnormalized(const V3& a) {  // MatrixBase::normalized: a / sqrt(squaredNorm) when > 0
  const double z = dot3(a, a);
  return z > 0 ? v3(a.v[0] / std::sqrt(z), a.v[1] / std::sqrt(z), a.v[2] / std::sqrt(z)) : a;
}
// quat_from_rotation (math_util.cpp:73-92); M3 column-major like Eigen.
void quat_of(const M3& r, double q[4]) {
  const double tr = sum3(r.at(0, 0), r.at(1, 1), r.at(2, 2));
  if (tr > 0) {
    const double s = std::sqrt(tr + 1.0) * 2;
    q[0] = 0.25 * s; q[1] = (r.at(2, 1) - r.at(1, 2)) / s; q[2] = (r.at(0, 2) - r.at(2, 0)) / s;
    q[3] = (r.at(1, 0) - r.at(0, 1)) / s;
  } else if (r.at(0, 0) > r.at(1, 1) && r.at(0, 0) > r.at(2, 2)) {
    const double s = std::sqrt(1.0 + r.at(0, 0) - r.at(1, 1) - r.at(2, 2)) * 2;
    q[0] = (r.at(2, 1) - r.at(1, 2)) / s; q[1] = 0.25 * s; q[2] = (r.at(0, 1) + r.at(1, 0)) / s;
    q[3] = (r.at(0, 2) + r.at(2, 0)) / s;
  } else if (r.at(1, 1) > r.at(2, 2)) {
    const double s = std::sqrt(1.0 + r.at(1, 1) - r.at(0, 0) - r.at(2, 2)) * 2;
    q[0] = (r.at(0, 2) - r.at(2, 0)) / s; q[1] = (r.at(0, 1) + r.at(1, 0)) / s; q[2] = 0.25 * s;
    q[3] = (r.at(1, 2) + r.at(2, 1)) / s;
  } else {
    const double s = std::sqrt(1.0 + r.at(2, 2) - r.at(0, 0) - r.at(1, 1)) * 2;
    q[0] = (r.at(1, 0) - r.at(0, 1)) / s; q[1] = (r.at(0, 2) + r.at(2, 0)) / s; q[2] = (r.at(1, 2) + r.at(2, 1)) / s;
    q[3] = 0.25 * s;
  }
  if (q[0] < 0) for (int i = 0; i < 4; ++i) q[i] = -q[i];
  const double n = std::sqrt((q[0] * q[0] + q[2] * q[2]) + (q[1] * q[1] + q[3] * q[3]));  // Vector4d::norm
  for (int i = 0; i < 4; ++i) q[i] = q[i] / n;
}
void quat_axes(const V3& tu, const V3& tv, double q[4]) {  // synthetic.cpp:21-27
  M3 r;
  const V3 c0 = vnormalized(tu), c2 = vnormalized(vcross(tu, tv)), c1 = vcross(c2, c0);
  for (int i = 0; i < 3; ++i) { r.at(i, 0) = c0.v[i]; r.at(i, 1) = c1.v[i]; r.at(i, 2) = c2.v[i]; }
  quat_of(r, q);
}
// Camera::look_at (core_types.cpp:40-60) -> psm_camera (r_cw column-major).
bool look_at(const V3& eye, const V3& target, const V3& up, double fx, double fy, int w, int h, double nc,
             double fc, psm_camera* out) {
  V3 fwd = v3(target.v[0] - eye.v[0], target.v[1] - eye.v[1], target.v[2] - eye.v[2]);
  if (norm3(fwd) < 1e-12) return false;
  fwd = vnormalized(fwd);
  V3 right = vcross(fwd, up);
  if (norm3(right) < 1e-9) {
    right = vcross(fwd, v3(1, 0, 0));
    if (norm3(right) < 1e-9) right = vcross(fwd, v3(0, 1, 0));
  }
  right = vnormalized(right);
  const V3 down = vcross(fwd, right);
  M3 rcw;  // r_wc = [right down fwd]; r_cw = r_wc^T
  for (int j = 0; j < 3; ++j) { rcw.at(0, j) = right.v[j]; rcw.at(1, j) = down.v[j]; rcw.at(2, j) = fwd.v[j]; }
  M3 neg;
  for (int i = 0; i < 9; ++i) neg.m[i] = -rcw.m[i];
  const V3 t = matvec(neg, eye);  // -r_cw * eye
  std::memcpy(out->r_cw, rcw.m, sizeof out->r_cw);
  for (int i = 0; i < 3; ++i) out->t_cw[i] = t.v[i];
  out->fx = fx; out->fy = fy; out->cx = 0.5 * w; out->cy = 0.5 * h;
  out->width = w; out->height = h; out->near_clip = nc; out->far_clip = fc;
  return true;
}
}  // namespace

extern "C" {

// Diagnostic counters of one render (not part of the reference API).
typedef struct oracle_stats {
  uint64_t candidates_tested;  // (pixel, list entry) pairs reaching the support test
  uint64_t support_pass;       // ... passing it
  uint64_t contributors;       // entries pushed (alpha >= alpha_min)
  double t_project_ms, t_bin_ms, t_blend_ms, t_total_ms;
} oracle_stats;

// One projected surfel, flattened for the known-answer tests.
typedef struct oracle_projected {
  int32_t status;  // 1 projected, 0 culled, -1 degenerate quaternion
  double center[2];
  double sigma[4];      // column-major
  double sort_depth;
  double h[9], h_inv[9];  // column-major
  double finv[4];       // column-major
  double normal_vis[3];
} oracle_projected;

int oracle_project_surfel(const double* s13, const psm_camera* cam, double chi2, oracle_projected* out) {
  Projected p;
  const int st = project_surfel(s13, cam_from(cam), chi2, p);
  std::memset(out, 0, sizeof *out);
  out->status = st;
  if (st != 1) return st;
  out->center[0] = p.center[0]; out->center[1] = p.center[1];
  std::memcpy(out->sigma, p.sigma.m, sizeof out->sigma);
  out->sort_depth = p.sort_depth;
  std::memcpy(out->h, p.h.m, sizeof out->h);
  std::memcpy(out->h_inv, p.h_inv.m, sizeof out->h_inv);
  std::memcpy(out->finv, p.finv.m, sizeof out->finv);
  std::memcpy(out->normal_vis, p.normal_vis, sizeof out->normal_vis);
  return 1;
}

// project_surfel_backward (raster.cpp:179-203) of one surfel under its own projection, through
// the shared psm_geom_backward: g_hinv row-major in; returns the projection status.
int oracle_project_surfel_backward(const double* s13, const psm_camera* pcam, double chi2, const double* g_hinv,
                                   double* d_center, double* d_rot, double* d_scales) {
  const Cam cam = cam_from(pcam);
  Projected p;
  const int st = project_surfel(s13, cam, chi2, p);
  if (st != 1) return st;
  double hinv[9];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) hinv[r * 3 + c] = p.h_inv.at(r, c);
  psm_geom_backward(s13, cam.r.m, hinv, g_hinv, d_center, d_rot, d_scales);
  return 1;
}

// sample_surfel_alpha + evaluate_alpha, raster.cpp:154-177
double oracle_evaluate_alpha(const double* s13, const psm_camera* pcam, double px, double py,
                             const psm_raster_config* cfg, double* u_out, double* v_out, double* w2_out,
                             int32_t* inside_out) {
  const Cam cam = cam_from(pcam);
  Projected p;
  *inside_out = 0;
  if (project_surfel(s13, cam, cfg->chi2, p) != 1) return 0.0;
  if (cfg->support_cutoff) {
    const double d0 = px - p.center[0], d1 = py - p.center[1];
    // d.dot(finv * d): (finv*d)_i = finv(i,0) d0 + finv(i,1) d1
    const double fd0 = p.finv.at(0, 0) * d0 + p.finv.at(0, 1) * d1;
    const double fd1 = p.finv.at(1, 0) * d0 + p.finv.at(1, 1) * d1;
    if (d0 * fd0 + d1 * fd1 > cfg->chi2) return 0.0;
  }
  const V3 ray{{(px - cam.cx) / cam.fx, (py - cam.cy) / cam.fy, 1.0}};
  const V3 w = matvec(p.h_inv, ray);
  if (!(w.v[2] > 1e-14)) return 0.0;
  const double u = w.v[0] / w.v[2], v = w.v[1] / w.v[2];
  *u_out = u; *v_out = v; *w2_out = w.v[2]; *inside_out = 1;
  const double alpha = s13[9] * oexp(-0.5 * (u * u + v * v));
  return alpha < cfg->alpha_min ? 0.0 : alpha;
}

// Projects every surfel and bins them. Outputs (any may be NULL):
//   tile_counts[tiles]; list_src[cap] concatenated per-tile lists (source ids);
//   per_surfel_tiles[n] number of tiles each source surfel was assigned.
int oracle_bin(const double* surfels13, int64_t n, const psm_camera* pcam, const psm_raster_config* cfg,
               int32_t binning, double chi2, int32_t* tile_counts, int32_t* list_src, int64_t cap,
               int32_t* per_surfel_tiles, psm_counters* counters) {
  const Cam cam = cam_from(pcam);
  std::vector<Projected> projected;
  for (int64_t i = 0; i < n; ++i) {
    Projected p;
    const int st = project_surfel(surfels13 + 13 * i, cam, cfg->chi2, p);
    if (st < 0) return PSM_EINVAL;
    if (st == 1) { p.source = static_cast<int>(i); projected.push_back(p); }
  }
  const Grid g = bin(projected, cam, cfg->tile_size, chi2, binning);
  int64_t at = 0;
  if (per_surfel_tiles) std::memset(per_surfel_tiles, 0, sizeof(int32_t) * n);
  for (size_t t = 0; t < g.tiles.size(); ++t) {
    if (tile_counts) tile_counts[t] = static_cast<int32_t>(g.tiles[t].size());
    for (int idx : g.tiles[t]) {
      if (list_src && at < cap) list_src[at] = projected[idx].source;
      if (per_surfel_tiles) per_surfel_tiles[projected[idx].source]++;
      ++at;
    }
  }
  if (counters) {
    counters->rn_total = g.rn_total;
    counters->rn_per_tile = g.rn_per_tile;
    counters->n_proj = static_cast<int64_t>(projected.size());
    counters->tiles_x = g.tiles_x;
    counters->tiles_y = g.tiles_y;
    counters->nonempty_tiles = g.nonempty;
    counters->blended_total = 0;
  }
  return PSM_OK;
}

// assign_labels (panoptic.cpp:36-91). surfels13: N x 13 (centre = columns 0..2);
// f_ins: N x c_ins; queries: feat [n_queries x c_ins], mean [n_queries x 3], cov
// [n_queries x 9] column-major, alive flags. dist_out: N x n_queries (per-surfel
// contiguous, the MatX column of surfel s); argmax_out: N (query index, -1 when no
// query is alive). Parallel over surfels; each surfel is independent.
void oracle_assign_labels(const double* surfels13, int64_t n, const double* f_ins, int32_t c_ins, int32_t n_queries,
                          const double* q_feat, const double* q_mean, const double* q_cov, const int32_t* q_alive,
                          double* dist_out, int32_t* argmax_out, int32_t threads) {
  std::vector<int> alive;
  for (int q = 0; q < n_queries; ++q)
    if (q_alive[q]) alive.push_back(q);
  const int na = static_cast<int>(alive.size());
  std::vector<double> fq(static_cast<size_t>(na) * c_ins), mean(3 * na), inv(9 * na);
  for (int a = 0; a < na; ++a) {
    for (int c = 0; c < c_ins; ++c) fq[a * c_ins + c] = q_feat[static_cast<int64_t>(alive[a]) * c_ins + c];
    for (int i = 0; i < 3; ++i) mean[a * 3 + i] = q_mean[alive[a] * 3 + i];
    psm_query_inverse(q_cov + alive[a] * 9, inv.data() + a * 9);
  }
  parallel_chunks(n, threads, [&](int64_t b, int64_t e) {
    std::vector<double> av(na > 0 ? na : 1);
    for (int64_t s = b; s < e; ++s) {
      double* row = dist_out + s * n_queries;
      for (int q = 0; q < n_queries; ++q) row[q] = 0.0;
      if (na == 0) {
        argmax_out[s] = -1;
        continue;
      }
      const int best = psm_assign_one(f_ins + s * c_ins, c_ins, surfels13 + s * 13, na, fq.data(), mean.data(),
                                      inv.data(), av.data(), 1, psm_exp_tab_host);
      for (int a = 0; a < na; ++a) row[alive[a]] = av[a];
      argmax_out[s] = alive[best];
    }
  });
}

// psm_exp itself, vectorised, for the libm-substitution pin.
void oracle_psm_exp(const double* x, int64_t n, double* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = psm_exp(x[i]);
}

// glibc exp exactly as the reference calls it (raster.cpp:390), for the libm pin.
void oracle_libm_exp(const double* x, int64_t n, double* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = std::exp(x[i]);
}

// topk_select over explicit keys (raster.cpp:225-251); selected[m] out.
void oracle_topk_select(const double* weights, const int32_t* proj, int32_t m, int32_t k, int8_t* selected) {
  std::vector<WeightKey> keys(m), best;
  std::vector<char> sel;
  for (int i = 0; i < m; ++i) keys[i] = {weights[i], proj[i], i};
  topk_select(keys.data(), m, k, best, sel);
  for (int i = 0; i < m; ++i) selected[i] = sel[i];
}

// render_into, raster.cpp:273-511. Planes are fp64 HWC (reference types);
// any plane pointer may be NULL (computed, not stored). debug / stats optional.
// RenderCache::pixels (raster.hpp:75-82, filled at raster.cpp:399-403): per-pixel
// contributor (source, alpha) in blend order, CSR over pixels.
typedef struct oracle_cache {
  int64_t* offsets;  // [W*H + 1]
  int32_t* src;      // [cap]
  double* alpha;     // [cap]
  int64_t cap;
} oracle_cache;


// make_street_scene on the oracle (see the workload section). Two-phase like
// psm_make_street_scene: NULL surfels13 returns n (and the camera) only.
int oracle_make_street_scene(const psm_street_spec* spec, int64_t* n_out, double* surfels13, double* f_sem,
                             double* labels, double* f_ins, psm_camera* cam) {
  struct Group { V3 o, e1, e2; int inst; double share; };
  std::vector<Group> gs = {{v3(-4, 1.5, 1.5), v3(8, 0, 0), v3(0, 0, 38), 0, 0.10},
                           {v3(-4.0, 1.5, 1.5), v3(0.9, -4.0, 0), v3(0, 0, 38), 1, 0.06},
                           {v3(4.0, 1.5, 1.5), v3(-0.9, -4.0, 0), v3(0, 0, 38), 2, 0.06}};
  const int ninst = spec->n_instances, layers = 18;
  const int bands = std::max(1, (ninst - 3) / layers + 1);
  for (int l = 0; l < layers; ++l)
    for (int b = 0; b < bands; ++b) {
      const double bw = 7.2 / bands;
      gs.push_back({v3(-3.6 + b * bw, -2.6, 3.2 + 2.0 * l), v3(bw, 0, 0), v3(0, 5.2, 0),
                    3 + (b % std::max(1, ninst - 3)), 0.78 / (layers * bands)});
    }
  std::vector<int> counts;
  int64_t n = 0;
  for (const Group& g : gs) {
    counts.push_back(static_cast<int>(std::round(g.share * spec->n_surfels)));
    n += counts.back();
  }
  *n_out = n;
  if (cam && !look_at(v3(0, 0, 0), v3(0, 0, 20), v3(0, -1, 0), 0.8 * spec->image_w, 0.8 * spec->image_w,
                      spec->image_w, spec->image_h, 0.1, 200.0, cam))
    return PSM_EINVAL;
  if (!surfels13) return PSM_OK;
  SplitMix rng{spec->seed};
  const double k = spec->scale_mult > 0 ? spec->scale_mult : 1.0;
  int64_t at = 0;
  for (size_t gi = 0; gi < gs.size(); ++gi) {
    const Group& g = gs[gi];
    const V3 u1 = vnormalized(g.e1), u2 = vnormalized(g.e2), nrm = vnormalized(vcross(u1, u2));
    for (int i = 0; i < counts[gi]; ++i, ++at) {
      double* s = surfels13 + 13 * at;
      const double jit = rng.uni(-0.03, 0.03), b2 = rng.u01(), b1 = rng.u01();  // right-to-left operands
      const V3 c = vadd(vadd(vadd(g.o, vmul(b1, g.e1)), vmul(b2, g.e2)), vmul(jit, nrm));
      for (int d = 0; d < 3; ++d) s[d] = c.v[d];
      const double phi = rng.uni(0, M_PI);
      quat_axes(vadd(vmul(std::cos(phi), u1), vmul(std::sin(phi), u2)),
                vadd(vmul(-std::sin(phi), u1), vmul(std::cos(phi), u2)), s + 3);
      const double s1 = rng.uni(0.45, 1.1) * k;
      const double aspect = rng.uni(spec->min_aspect, 2.0 * spec->min_aspect);
      s[7] = s1; s[8] = s1 / aspect;
      s[9] = rng.uni(0.30, 0.70);
      for (int d = 2; d >= 0; --d) s[10 + d] = rng.uni(0.2, 0.9);  // Vec3(u, u, u) constructor args
      for (int c2 = 0; c2 < spec->c_sem; ++c2) {
        const double v = rng.gauss();
        if (f_sem) f_sem[at * spec->c_sem + c2] = v;
      }
      for (int c2 = 0; c2 < 8; ++c2) {
        const double v = 0.3 * rng.gauss();
        if (f_ins) f_ins[at * 8 + c2] = v;
      }
      if (labels)
        for (int q = 0; q < ninst; ++q) labels[at * ninst + q] = q == g.inst ? 0.92 : 0.08 / (ninst - 1);
    }
  }
  return PSM_OK;
}

// Backward state (pipeline.cpp:347-460): upstream plane gradients in, per-surfel sums out.
struct BackwardAcc {
  const psm_plane_grads* g;
  std::vector<double> opacity, color, fsem, lab, hinv;  // per source; hinv per projected (row-major)
  std::vector<double> center, rotation, scales;         // per source
  std::vector<std::vector<Scratch::Entry>> rows;        // per pixel: the forward's contributors
};

// Blending backward (pipeline.cpp:347-460) in the reference's summation order: the pixels in
// kGradChunks = 16 linear ranges, each summed (pixel order) into its own zeroed buffers, the
// buffers then added to the totals in chunk order (pipeline.cpp:355-376,455-463). With that
// order the sums are the reference's bit for bit (tests/test_ref_pin.py).
static void blend_backward(BackwardAcc* bwd, const double* surfels13, const double* f_sem, int c_sem,
                           const double* labels, int n_q, const Cam& cam, const psm_raster_config* cfg,
                           const std::vector<Projected>& projected, int n) {
  const int n_proj = static_cast<int>(projected.size());
  const int64_t total_px = static_cast<int64_t>(cam.w) * cam.h;
  const bool topk = cfg->blending == PSM_BLEND_TOPK;
  const int k_sel = std::max(cfg->top_k, 1);
  constexpr int kGradChunks = 16;
  bwd->hinv.assign(static_cast<size_t>(n_proj) * 9, 0.0);
  std::vector<double> b_hinv, b_op, b_col, b_fsem, b_lab;
  std::vector<double> t_chain, wbuf;
  std::vector<WeightKey> keys, best;
  std::vector<char> selected;
  for (int c = 0; c < kGradChunks; ++c) {
    b_hinv.assign(static_cast<size_t>(n_proj) * 9, 0.0);
    b_op.assign(static_cast<size_t>(n), 0.0);
    b_col.assign(static_cast<size_t>(n) * 3, 0.0);
    b_fsem.assign(static_cast<size_t>(n) * c_sem, 0.0);
    b_lab.assign(static_cast<size_t>(n) * n_q, 0.0);
    for (int64_t pix = total_px * c / kGradChunks; pix < total_px * (c + 1) / kGradChunks; ++pix) {
      const auto& ent = bwd->rows[pix];
      const int m = static_cast<int>(ent.size());
      if (m == 0) continue;
      const int x = static_cast<int>(pix % cam.w), y = static_cast<int>(pix / cam.w);
      const double rx = (x + 0.5 - cam.cx) / cam.fx, ry = (y + 0.5 - cam.cy) / cam.fy;
      const double zero3[3] = {0, 0, 0};
      const double* gc = bwd->g->color ? bwd->g->color + 3 * pix : zero3;
      const double* gf = (c_sem > 0 && bwd->g->sem_feat) ? bwd->g->sem_feat + pix * c_sem : nullptr;
      const double* gi = (n_q > 0 && bwd->g->ins_dist) ? bwd->g->ins_dist + pix * n_q : nullptr;
      t_chain.assign(m + 1, 1.0);
      wbuf.assign(m, 0.0);
      for (int j = 0; j < m; ++j) {
        wbuf[j] = ent[j].alpha * t_chain[j];
        t_chain[j + 1] = t_chain[j] * (1.0 - ent[j].alpha);
      }
      if (topk && m > k_sel) {  // the forward's Top-K selection, replayed (pipeline.cpp:383-388)
        keys.resize(m);
        for (int i = 0; i < m; ++i) keys[i] = {wbuf[i], ent[i].proj, i};
        topk_select(keys.data(), m, k_sel, best, selected);
      } else {
        selected.assign(m, 1);
      }
      double suffix = t_chain[m] * (gc[0] * cfg->background[0] + gc[1] * cfg->background[1] + gc[2] * cfg->background[2]);
      for (int j = m - 1; j >= 0; --j) {
        const auto& e = ent[j];
        const int64_t src = projected[e.proj].source;
        const double* sf = surfels13 + 13 * src;
        const double w_j = wbuf[j];
        double direct = gc[0] * sf[10] + gc[1] * sf[11] + gc[2] * sf[12];
        for (int k = 0; k < 3; ++k) b_col[src * 3 + k] += w_j * gc[k];
        if (selected[j]) {
          if (gf) {
            double dot = 0;
            for (int i = 0; i < c_sem; ++i) {
              dot += gf[i] * f_sem[src * c_sem + i];
              b_fsem[src * c_sem + i] += w_j * gf[i];
            }
            direct += dot;
          }
          if (gi) {
            double dot = 0;
            for (int i = 0; i < n_q; ++i) {
              dot += gi[i] * labels[src * n_q + i];
              b_lab[src * n_q + i] += w_j * gi[i];
            }
            direct += dot;
          }
        }
        const double one_minus = 1.0 - e.alpha;
        const double g_alpha = t_chain[j] * direct - (one_minus > 0 ? suffix / one_minus : 0.0);
        suffix += w_j * direct;
        const double d_sigma = oexp(-0.5 * (e.u * e.u + e.v * e.v));
        b_op[src] += d_sigma * g_alpha;
        const double g_dsigma = sf[9] * g_alpha;
        const double g_u = -e.u * d_sigma * g_dsigma;
        const double g_v = -e.v * d_sigma * g_dsigma;
        const Projected& pr = projected[e.proj];
        const double w2 = pr.h_inv.at(2, 0) * rx + pr.h_inv.at(2, 1) * ry + pr.h_inv.at(2, 2) * 1.0;
        const double gw[3] = {g_u / w2, g_v / w2, -(e.u * g_u + e.v * g_v) / w2};
        const double ray[3] = {rx, ry, 1.0};
        double* gh = &b_hinv[static_cast<size_t>(e.proj) * 9];
        for (int r = 0; r < 3; ++r)
          for (int k = 0; k < 3; ++k) gh[r * 3 + k] += gw[r] * ray[k];
      }
    }
    // deterministic ordered merge (pipeline.cpp:455-463)
    for (size_t i = 0; i < b_hinv.size(); ++i) bwd->hinv[i] += b_hinv[i];
    for (int64_t s2 = 0; s2 < n; ++s2) {
      bwd->opacity[s2] += b_op[s2];
      for (int k = 0; k < 3; ++k) bwd->color[s2 * 3 + k] += b_col[s2 * 3 + k];
    }
    for (size_t i = 0; i < b_fsem.size(); ++i) bwd->fsem[i] += b_fsem[i];
    for (size_t i = 0; i < b_lab.size(); ++i) bwd->lab[i] += b_lab[i];
  }
}

static int render_impl(const double* surfels13, int64_t n, const double* f_sem, int32_t c_sem,
                       const double* labels, int32_t n_q, const psm_camera* pcam, const psm_raster_config* cfg_in,
                       double* color, double* depth, double* normal, double* sem_feat, double* ins_dist,
                       int32_t* ins_argmax, double* alpha_acc, int32_t* blend_count, psm_counters* counters,
                       psm_debug* dbg, oracle_stats* stats, oracle_cache* cache, BackwardAcc* bwd = nullptr) {
  psm_raster_config cfg_local = *cfg_in;
  if (bwd) cfg_local.threads = 1;  // the backward sums into shared arrays: one deterministic pass
  const psm_raster_config* cfg = &cfg_local;
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  const Cam cam = cam_from(pcam);
  const int w = cam.w, h = cam.h;
  if (n == 0) c_sem = 0;  // SceneMap::c_sem() of an empty scene (core_types.hpp:108)
  if (labels == nullptr) n_q = 0;
  const int ts = cfg->tile_size;

  // reset_plane x8 (raster.cpp:279-295)
  const size_t npx = static_cast<size_t>(w) * h;
  std::vector<double> own_color, own_alpha;
  std::vector<int32_t> own_count, own_arg;
  if (!color) { own_color.resize(npx * 3); color = own_color.data(); }
  if (!alpha_acc) { own_alpha.resize(npx); alpha_acc = own_alpha.data(); }
  if (!blend_count) { own_count.resize(npx); blend_count = own_count.data(); }
  if (!ins_argmax) { own_arg.resize(npx); ins_argmax = own_arg.data(); }
  for (size_t p = 0; p < npx; ++p) {
    color[3 * p] = cfg->background[0];
    color[3 * p + 1] = cfg->background[1];
    color[3 * p + 2] = cfg->background[2];
    alpha_acc[p] = 0; blend_count[p] = 0; ins_argmax[p] = -1;
  }
  if (depth) std::fill(depth, depth + npx * 2, 0.0);
  if (normal) std::fill(normal, normal + npx * 3, 0.0);
  if (sem_feat) std::fill(sem_feat, sem_feat + npx * c_sem, 0.0);
  if (ins_dist) std::fill(ins_dist, ins_dist + npx * n_q, 0.0);

  // projection (raster.cpp:297-305), serial like the reference
  std::vector<Projected> projected;
  projected.reserve(n);
  for (int64_t i = 0; i < n; ++i) {
    Projected p;
    const int st = project_surfel(surfels13 + 13 * i, cam, cfg->chi2, p);
    if (st < 0) return PSM_EINVAL;  // rotation_from_quat throws
    if (st == 1) { p.source = static_cast<int>(i); projected.push_back(p); }
  }
  const auto t1 = clk::now();
  int binning = cfg->binning;
  if (binning == PSM_BIN_ELLIPSE && !cfg->support_cutoff) binning = PSM_BIN_AABB;
  const Grid grid = bin(projected, cam, ts, cfg->chi2, binning);
  const auto t2 = clk::now();

  const bool topk = cfg->blending == PSM_BLEND_TOPK;
  const int k_sel = std::max(cfg->top_k, 1);
  std::vector<uint64_t> tile_blend(grid.tiles.size(), 0), tile_tested(grid.tiles.size(), 0),
      tile_pass(grid.tiles.size(), 0), tile_contrib(grid.tiles.size(), 0);

  // hot SoA (raster.cpp:321-353)
  const int n_proj = static_cast<int>(projected.size());
  struct HotReject { double cx, cy, f00, f01, f11; };
  struct HotGeom { double h[9]; double opacity; };
  std::vector<HotReject> hot_reject(n_proj);
  std::vector<HotGeom> hot_geom(n_proj);
  std::vector<double> hot_color(static_cast<size_t>(n_proj) * 3), hot_normal(static_cast<size_t>(n_proj) * 3);
  for (int i = 0; i < n_proj; ++i) {
    const Projected& pr = projected[i];
    hot_reject[i] = {pr.center[0], pr.center[1], pr.finv.at(0, 0), pr.finv.at(0, 1), pr.finv.at(1, 1)};
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) hot_geom[i].h[r * 3 + c] = pr.h_inv.at(r, c);
    const double* sf = surfels13 + 13 * static_cast<int64_t>(pr.source);
    hot_geom[i].opacity = sf[9];
    for (int c = 0; c < 3; ++c) {
      hot_color[static_cast<size_t>(i) * 3 + c] = sf[10 + c];
      hot_normal[static_cast<size_t>(i) * 3 + c] = pr.normal_vis[c];
    }
  }
  if (bwd) bwd->rows.assign(npx, {});
  const double rd_bg0 = cfg->background[0], rd_bg1 = cfg->background[1], rd_bg2 = cfg->background[2];
  std::vector<std::vector<std::pair<int, double>>> cache_rows(cache ? npx : 0);
  const bool rdn = cfg->render_depth_normal != 0;

  parallel_chunks(static_cast<int64_t>(grid.tiles.size()), cfg->threads, [&](int64_t t_begin, int64_t t_end) {
    Scratch scratch;
    for (int64_t t = t_begin; t < t_end; ++t) {
      const auto& list = grid.tiles[t];
      if (list.empty()) continue;
      const int tx = static_cast<int>(t) % grid.tiles_x;
      const int ty = static_cast<int>(t) / grid.tiles_x;
      const int x0 = tx * ts, x1 = std::min(w, x0 + ts);
      const int y0 = ty * ts, y1 = std::min(h, y0 + ts);
      uint64_t blends = 0, tested = 0, passed = 0, contrib = 0;
      scratch.entries.reserve(list.size());
      scratch.accum.resize(std::max(c_sem + n_q, 1));
      for (int y = y0; y < y1; ++y) {
        for (int x = x0; x < x1; ++x) {
          const size_t pix = static_cast<size_t>(y) * w + x;
          const double px = x + 0.5, py = y + 0.5;
          const double rx = (px - cam.cx) / cam.fx;
          const double ry = (py - cam.cy) / cam.fy;
          scratch.entries.clear();
          double transmit = 1.0;
          for (int idx : list) {
            ++tested;
            if (cfg->support_cutoff) {
              const HotReject& hr = hot_reject[idx];
              const double dx = px - hr.cx;
              const double dy = py - hr.cy;
              if (hr.f00 * dx * dx + 2.0 * hr.f01 * dx * dy + hr.f11 * dy * dy > cfg->chi2) continue;
            }
            ++passed;
            const HotGeom& hg = hot_geom[idx];
            const double w0 = hg.h[0] * rx + hg.h[1] * ry + hg.h[2];
            const double w1 = hg.h[3] * rx + hg.h[4] * ry + hg.h[5];
            const double w2 = hg.h[6] * rx + hg.h[7] * ry + hg.h[8];
            if (!(w2 > 1e-14)) continue;
            const double rcp = 1.0 / w2;
            const double u = w0 * rcp, v = w1 * rcp;
            const double alpha = hg.opacity * oexp(-0.5 * (u * u + v * v));
            if (alpha < cfg->alpha_min || alpha <= 0.0) continue;
            scratch.entries.push_back({idx, alpha, u, v, alpha * transmit, rcp});
            transmit *= 1.0 - alpha;
            if (transmit < cfg->t_min) break;
          }
          const int m = static_cast<int>(scratch.entries.size());
          contrib += m;
          if (cache) {
            std::vector<std::pair<int, double>>& rec = cache_rows[pix];
            rec.reserve(m);
            for (const auto& e : scratch.entries) rec.push_back({projected[e.proj].source, e.alpha});
          }
          blend_count[pix] = m;
          alpha_acc[pix] = 1.0 - transmit;

          double acc_r = 0, acc_g = 0, acc_b = 0, exp_depth = 0, dom_depth = 0, dom_w = 0, nx = 0, ny = 0, nz = 0;
          for (const auto& e : scratch.entries) {
            const double* c = &hot_color[static_cast<size_t>(e.proj) * 3];
            acc_r += e.weight * c[0];
            acc_g += e.weight * c[1];
            acc_b += e.weight * c[2];
            if (rdn) {
              exp_depth += e.weight * e.depth;
              if (e.weight > dom_w) { dom_w = e.weight; dom_depth = e.depth; }
              const double* nrm = &hot_normal[static_cast<size_t>(e.proj) * 3];
              nx += e.weight * nrm[0];
              ny += e.weight * nrm[1];
              nz += e.weight * nrm[2];
            }
          }
          color[3 * pix] = acc_r + transmit * rd_bg0;
          color[3 * pix + 1] = acc_g + transmit * rd_bg1;
          color[3 * pix + 2] = acc_b + transmit * rd_bg2;
          if (rdn) {
            if (depth) { depth[2 * pix] = exp_depth; depth[2 * pix + 1] = dom_depth; }
            if (normal) { normal[3 * pix] = nx; normal[3 * pix + 1] = ny; normal[3 * pix + 2] = nz; }
          }

          const Scratch::Entry* blend_list = scratch.entries.data();
          int blend_n = m;
          if (topk && m > k_sel) {
            scratch.keys.resize(m);
            for (int i = 0; i < m; ++i) scratch.keys[i] = {scratch.entries[i].weight, scratch.entries[i].proj, i};
            topk_select(scratch.keys.data(), m, k_sel, scratch.best, scratch.selected);
            scratch.selected_entries.clear();
            for (int i = 0; i < m; ++i)
              if (scratch.selected[i]) scratch.selected_entries.push_back(scratch.entries[i]);
            blend_list = scratch.selected_entries.data();
            blend_n = static_cast<int>(scratch.selected_entries.size());
          }
          if (topk && dbg && dbg->topk_src) {
            int32_t* slot = dbg->topk_src + pix * k_sel;
            for (int i = 0; i < k_sel; ++i) slot[i] = i < blend_n ? projected[blend_list[i].proj].source : -1;
          }

          if (bwd) bwd->rows[pix] = scratch.entries;  // the RenderCache row (raster.cpp:399-403)

          const int feat_dims = c_sem + n_q;
          blends += blend_n;
          if (feat_dims > 0 && blend_n > 0) {
            double* acc_sem = scratch.accum.data();
            double* acc_ins = scratch.accum.data() + c_sem;
            for (int i = 0; i < blend_n; ++i) {
              const auto& e = blend_list[i];
              const double wgt = e.weight;
              const int64_t src = projected[e.proj].source;
              const double* f = c_sem > 0 ? f_sem + src * c_sem : nullptr;
              const double* col = n_q > 0 ? labels + src * n_q : nullptr;
              if (i == 0) {
                for (int c = 0; c < c_sem; ++c) acc_sem[c] = wgt * f[c];
                for (int c = 0; c < n_q; ++c) acc_ins[c] = wgt * col[c];
                continue;
              }
              for (int c = 0; c < c_sem; ++c) acc_sem[c] += wgt * f[c];
              for (int c = 0; c < n_q; ++c) acc_ins[c] += wgt * col[c];
            }
            if (c_sem > 0 && sem_feat) {
              double* sem_px = sem_feat + pix * c_sem;
              for (int c = 0; c < c_sem; ++c) sem_px[c] = acc_sem[c];
            }
            if (n_q > 0) {
              int arg = 0;
              for (int c = 0; c < n_q; ++c) {
                if (ins_dist) ins_dist[pix * n_q + c] = acc_ins[c];
                if (acc_ins[c] > acc_ins[arg]) arg = c;
              }
              ins_argmax[pix] = arg;
            }
          }
        }
      }
      tile_blend[t] = blends;
      tile_tested[t] = tested;
      tile_pass[t] = passed;
      tile_contrib[t] = contrib;
    }
  });
  const auto t3 = clk::now();

  if (bwd) {  // blending backward, then project_surfel_backward per projected surfel (pipeline.cpp:478-486)
    blend_backward(bwd, surfels13, f_sem, c_sem, labels, n_q, cam, cfg, projected, static_cast<int>(n));
    bwd->rows.clear();
    bwd->center.assign(static_cast<size_t>(n) * 3, 0.0);
    bwd->rotation.assign(static_cast<size_t>(n) * 4, 0.0);
    bwd->scales.assign(static_cast<size_t>(n) * 2, 0.0);
    for (int i = 0; i < n_proj; ++i) {
      const int64_t src = projected[i].source;
      double dc[3], dq[4], ds[2];
      psm_geom_backward(surfels13 + 13 * src, cam.r.m, hot_geom[i].h, &bwd->hinv[static_cast<size_t>(i) * 9], dc, dq,
                        ds);
      for (int k = 0; k < 3; ++k) bwd->center[src * 3 + k] += dc[k];
      for (int k = 0; k < 4; ++k) bwd->rotation[src * 4 + k] += dq[k];
      for (int k = 0; k < 2; ++k) bwd->scales[src * 2 + k] += ds[k];
    }
  }
  const uint64_t blended_total = std::accumulate(tile_blend.begin(), tile_blend.end(), uint64_t{0});
  if (counters) {
    counters->rn_total = grid.rn_total;
    counters->rn_per_tile = grid.rn_per_tile;
    counters->blended_total = blended_total;
    counters->n_proj = n_proj;
    counters->tiles_x = grid.tiles_x;
    counters->tiles_y = grid.tiles_y;
    counters->nonempty_tiles = grid.nonempty;
  }
  if (dbg) {
    // depth rank of every projected surfel: (sort_depth, source) order (raster.cpp:78-83)
    std::vector<int> order(n_proj);
    std::iota(order.begin(), order.end(), 0);
    std::sort(order.begin(), order.end(), [&](int a, int b) {
      if (projected[a].sort_depth != projected[b].sort_depth) return projected[a].sort_depth < projected[b].sort_depth;
      return projected[a].source < projected[b].source;
    });
    std::vector<int64_t> rank(n_proj);
    for (int r = 0; r < n_proj; ++r) rank[order[r]] = r;
    if (dbg->depth_order)
      for (int r = 0; r < n_proj && r < dbg->cap_proj; ++r) dbg->depth_order[r] = projected[order[r]].source;
    int64_t at = 0;
    for (size_t t = 0; t < grid.tiles.size(); ++t) {
      if (dbg->tile_ranges) dbg->tile_ranges[2 * t] = static_cast<int32_t>(at);
      for (int idx : grid.tiles[t]) {
        if (at < dbg->cap_keys) {
          if (dbg->tile_keys) dbg->tile_keys[at] = (static_cast<uint64_t>(t) << 32) | static_cast<uint64_t>(rank[idx]);
          if (dbg->tile_vals) dbg->tile_vals[at] = projected[idx].source;
        }
        ++at;
      }
      if (dbg->tile_ranges) dbg->tile_ranges[2 * t + 1] = static_cast<int32_t>(at);
    }
  }
  if (cache) {
    int64_t at = 0;
    for (size_t p = 0; p < npx; ++p) {
      cache->offsets[p] = at;
      for (const auto& e : cache_rows[p]) {
        if (at < cache->cap) { cache->src[at] = e.first; cache->alpha[at] = e.second; }
        ++at;
      }
    }
    cache->offsets[npx] = at;
  }
  if (stats) {
    stats->candidates_tested = std::accumulate(tile_tested.begin(), tile_tested.end(), uint64_t{0});
    stats->support_pass = std::accumulate(tile_pass.begin(), tile_pass.end(), uint64_t{0});
    stats->contributors = std::accumulate(tile_contrib.begin(), tile_contrib.end(), uint64_t{0});
    auto ms = [](clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    stats->t_project_ms = ms(t0, t1);
    stats->t_bin_ms = ms(t1, t2);
    stats->t_blend_ms = ms(t2, t3);
    stats->t_total_ms = ms(t0, t3);
  }
  return PSM_OK;
}

int oracle_render(const double* surfels13, int64_t n, const double* f_sem, int32_t c_sem,
                  const double* labels, int32_t n_q, const psm_camera* pcam, const psm_raster_config* cfg,
                  double* color, double* depth, double* normal, double* sem_feat, double* ins_dist,
                  int32_t* ins_argmax, double* alpha_acc, int32_t* blend_count, psm_counters* counters,
                  psm_debug* dbg, oracle_stats* stats) {
  return render_impl(surfels13, n, f_sem, c_sem, labels, n_q, pcam, cfg, color, depth, normal, sem_feat, ins_dist,
                     ins_argmax, alpha_acc, blend_count, counters, dbg, stats, nullptr);
}

// render(..., RenderCache*) (raster.hpp:142-143): also returns the per-pixel contributor lists.
int oracle_render_cache(const double* surfels13, int64_t n, const double* f_sem, int32_t c_sem,
                        const double* labels, int32_t n_q, const psm_camera* pcam, const psm_raster_config* cfg,
                        double* color, double* sem_feat, int32_t* ins_argmax, int32_t* blend_count,
                        oracle_cache* cache) {
  return render_impl(surfels13, n, f_sem, c_sem, labels, n_q, pcam, cfg, color, nullptr, nullptr, sem_feat, nullptr,
                     ins_argmax, nullptr, blend_count, nullptr, nullptr, nullptr, cache);
}

// Blending backward + geometry chain (pipeline.cpp:347-486) on the oracle.
int oracle_render_backward(const double* surfels13, int64_t n, const double* f_sem, int32_t c_sem,
                           const double* labels, int32_t n_q, const psm_camera* pcam, const psm_raster_config* cfg,
                           const psm_plane_grads* g, psm_scene_grads* out) {
  if (n == 0) c_sem = 0;
  if (labels == nullptr) n_q = 0;
  BackwardAcc acc;
  acc.g = g;
  acc.opacity.assign(static_cast<size_t>(n), 0.0);
  acc.color.assign(static_cast<size_t>(n) * 3, 0.0);
  acc.fsem.assign(static_cast<size_t>(n) * c_sem, 0.0);
  acc.lab.assign(static_cast<size_t>(n) * n_q, 0.0);
  const int st = render_impl(surfels13, n, f_sem, c_sem, labels, n_q, pcam, cfg, nullptr, nullptr, nullptr, nullptr,
                             nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, &acc);
  if (st != PSM_OK) return st;
  if (acc.center.empty()) {
    acc.center.assign(static_cast<size_t>(n) * 3, 0.0);
    acc.rotation.assign(static_cast<size_t>(n) * 4, 0.0);
    acc.scales.assign(static_cast<size_t>(n) * 2, 0.0);
  }
  auto put = [](double* dst, const std::vector<double>& v) {
    if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(double));
  };
  put(out->opacity, acc.opacity);
  put(out->color, acc.color);
  put(out->f_sem, acc.fsem);
  put(out->labels, acc.lab);
  put(out->center, acc.center);
  put(out->rotation, acc.rotation);
  put(out->scales, acc.scales);
  return PSM_OK;
}

}  // extern "C"
