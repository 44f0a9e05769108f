// psimap_b200.hpp — C++ drop-in for the reference's render API, over the C-ABI (psm.h).
//
// Same namespace, names, argument meaning and error behaviour as the reference's
// proj/include/psimap/raster.hpp:42-172 and core_types.hpp:17-111, without Eigen:
//   psimap::render(scene, labels, cam, cfg)            raster.hpp:142-143
//   psimap::render_into(out, scene, labels, cam, cfg)  raster.hpp:147-148
//   psimap::bench_render(scene, labels, cam, reps, cfg) raster.hpp:171-172
// Types keep the reference's field names (Surfel::center/rotation/scales/opacity/
// color/f_sem/f_ins, Camera::r_cw/t_cw/fx/fy/cx/cy/width/height/near_clip/far_clip,
// RasterConfig, RenderTargets with double Plane<> outputs in HWC layout). Small
// fixed-size vectors replace Eigen's Vec2/3/4 and Mat3 (column-major like Eigen).
// `labels` is the N_q x N column-major matrix the reference passes as `const MatX*`.
//
// Every render runs on the GPU (libpsm.so); there is no CPU fallback. A degenerate
// quaternion throws std::invalid_argument like rotation_from_quat
// (math_util.cpp:48-50); other failures throw std::runtime_error. The stage functions
// (project_surfel, bin_circle, bin_aabb, sample_surfel_alpha, evaluate_alpha, topk_select,
// raster.hpp:87-126) and RenderCache (raster.hpp:76-82) run on the GPU too.
//
// Link: -I<repo>/include -L<repo>/paper_2604_10982_b200 -lpsm
#ifndef PSIMAP_B200_HPP
#define PSIMAP_B200_HPP

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "psm.h"

namespace psimap {

template <int N>
struct VecN {
  std::array<double, N> v{};
  double& operator[](int i) { return v[i]; }
  double operator[](int i) const { return v[i]; }
};
using Vec2 = VecN<2>;
using Vec3 = VecN<3>;
using Vec4 = VecN<4>;
inline Vec2 vec2(double a, double b) { return Vec2{{a, b}}; }
inline Vec3 vec3(double a, double b, double c) { return Vec3{{a, b, c}}; }
inline Vec4 vec4(double a, double b, double c, double d) { return Vec4{{a, b, c, d}}; }

struct Mat3 {  // column-major like Eigen::Matrix3d
  std::array<double, 9> m{{1, 0, 0, 0, 1, 0, 0, 0, 1}};
  double& operator()(int r, int c) { return m[c * 3 + r]; }
  double operator()(int r, int c) const { return m[c * 3 + r]; }
  static Mat3 Identity() { return Mat3{}; }
};

struct Mat2 {  // column-major like Eigen::Matrix2d
  std::array<double, 4> m{{0, 0, 0, 0}};
  double& operator()(int r, int c) { return m[c * 2 + r]; }
  double operator()(int r, int c) const { return m[c * 2 + r]; }
};

struct VecX : std::vector<double> {  // Eigen::VectorXd stand-in
  using std::vector<double>::vector;
};

// N_q x N, column-major: column s is surfel s's label distribution (const MatX*, raster.hpp:142)
struct MatX {
  int rows_ = 0, cols_ = 0;
  std::vector<double> data_;
  MatX() = default;
  MatX(int r, int c, double fill = 0.0) : rows_(r), cols_(c), data_(static_cast<size_t>(r) * c, fill) {}
  int rows() const { return rows_; }
  int cols() const { return cols_; }
  double& operator()(int r, int c) { return data_[static_cast<size_t>(c) * rows_ + r]; }
  double operator()(int r, int c) const { return data_[static_cast<size_t>(c) * rows_ + r]; }
  const double* data() const { return data_.data(); }
  double* data() { return data_.data(); }
};

struct Surfel {  // core_types.hpp:17-25
  Vec3 center{};
  Vec4 rotation{{1, 0, 0, 0}};
  Vec2 scales{{1, 1}};
  double opacity = 0.5;
  Vec3 color{};
  VecX f_sem;
  VecX f_ins;
};

struct Camera {  // core_types.hpp:36-53
  Mat3 r_cw = Mat3::Identity();
  Vec3 t_cw{};
  double fx = 1, fy = 1, cx = 0, cy = 0;
  int width = 0, height = 0;
  double near_clip = 0.01, far_clip = 100.0;

  static Camera from_c(const psm_camera& c) {
    Camera o;
    std::copy(c.r_cw, c.r_cw + 9, o.r_cw.m.begin());
    for (int i = 0; i < 3; ++i) o.t_cw[i] = c.t_cw[i];
    o.fx = c.fx; o.fy = c.fy; o.cx = c.cx; o.cy = c.cy;
    o.width = c.width; o.height = c.height;
    o.near_clip = c.near_clip; o.far_clip = c.far_clip;
    return o;
  }
  psm_camera to_c() const {
    psm_camera c{};
    std::copy(r_cw.m.begin(), r_cw.m.end(), c.r_cw);
    for (int i = 0; i < 3; ++i) c.t_cw[i] = t_cw[i];
    c.fx = fx; c.fy = fy; c.cx = cx; c.cy = cy;
    c.width = width; c.height = height;
    c.near_clip = near_clip; c.far_clip = far_clip;
    return c;
  }
  // Camera::make / look_at (core_types.cpp:18-60): throw std::invalid_argument on bad parameters
  static Camera make(const Mat3& r, const Vec3& t, double fx, double fy, double cx, double cy, int w, int h,
                     double near_clip, double far_clip) {
    psm_camera c{};
    if (psm_camera_make(r.m.data(), t.v.data(), fx, fy, cx, cy, w, h, near_clip, far_clip, &c) != PSM_OK)
      throw std::invalid_argument("camera: invalid parameters");
    return from_c(c);
  }
  static Camera look_at(const Vec3& eye, const Vec3& target, const Vec3& up, double fx, double fy, int w, int h,
                        double near_clip, double far_clip) {
    psm_camera c{};
    if (psm_camera_look_at(eye.v.data(), target.v.data(), up.v.data(), fx, fy, w, h, near_clip, far_clip, &c) != PSM_OK)
      throw std::invalid_argument("camera: invalid look_at");
    return from_c(c);
  }
};

struct InstanceQuery {  // core_types.hpp:76-84
  VecX feature;                 // C_ins entries
  Vec3 mean{};
  Mat3 cov = Mat3::Identity();  // SPD
  std::vector<int64_t> class_votes;
  int class_id = -1;
  int64_t assign_count = 0;
  bool alive = true;
};

struct AttentionWeights {  // core_types.hpp:89-100 (carried through checkpoints; not used by render)
  MatX w_q, w_k, w_v;  // C_ins x d
  int pos_enc_bands = 6;
  double pos_enc_base_freq = 0.5;
  uint64_t pos_enc_seed = 42;
};

struct SceneMap {  // core_types.hpp:102-111
  std::vector<Surfel> surfels;
  std::vector<std::string> vocabulary;
  std::vector<InstanceQuery> queries;
  AttentionWeights attn;
  int c_sem() const { return surfels.empty() ? 0 : static_cast<int>(surfels[0].f_sem.size()); }
  int c_ins() const { return surfels.empty() ? 0 : static_cast<int>(surfels[0].f_ins.size()); }
};

template <typename T>
struct Plane {  // image.hpp:11-43, HWC channel-fastest
  int width = 0, height = 0, channels = 0;
  std::vector<T> data;
  Plane() = default;
  Plane(int w, int h, int c, T fill = T{}) : width(w), height(h), channels(c), data(static_cast<size_t>(w) * h * c, fill) {}
  T& at(int x, int y, int c = 0) { return data[(static_cast<size_t>(y) * width + x) * channels + c]; }
  const T& at(int x, int y, int c = 0) const { return data[(static_cast<size_t>(y) * width + x) * channels + c]; }
  T* pixel(int x, int y) { return &data[(static_cast<size_t>(y) * width + x) * channels]; }
};
using Image = Plane<double>;
using IntPlane = Plane<int32_t>;

enum class Binning { Circle = PSM_BIN_CIRCLE, Aabb = PSM_BIN_AABB, Ellipse = PSM_BIN_ELLIPSE };
enum class Blending { Full = PSM_BLEND_FULL, TopK = PSM_BLEND_TOPK };

struct RasterConfig {  // raster.hpp:42-54
  int tile_size = 16;
  double chi2 = 9.0;
  double alpha_min = 1.0 / 255.0;
  double t_min = 1e-4;
  bool support_cutoff = true;
  Binning binning = Binning::Aabb;
  Blending blending = Blending::Full;
  int top_k = 16;
  Vec3 background{};
  bool render_depth_normal = true;
  int threads = 0;

  psm_raster_config to_c() const {
    psm_raster_config c{};
    c.tile_size = tile_size; c.chi2 = chi2; c.alpha_min = alpha_min; c.t_min = t_min;
    c.support_cutoff = support_cutoff; c.binning = static_cast<int>(binning);
    c.blending = static_cast<int>(blending); c.top_k = top_k;
    for (int i = 0; i < 3; ++i) c.background[i] = background[i];
    c.render_depth_normal = render_depth_normal; c.threads = threads;
    return c;
  }
};

struct RenderTargets {  // raster.hpp:56-66
  Image color, depth, normal, sem_feat, ins_dist;
  IntPlane ins_argmax;
  Image alpha_acc;
  IntPlane blend_count;
  uint64_t blended_total = 0;
};

struct ProjectedSurfel {  // raster.hpp:21-30
  int source = -1;
  Vec2 screen_center{};
  Mat2 sigma{};
  double sort_depth = 0;
  Mat3 h = Mat3{{{0, 0, 0, 0, 0, 0, 0, 0, 0}}};
  Mat3 h_inv = Mat3{{{0, 0, 0, 0, 0, 0, 0, 0, 0}}};
  Mat2 footprint_inv{};
  Vec3 normal_vis{{0, 0, 1}};

  static ProjectedSurfel from_c(const psm_projected& p) {
    ProjectedSurfel o;
    o.source = p.source;
    for (int i = 0; i < 2; ++i) o.screen_center[i] = p.screen_center[i];
    std::copy(p.sigma, p.sigma + 4, o.sigma.m.begin());
    o.sort_depth = p.sort_depth;
    std::copy(p.h, p.h + 9, o.h.m.begin());
    std::copy(p.h_inv, p.h_inv + 9, o.h_inv.m.begin());
    std::copy(p.footprint_inv, p.footprint_inv + 4, o.footprint_inv.m.begin());
    for (int i = 0; i < 3; ++i) o.normal_vis[i] = p.normal_vis[i];
    return o;
  }
  psm_projected to_c() const {
    psm_projected p{};
    p.source = source;
    for (int i = 0; i < 2; ++i) p.screen_center[i] = screen_center[i];
    std::copy(sigma.m.begin(), sigma.m.end(), p.sigma);
    p.sort_depth = sort_depth;
    std::copy(h.m.begin(), h.m.end(), p.h);
    std::copy(h_inv.m.begin(), h_inv.m.end(), p.h_inv);
    std::copy(footprint_inv.m.begin(), footprint_inv.m.end(), p.footprint_inv);
    for (int i = 0; i < 3; ++i) p.normal_vis[i] = normal_vis[i];
    return p;
  }
};

struct TileGrid {  // raster.hpp:32-40
  int tile_size = 16;
  int tiles_x = 0, tiles_y = 0;
  std::vector<std::vector<int>> tiles;  // projected indices, ascending (depth, source)
  uint64_t rn_total = 0;
  double rn_per_tile = 0;
  int tile_count() const { return tiles_x * tiles_y; }
};

struct PixelContribution {  // raster.hpp:69-74
  int proj;  // index into RenderCache::projected
  double alpha;
  double u, v;
};

struct RenderCache {  // raster.hpp:76-82, filled by render / render_into on the GPU (psm_render_cache)
  std::vector<ProjectedSurfel> projected;
  TileGrid grid;
  std::vector<std::vector<PixelContribution>> pixels;  // per pixel, blend order
  RasterConfig cfg;
  int width = 0, height = 0;
};

struct AlphaSample {  // raster.hpp:103-108
  double alpha = 0;
  double u = 0, v = 0;
  double w2 = 0;
  bool inside = false;
};

struct WeightKey {  // raster.hpp:120-124
  double weight;
  int proj;
  int index;
};

struct BenchRow {  // raster.hpp:150-160
  std::string name;
  Binning binning;
  Blending blending;
  double time_ms = 0, fps = 0;
  uint64_t rn_total = 0;
  double rn_per_tile = 0;
  uint64_t blended_total = 0;
  double blended_per_pixel = 0;
};
struct BenchReport {  // raster.hpp:162-167
  std::vector<BenchRow> rows;
  int repetitions = 0, width = 0, height = 0, surfel_count = 0;
};

namespace b200 {

// One context per device, created on first use (the reference keeps no globals; this
// is plumbing: a CUDA stream and grow-only scratch reused across calls).
inline psm_ctx* context(int device = 0) {
  struct Holder {
    psm_ctx* ctx = nullptr;
    ~Holder() { if (ctx) psm_destroy(ctx); }
  };
  static thread_local Holder h;
  if (!h.ctx) {
    if (psm_create(device, nullptr, &h.ctx) != PSM_OK) throw std::runtime_error("psimap::b200: no CUDA device");
  }
  return h.ctx;
}

inline void check(int st, psm_ctx* ctx) {
  if (st == PSM_OK) return;
  const std::string msg = ctx ? psm_last_error(ctx) : "psm error";
  if (st == PSM_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

// Flattens the scene and uploads it (the reference borrows the scene per call).
struct UploadedScene {
  psm_scene* sc = nullptr;
  psm_ctx* ctx = nullptr;
  ~UploadedScene() { if (sc) psm_scene_free(ctx, sc); }
};

inline std::unique_ptr<UploadedScene> upload(const SceneMap& scene, const MatX* labels, psm_ctx* ctx) {
  const int64_t n = static_cast<int64_t>(scene.surfels.size());
  const int c_sem = scene.c_sem();
  std::vector<double> geo(static_cast<size_t>(n) * 13), fs(static_cast<size_t>(n) * c_sem);
  for (int64_t i = 0; i < n; ++i) {
    const Surfel& s = scene.surfels[i];
    double* g = &geo[static_cast<size_t>(i) * 13];
    for (int k = 0; k < 3; ++k) g[k] = s.center[k];
    for (int k = 0; k < 4; ++k) g[3 + k] = s.rotation[k];
    g[7] = s.scales[0]; g[8] = s.scales[1]; g[9] = s.opacity;
    for (int k = 0; k < 3; ++k) g[10 + k] = s.color[k];
    for (int c = 0; c < c_sem; ++c) fs[static_cast<size_t>(i) * c_sem + c] = s.f_sem[c];
  }
  auto u = std::make_unique<UploadedScene>();
  u->ctx = ctx;
  const int n_q = labels ? labels->rows() : 0;
  check(psm_scene_upload(ctx, geo.data(), n, fs.data(), c_sem, labels ? labels->data() : nullptr, n_q, &u->sc), ctx);
  return u;
}

// Upload with f_ins and fp64 feature copies (PSM_SCENE_EXACT_FEATURES), for the panoptic layer.
inline std::unique_ptr<UploadedScene> upload_exact(const SceneMap& scene, psm_ctx* ctx) {
  const int64_t n = static_cast<int64_t>(scene.surfels.size());
  const int c_sem = scene.c_sem(), c_ins = scene.c_ins();
  std::vector<double> geo(static_cast<size_t>(n) * 13), fs(static_cast<size_t>(n) * c_sem),
      fi(static_cast<size_t>(n) * c_ins);
  for (int64_t i = 0; i < n; ++i) {
    const Surfel& s = scene.surfels[i];
    double* g = &geo[static_cast<size_t>(i) * 13];
    for (int k = 0; k < 3; ++k) g[k] = s.center[k];
    for (int k = 0; k < 4; ++k) g[3 + k] = s.rotation[k];
    g[7] = s.scales[0]; g[8] = s.scales[1]; g[9] = s.opacity;
    for (int k = 0; k < 3; ++k) g[10 + k] = s.color[k];
    for (int c = 0; c < c_sem; ++c) fs[static_cast<size_t>(i) * c_sem + c] = s.f_sem[c];
    for (int c = 0; c < c_ins; ++c) fi[static_cast<size_t>(i) * c_ins + c] = s.f_ins[c];
  }
  auto u = std::make_unique<UploadedScene>();
  u->ctx = ctx;
  psm_scene_desc d{geo.data(), n, fs.data(), c_sem, nullptr, 0, fi.data(), c_ins, PSM_SCENE_EXACT_FEATURES};
  check(psm_scene_create(ctx, &d, &u->sc), ctx);
  return u;
}

// Flat query arrays for psm_queries (features from `features` columns when given).
struct QueryArrays {
  std::vector<double> feat, mean, cov;
  std::vector<int32_t> alive, cls;
  psm_queries view(int c_ins) const {
    return psm_queries{static_cast<int32_t>(alive.size()), c_ins, feat.data(), mean.data(), cov.data(),
                       alive.data(), cls.data()};
  }
};
inline QueryArrays flatten(const std::vector<InstanceQuery>& qs, const MatX* features, int c_ins) {
  QueryArrays a;
  const size_t q = qs.size();
  a.feat.resize(q * c_ins);
  a.mean.resize(q * 3);
  a.cov.resize(q * 9);
  a.alive.resize(q);
  a.cls.resize(q);
  for (size_t i = 0; i < q; ++i) {
    for (int c = 0; c < c_ins; ++c) {
      const double v = features ? (*features)(c, static_cast<int>(i)) : qs[i].feature[c];
      a.feat[i * c_ins + c] = v;
    }
    if (!features && static_cast<int>(qs[i].feature.size()) != c_ins)
      throw std::invalid_argument("feature_similarity: dimension mismatch");  // panoptic.cpp:12-14
    for (int k = 0; k < 3; ++k) a.mean[i * 3 + k] = qs[i].mean[k];
    std::copy(qs[i].cov.m.begin(), qs[i].cov.m.end(), a.cov.begin() + i * 9);
    a.alive[i] = qs[i].alive ? 1 : 0;
    a.cls[i] = qs[i].class_id;
  }
  return a;
}

template <typename T>
inline void reset_plane(Plane<T>& p, int w, int h, int c) {  // raster.cpp:255-262
  if (p.width != w || p.height != h || p.channels != c) p = Plane<T>(w, h, c);
}

}  // namespace b200

// render_into (raster.cpp:273-511) on the GPU; outputs converted to the reference's double planes.
inline void render_into(RenderTargets& out, const SceneMap& scene, const MatX* labels, const Camera& cam,
                        const RasterConfig& cfg, RenderCache* cache = nullptr) {
  psm_ctx* ctx = b200::context();
  auto up = b200::upload(scene, labels, ctx);
  const int w = cam.width, h = cam.height, c_sem = scene.c_sem(), n_q = labels ? labels->rows() : 0;
  const size_t npx = static_cast<size_t>(w) * h;
  std::vector<float> col(npx * 3), dep(npx * 2), nrm(npx * 3), sem(npx * c_sem), ins(npx * n_q), alp(npx);
  std::vector<int32_t> arg(npx), cnt(npx);
  psm_targets tg{col.data(), dep.data(), nrm.data(), c_sem ? sem.data() : nullptr, n_q ? ins.data() : nullptr,
                 arg.data(), alp.data(), cnt.data(), 0};
  const psm_camera cc = cam.to_c();
  const psm_raster_config rc = cfg.to_c();
  psm_counters counters{};
  if (!cache) {
    b200::check(psm_render(ctx, up->sc, &cc, &rc, &tg, &counters), ctx);
  } else {  // RenderCache (raster.cpp:310-315,399-403,507-510): sizes first, then the arrays
    psm_render_cache_out co{};
    b200::check(psm_render_cache(ctx, up->sc, &cc, &rc, &tg, &counters, &co), ctx);
    const int tiles_x = (w + cfg.tile_size - 1) / cfg.tile_size, tiles_y = (h + cfg.tile_size - 1) / cfg.tile_size;
    std::vector<psm_projected> proj(static_cast<size_t>(co.n_projected));
    std::vector<int32_t> counts(static_cast<size_t>(tiles_x) * tiles_y), lists(static_cast<size_t>(co.n_tile_entries));
    std::vector<int64_t> offs(npx + 1);
    std::vector<psm_contribution> con(static_cast<size_t>(co.n_contribs));
    co.projected = proj.data(); co.projected_cap = co.n_projected;
    co.tile_counts = counts.data(); co.tile_lists = lists.data(); co.tile_lists_cap = co.n_tile_entries;
    co.pixel_offsets = offs.data(); co.contribs = con.data(); co.contribs_cap = co.n_contribs;
    b200::check(psm_render_cache(ctx, up->sc, &cc, &rc, &tg, &counters, &co), ctx);
    cache->cfg = cfg;
    cache->width = w;
    cache->height = h;
    cache->projected.clear();
    for (const psm_projected& p : proj) cache->projected.push_back(ProjectedSurfel::from_c(p));
    cache->grid = TileGrid{};
    cache->grid.tile_size = cfg.tile_size;
    cache->grid.tiles_x = tiles_x;
    cache->grid.tiles_y = tiles_y;
    cache->grid.rn_total = counters.rn_total;
    cache->grid.rn_per_tile = counters.rn_per_tile;
    cache->grid.tiles.assign(counts.size(), {});
    size_t at = 0;
    for (size_t t = 0; t < counts.size(); ++t)
      for (int32_t k = 0; k < counts[t]; ++k) cache->grid.tiles[t].push_back(lists[at++]);
    cache->pixels.assign(npx, {});
    for (size_t px = 0; px < npx; ++px)
      for (int64_t e = offs[px]; e < offs[px + 1]; ++e)
        cache->pixels[px].push_back({con[e].proj, con[e].alpha, con[e].u, con[e].v});
  }
  b200::reset_plane(out.color, w, h, 3);
  b200::reset_plane(out.depth, w, h, 2);
  b200::reset_plane(out.normal, w, h, 3);
  b200::reset_plane(out.sem_feat, w, h, c_sem);
  b200::reset_plane(out.ins_dist, w, h, n_q);
  b200::reset_plane(out.ins_argmax, w, h, 1);
  b200::reset_plane(out.alpha_acc, w, h, 1);
  b200::reset_plane(out.blend_count, w, h, 1);
  std::copy(col.begin(), col.end(), out.color.data.begin());
  std::copy(dep.begin(), dep.end(), out.depth.data.begin());
  std::copy(nrm.begin(), nrm.end(), out.normal.data.begin());
  std::copy(sem.begin(), sem.end(), out.sem_feat.data.begin());
  std::copy(ins.begin(), ins.end(), out.ins_dist.data.begin());
  std::copy(arg.begin(), arg.end(), out.ins_argmax.data.begin());
  std::copy(alp.begin(), alp.end(), out.alpha_acc.data.begin());
  std::copy(cnt.begin(), cnt.end(), out.blend_count.data.begin());
  out.blended_total = counters.blended_total;
}

inline RenderTargets render(const SceneMap& scene, const MatX* labels, const Camera& cam, const RasterConfig& cfg,
                            RenderCache* cache = nullptr) {
  RenderTargets out;
  render_into(out, scene, labels, cam, cfg, cache);
  return out;
}

// ---- stage functions (raster.hpp:87-126), device-backed (include/psm.h "Stage entry points")

// project_surfel (raster.cpp:94-142): nullopt when culled; throws std::invalid_argument on a
// degenerate quaternion of a surfel inside the depth range.
inline std::optional<ProjectedSurfel> project_surfel(const Surfel& s, const Camera& cam, const RasterConfig& cfg) {
  psm_ctx* ctx = b200::context();
  double g[13];
  for (int k = 0; k < 3; ++k) g[k] = s.center[k];
  for (int k = 0; k < 4; ++k) g[3 + k] = s.rotation[k];
  g[7] = s.scales[0]; g[8] = s.scales[1]; g[9] = s.opacity;
  for (int k = 0; k < 3; ++k) g[10 + k] = s.color[k];
  const psm_camera cc = cam.to_c();
  const psm_raster_config rc = cfg.to_c();
  psm_projected p{};
  int32_t status = 0;
  b200::check(psm_project_surfels(ctx, g, 1, &cc, &rc, &p, &status, nullptr), ctx);
  if (!status) return std::nullopt;
  return ProjectedSurfel::from_c(p);
}

namespace b200 {
inline TileGrid bin(const std::vector<ProjectedSurfel>& projected, const Camera& cam, const RasterConfig& cfg,
                    int binning, double chi2) {
  psm_ctx* ctx = context();
  std::vector<psm_projected> pc;
  pc.reserve(projected.size());
  for (const auto& p : projected) pc.push_back(p.to_c());
  TileGrid g;
  g.tile_size = cfg.tile_size;
  g.tiles_x = (cam.width + cfg.tile_size - 1) / cfg.tile_size;
  g.tiles_y = (cam.height + cfg.tile_size - 1) / cfg.tile_size;
  std::vector<int32_t> counts(static_cast<size_t>(g.tiles_x) * g.tiles_y);
  const psm_camera cc = cam.to_c();
  const psm_raster_config rc = cfg.to_c();
  psm_counters c{};
  const int64_t n = static_cast<int64_t>(pc.size());
  check(psm_bin_projected(ctx, pc.data(), n, &cc, &rc, binning, chi2, counts.data(), nullptr, 0, &c), ctx);
  std::vector<int32_t> lists(static_cast<size_t>(c.rn_total));
  if (c.rn_total)
    check(psm_bin_projected(ctx, pc.data(), n, &cc, &rc, binning, chi2, counts.data(), lists.data(),
                            static_cast<int64_t>(c.rn_total), &c), ctx);
  g.tiles.assign(counts.size(), {});
  size_t at = 0;
  for (size_t t = 0; t < counts.size(); ++t)
    for (int32_t k = 0; k < counts[t]; ++k) g.tiles[t].push_back(lists[at++]);
  g.rn_total = c.rn_total;
  g.rn_per_tile = c.rn_per_tile;
  return g;
}
}  // namespace b200

// bin_circle / bin_aabb (raster.cpp:51-90,144-152)
inline TileGrid bin_circle(const std::vector<ProjectedSurfel>& projected, const Camera& cam, const RasterConfig& cfg) {
  return b200::bin(projected, cam, cfg, PSM_BIN_CIRCLE, cfg.chi2);
}
inline TileGrid bin_aabb(const std::vector<ProjectedSurfel>& projected, const Camera& cam, const RasterConfig& cfg,
                         double chi2) {
  return b200::bin(projected, cam, cfg, PSM_BIN_AABB, chi2);
}

// sample_surfel_alpha / evaluate_alpha (raster.cpp:154-177)
inline AlphaSample sample_surfel_alpha(const ProjectedSurfel& proj, const Camera& cam, double px, double py,
                                       const RasterConfig& cfg) {
  psm_ctx* ctx = b200::context();
  const psm_projected p = proj.to_c();
  const double op = 0.0;
  const int32_t idx = 0;
  const psm_camera cc = cam.to_c();
  const psm_raster_config rc = cfg.to_c();
  psm_alpha_sample o{};
  b200::check(psm_sample_alpha(ctx, &p, &op, 1, &idx, &px, &py, 1, &cc, &rc, &o), ctx);
  AlphaSample a;
  a.u = o.u; a.v = o.v; a.w2 = o.w2; a.inside = o.inside != 0;  // .alpha stays 0, as the reference leaves it
  return a;
}
inline double evaluate_alpha(const ProjectedSurfel& proj, const Surfel& s, const Camera& cam, double px, double py,
                             const RasterConfig& cfg) {
  psm_ctx* ctx = b200::context();
  const psm_projected p = proj.to_c();
  const double op = s.opacity;
  const int32_t idx = 0;
  const psm_camera cc = cam.to_c();
  const psm_raster_config rc = cfg.to_c();
  psm_alpha_sample o{};
  b200::check(psm_sample_alpha(ctx, &p, &op, 1, &idx, &px, &py, 1, &cc, &rc, &o), ctx);
  return o.alpha;
}

// topk_select (raster.cpp:225-251); best_scratch receives the winners in (weight desc, proj asc) order
inline void topk_select(const WeightKey* keys, int m, int k, std::vector<WeightKey>& best_scratch,
                        std::vector<char>& selected) {
  psm_ctx* ctx = b200::context();
  std::vector<double> w(m);
  std::vector<int32_t> pj(m);
  for (int i = 0; i < m; ++i) {
    w[i] = keys[i].weight;
    pj[i] = keys[i].proj;
  }
  const int64_t offs[2] = {0, m};
  std::vector<int8_t> sel(m > 0 ? m : 1);
  b200::check(psm_topk_select(ctx, w.data(), pj.data(), offs, 1, k, sel.data()), ctx);
  selected.assign(m, 0);
  best_scratch.clear();
  for (int i = 0; i < m; ++i)
    if (sel[i]) {
      selected[i] = 1;
      best_scratch.push_back(keys[i]);
    }
  std::sort(best_scratch.begin(), best_scratch.end(), [](const WeightKey& a, const WeightKey& b) {
    return a.weight != b.weight ? a.weight > b.weight : a.proj < b.proj;
  });
}

// bench_render (raster.cpp:513-573): the 4-row grid; the scene is uploaded once and
// each row times `repetitions` whole renders (device clock, min), counters from the frame.
inline BenchReport bench_render(const SceneMap& scene, const MatX* labels, const Camera& cam, int repetitions,
                                const RasterConfig& base_cfg) {
  psm_ctx* ctx = b200::context();
  auto up = b200::upload(scene, labels, ctx);
  BenchReport report;
  report.repetitions = repetitions;
  report.width = cam.width;
  report.height = cam.height;
  report.surfel_count = static_cast<int>(scene.surfels.size());
  const std::array<std::pair<const char*, std::pair<Binning, Blending>>, 4> rows = {{
      {"baseline", {Binning::Circle, Blending::Full}},
      {"precise_tile", {Binning::Aabb, Blending::Full}},
      {"topk", {Binning::Circle, Blending::TopK}},
      {"full_method", {Binning::Aabb, Blending::TopK}},
  }};
  const psm_camera cc = cam.to_c();
  psm_set_profiling(ctx, 1);
  psm_targets tg{};  // planes stay in device scratch
  tg.on_device = 1;
  for (const auto& row : rows) {
    RasterConfig cfg = base_cfg;
    cfg.binning = row.second.first;
    cfg.blending = row.second.second;
    const psm_raster_config rc = cfg.to_c();
    psm_counters counters{};
    b200::check(psm_render(ctx, up->sc, &cc, &rc, &tg, &counters), ctx);  // warm-up
    double best = 1e300;
    for (int r = 0; r < std::max(repetitions, 1); ++r) {
      b200::check(psm_render(ctx, up->sc, &cc, &rc, &tg, &counters), ctx);
      psm_stage_times t{};
      psm_get_stage_times(ctx, &t);
      best = std::min(best, static_cast<double>(t.total));
    }
    BenchRow br;
    br.name = row.first;
    br.binning = cfg.binning;
    br.blending = cfg.blending;
    br.time_ms = best;
    br.fps = best > 0 ? 1000.0 / best : 0;
    br.rn_total = counters.rn_total;
    br.rn_per_tile = counters.rn_per_tile;
    br.blended_total = counters.blended_total;
    br.blended_per_pixel = static_cast<double>(counters.blended_total) / (static_cast<double>(cam.width) * cam.height);
    report.rows.push_back(br);
  }
  psm_set_profiling(ctx, 0);
  return report;
}

struct StreetSpec {  // synthetic.hpp (make_street_scene parameters)
  int n_surfels = 12000;
  uint64_t seed = 7;
  double min_aspect = 5.0;
  int image_w = 256, image_h = 192;
  int c_sem = 32;
  int n_instances = 256;
  double scale_mult = 1.0;  // extension: s1 multiplier (1 = the reference's scales)
};
struct StreetScene {
  SceneMap scene;
  MatX labels;  // n_instances x N near one-hot
  Camera camera;
};

// make_street_scene (synthetic.cpp:236-312), generated by libpsm's host code.
inline StreetScene make_street_scene(const StreetSpec& spec) {
  psm_street_spec cs{spec.n_surfels, spec.seed, spec.min_aspect, spec.image_w, spec.image_h, spec.c_sem,
                     spec.n_instances, spec.scale_mult};
  int64_t n = 0;
  psm_camera cam{};
  if (psm_make_street_scene(&cs, &n, nullptr, nullptr, nullptr, &cam) != PSM_OK)
    throw std::invalid_argument("make_street_scene: bad spec");
  std::vector<double> geo(static_cast<size_t>(n) * 13), fs(static_cast<size_t>(n) * spec.c_sem),
      fi(static_cast<size_t>(n) * 8);
  StreetScene out;
  out.labels = MatX(spec.n_instances, static_cast<int>(n));
  b200::check(psm_make_street_scene(&cs, &n, geo.data(), fs.data(), out.labels.data(), &cam), nullptr);
  b200::check(psm_make_street_scene_ins(&cs, &n, fi.data()), nullptr);
  out.camera = Camera::from_c(cam);
  out.scene.vocabulary = {"street"};
  out.scene.surfels.resize(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    Surfel& s = out.scene.surfels[static_cast<size_t>(i)];
    const double* g = &geo[static_cast<size_t>(i) * 13];
    for (int k = 0; k < 3; ++k) s.center[k] = g[k];
    for (int k = 0; k < 4; ++k) s.rotation[k] = g[3 + k];
    s.scales = vec2(g[7], g[8]);
    s.opacity = g[9];
    for (int k = 0; k < 3; ++k) s.color[k] = g[10 + k];
    s.f_sem.assign(fs.begin() + i * spec.c_sem, fs.begin() + (i + 1) * spec.c_sem);
    s.f_ins.assign(fi.begin() + i * 8, fi.begin() + (i + 1) * 8);
  }
  return out;
}

struct LabelAssignment {  // panoptic.hpp:28-31
  MatX dist;                // N_queries x N_surfels, columns sum to 1
  std::vector<int> argmax;  // ties to the lowest query index
};

// assign_labels (panoptic.cpp:36-91) on the GPU.
inline LabelAssignment assign_labels(const std::vector<InstanceQuery>& queries, const MatX* features,
                                     const SceneMap& scene) {
  psm_ctx* ctx = b200::context();
  auto up = b200::upload_exact(scene, ctx);
  const int n_q = static_cast<int>(queries.size()), n_s = static_cast<int>(scene.surfels.size());
  const b200::QueryArrays qa = b200::flatten(queries, features, scene.c_ins());
  const psm_queries qv = qa.view(scene.c_ins());
  LabelAssignment out;
  out.dist = MatX(n_q, n_s);
  std::vector<int32_t> arg(static_cast<size_t>(n_s), -1);
  b200::check(psm_assign_labels(ctx, up->sc, &qv, out.dist.data(), arg.data()), ctx);
  out.argmax.assign(arg.begin(), arg.end());
  return out;
}

struct PanopticRender {  // metrics.hpp:70-78
  IntPlane ids;
  IntPlane classes;
  IntPlane sem_classes;
};

// render_panoptic (metrics.cpp:339-369): assign_labels over scene.queries, render with
// the label distribution, and the alpha >= 0.5 id / class / semantic-class epilogue,
// fused into the GPU blend (bit-identical argmaxes).
inline PanopticRender render_panoptic(const SceneMap& scene, const Camera& cam, const RasterConfig& cfg) {
  psm_ctx* ctx = b200::context();
  auto up = b200::upload_exact(scene, ctx);
  const b200::QueryArrays qa = b200::flatten(scene.queries, nullptr, scene.c_ins());
  if (!scene.queries.empty()) {
    const psm_queries qv = qa.view(scene.c_ins());
    b200::check(psm_assign_labels(ctx, up->sc, &qv, nullptr, nullptr), ctx);
  }
  PanopticRender out;
  out.ids = IntPlane(cam.width, cam.height, 1, -1);
  out.classes = IntPlane(cam.width, cam.height, 1, -1);
  out.sem_classes = IntPlane(cam.width, cam.height, 1, -1);
  psm_panoptic_targets pt{out.ids.data.data(), out.classes.data.data(), out.sem_classes.data.data(), 0};
  const psm_camera cc = cam.to_c();
  const psm_raster_config rc = cfg.to_c();
  psm_counters counters{};
  b200::check(psm_render_panoptic(ctx, up->sc, &cc, &rc, qa.cls.data(), static_cast<int32_t>(qa.cls.size()), &pt,
                                  &counters),
              ctx);
  return out;
}

}  // namespace psimap

#endif  // PSIMAP_B200_HPP
