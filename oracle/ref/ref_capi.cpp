// ref_capi.cpp — C-ABI over the REFERENCE'S OWN render path, compiled unchanged from
// /root/reference/proj/src/{raster,math_util,core_types,synthetic,panoptic,metrics,losses,sogmm,pipeline}.cpp
// against the minimal Eigen stand-in in oracle/eigen_min (see its headers for the numerics
// they keep).
// TEST INFRASTRUCTURE ONLY: tests/ use it to pin oracle/oracle.cpp (and, through it,
// the GPU path) to the reference's actual code; bench.py --impl reference times it as
// the reference CPU renderer. The product library never links it.
//
// Build: oracle/ref/Makefile -> oracle/_ref/libpsimap_ref.so (git-ignored; travels to
// the GPU box with the gpurun snapshot). Nothing from the reference tree is copied: the
// sources are compiled where they lie.
#include <cstring>
#include <stdexcept>
#include <vector>

#include "psimap/core_types.hpp"
#include "psimap/losses.hpp"
#include "psimap/metrics.hpp"
#include "psimap/panoptic.hpp"
#include "psimap/pipeline.hpp"
#include "psimap/raster.hpp"
#include "psimap/synthetic.hpp"

#include "../../include/psm.h"

using namespace psimap;

namespace {

Camera to_cam(const psm_camera* c) {
  Camera cam;
  for (int col = 0; col < 3; ++col)
    for (int row = 0; row < 3; ++row) cam.r_cw(row, col) = c->r_cw[col * 3 + row];
  cam.t_cw = Vec3(c->t_cw[0], c->t_cw[1], c->t_cw[2]);
  cam.fx = c->fx; cam.fy = c->fy; cam.cx = c->cx; cam.cy = c->cy;
  cam.width = c->width; cam.height = c->height;
  cam.near_clip = c->near_clip; cam.far_clip = c->far_clip;
  return cam;
}

void from_cam(const Camera& cam, psm_camera* c) {
  for (int col = 0; col < 3; ++col)
    for (int row = 0; row < 3; ++row) c->r_cw[col * 3 + row] = cam.r_cw(row, col);
  for (int i = 0; i < 3; ++i) c->t_cw[i] = cam.t_cw[i];
  c->fx = cam.fx; c->fy = cam.fy; c->cx = cam.cx; c->cy = cam.cy;
  c->width = cam.width; c->height = cam.height;
  c->near_clip = cam.near_clip; c->far_clip = cam.far_clip;
}

// psm_raster_config -> RasterConfig. ELLIPSE is not a reference mode; it renders as
// AABB (identical planes whenever support_cutoff is on).
RasterConfig to_cfg(const psm_raster_config* k) {
  RasterConfig cfg;
  cfg.tile_size = k->tile_size;
  cfg.chi2 = k->chi2;
  cfg.alpha_min = k->alpha_min;
  cfg.t_min = k->t_min;
  cfg.support_cutoff = k->support_cutoff != 0;
  cfg.binning = k->binning == PSM_BIN_CIRCLE ? Binning::Circle : Binning::Aabb;
  cfg.blending = k->blending == PSM_BLEND_TOPK ? Blending::TopK : Blending::Full;
  cfg.top_k = k->top_k;
  cfg.background = Vec3(k->background[0], k->background[1], k->background[2]);
  cfg.render_depth_normal = k->render_depth_normal != 0;
  cfg.threads = k->threads;
  return cfg;
}

Surfel to_surfel(const double* s) {
  Surfel sf;
  sf.center = Vec3(s[0], s[1], s[2]);
  sf.rotation = Vec4(s[3], s[4], s[5], s[6]);
  sf.scales = Vec2(s[7], s[8]);
  sf.opacity = s[9];
  sf.color = Vec3(s[10], s[11], s[12]);
  return sf;
}

struct RefScene {
  SceneMap scene;
  MatX labels;
  bool has_labels = false;
  RenderTargets targets;  // persistent framebuffers (render_into reuse, raster.cpp:255-262)
};

template <typename T>
void put(T* dst, const Plane<T>& p) {
  if (dst && !p.data.empty()) std::memcpy(dst, p.data.data(), p.data.size() * sizeof(T));
}

}  // namespace

extern "C" {

// make_street_scene (synthetic.cpp:236-312) as the reference generates it. spec->scale_mult
// is ignored (the reference has no such knob; callers compare verbatim scenes). Two-phase:
// NULL outputs return n only. labels: n x n_instances per-surfel rows; f_ins: n x 8.
int ref_make_street_scene(const psm_street_spec* spec, int64_t* n_out, double* surfels13, double* f_sem,
                          double* labels, double* f_ins, psm_camera* cam) {
  StreetSpec s;
  s.n_surfels = spec->n_surfels;
  s.seed = spec->seed;
  s.min_aspect = spec->min_aspect;
  s.image_w = spec->image_w;
  s.image_h = spec->image_h;
  s.c_sem = spec->c_sem;
  s.n_instances = spec->n_instances;
  try {
    const StreetScene st = make_street_scene(s);
    const int64_t n = static_cast<int64_t>(st.scene.surfels.size());
    *n_out = n;
    if (cam) from_cam(st.camera, cam);
    for (int64_t i = 0; i < n; ++i) {
      const Surfel& sf = st.scene.surfels[i];
      if (surfels13) {
        double* o = surfels13 + 13 * i;
        for (int k = 0; k < 3; ++k) o[k] = sf.center[k];
        for (int k = 0; k < 4; ++k) o[3 + k] = sf.rotation[k];
        o[7] = sf.scales[0]; o[8] = sf.scales[1];
        o[9] = sf.opacity;
        for (int k = 0; k < 3; ++k) o[10 + k] = sf.color[k];
      }
      if (f_sem)
        for (int c = 0; c < spec->c_sem; ++c) f_sem[i * spec->c_sem + c] = sf.f_sem[c];
      if (f_ins)
        for (int c = 0; c < sf.f_ins.size(); ++c) f_ins[i * sf.f_ins.size() + c] = sf.f_ins[c];
      if (labels)
        for (int q = 0; q < spec->n_instances; ++q) labels[i * spec->n_instances + q] = st.labels(q, i);
    }
  } catch (const std::invalid_argument&) {
    return PSM_EINVAL;
  }
  return PSM_OK;
}

int ref_camera_look_at(const double eye[3], const double target[3], const double up[3], double fx, double fy,
                       int32_t width, int32_t height, double near_clip, double far_clip, psm_camera* out) {
  try {
    from_cam(Camera::look_at(Vec3(eye[0], eye[1], eye[2]), Vec3(target[0], target[1], target[2]),
                             Vec3(up[0], up[1], up[2]), fx, fy, width, height, near_clip, far_clip),
             out);
  } catch (const std::invalid_argument&) {
    return PSM_EINVAL;
  }
  return PSM_OK;
}

// A SceneMap (and optional labels MatX, N_q x N column-major = per-surfel rows) built once.
void* ref_scene_create(const double* surfels13, int64_t n, const double* f_sem, int32_t c_sem,
                       const double* labels, int32_t n_q) {
  auto* r = new RefScene();
  r->scene.surfels.resize(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    Surfel& sf = r->scene.surfels[i];
    sf = to_surfel(surfels13 + 13 * i);
    sf.f_sem = VecX(c_sem);
    for (int c = 0; c < c_sem; ++c) sf.f_sem[c] = f_sem[i * c_sem + c];
  }
  if (labels && n_q > 0) {
    r->labels = MatX(n_q, n);
    std::memcpy(r->labels.data(), labels, sizeof(double) * n_q * n);
    r->has_labels = true;
  }
  return r;
}

void ref_scene_free(void* h) { delete static_cast<RefScene*>(h); }

// render_into (raster.cpp:273-511) into the scene's persistent targets.
int ref_render_into(void* h, const psm_camera* cam, const psm_raster_config* cfg, uint64_t* blended_total) {
  auto* r = static_cast<RefScene*>(h);
  try {
    render_into(r->targets, r->scene, r->has_labels ? &r->labels : nullptr, to_cam(cam), to_cfg(cfg));
  } catch (const std::invalid_argument&) {
    return PSM_EINVAL;
  }
  if (blended_total) *blended_total = r->targets.blended_total;
  return PSM_OK;
}

// The last render's fp64 / int32 planes (HWC), any pointer may be NULL.
void ref_targets_copy(void* h, double* color, double* depth, double* normal, double* sem_feat, double* ins_dist,
                      int32_t* ins_argmax, double* alpha_acc, int32_t* blend_count) {
  const RenderTargets& t = static_cast<RefScene*>(h)->targets;
  put(color, t.color); put(depth, t.depth); put(normal, t.normal); put(sem_feat, t.sem_feat);
  put(ins_dist, t.ins_dist); put(ins_argmax, t.ins_argmax); put(alpha_acc, t.alpha_acc);
  put(blend_count, t.blend_count);
}

// project_surfel over the scene + bin_circle / bin_aabb (raster.cpp:94-152). Outputs as
// oracle_bin: tile_counts[tiles], list_src[cap] (source ids in list order), counters.
int ref_bin(void* h, const psm_camera* pcam, const psm_raster_config* pcfg, int32_t binning, double chi2,
            int32_t* tile_counts, int32_t* list_src, int64_t cap, psm_counters* counters) {
  auto* r = static_cast<RefScene*>(h);
  const Camera cam = to_cam(pcam);
  const RasterConfig cfg = to_cfg(pcfg);
  std::vector<ProjectedSurfel> projected;
  try {
    for (size_t i = 0; i < r->scene.surfels.size(); ++i) {
      auto p = project_surfel(r->scene.surfels[i], cam, cfg);
      if (p.has_value()) {
        p->source = static_cast<int>(i);
        projected.push_back(*p);
      }
    }
  } catch (const std::invalid_argument&) {
    return PSM_EINVAL;
  }
  const TileGrid g = binning == PSM_BIN_CIRCLE ? bin_circle(projected, cam, cfg) : bin_aabb(projected, cam, cfg, chi2);
  int64_t at = 0, nonempty = 0;
  for (size_t t = 0; t < g.tiles.size(); ++t) {
    if (tile_counts) tile_counts[t] = static_cast<int32_t>(g.tiles[t].size());
    nonempty += !g.tiles[t].empty();
    for (int idx : g.tiles[t]) {
      if (list_src && at < cap) list_src[at] = projected[idx].source;
      ++at;
    }
  }
  if (counters) {
    counters->rn_total = g.rn_total;
    counters->rn_per_tile = g.rn_per_tile;
    counters->n_proj = static_cast<int64_t>(projected.size());
    counters->tiles_x = g.tiles_x;
    counters->tiles_y = g.tiles_y;
    counters->nonempty_tiles = nonempty;
    counters->blended_total = 0;
  }
  return PSM_OK;
}

// One ProjectedSurfel, flattened like oracle_projected (status 1 projected, 0 culled,
// -1 degenerate quaternion).
typedef struct ref_projected {
  int32_t status;
  double center[2];
  double sigma[4];
  double sort_depth;
  double h[9], h_inv[9];
  double finv[4];
  double normal_vis[3];
} ref_projected;

int ref_project_surfel(const double* s13, const psm_camera* cam, const psm_raster_config* cfg, ref_projected* out) {
  std::memset(out, 0, sizeof *out);
  try {
    auto p = project_surfel(to_surfel(s13), to_cam(cam), to_cfg(cfg));
    if (!p.has_value()) return out->status = 0;
    out->status = 1;
    out->center[0] = p->screen_center[0]; out->center[1] = p->screen_center[1];
    std::memcpy(out->sigma, p->sigma.data(), sizeof out->sigma);
    out->sort_depth = p->sort_depth;
    std::memcpy(out->h, p->h.data(), sizeof out->h);
    std::memcpy(out->h_inv, p->h_inv.data(), sizeof out->h_inv);
    std::memcpy(out->finv, p->footprint_inv.data(), sizeof out->finv);
    for (int i = 0; i < 3; ++i) out->normal_vis[i] = p->normal_vis[i];
  } catch (const std::invalid_argument&) {
    out->status = -1;
  }
  return out->status;
}

// sample_surfel_alpha + evaluate_alpha (raster.cpp:154-177) at pixel centre (px, py).
double ref_evaluate_alpha(const double* s13, const psm_camera* pcam, double px, double py,
                          const psm_raster_config* pcfg, double* u, double* v, double* w2, int32_t* inside) {
  const Surfel sf = to_surfel(s13);
  const Camera cam = to_cam(pcam);
  const RasterConfig cfg = to_cfg(pcfg);
  *inside = 0;
  auto p = project_surfel(sf, cam, cfg);
  if (!p.has_value()) return 0.0;
  const AlphaSample smp = sample_surfel_alpha(*p, cam, px, py, cfg);
  *u = smp.u; *v = smp.v; *w2 = smp.w2; *inside = smp.inside ? 1 : 0;
  return evaluate_alpha(*p, sf, cam, px, py, cfg);
}

// topk_select (raster.cpp:225-251) over m (weight, proj) keys.
void ref_topk_select(const double* weights, const int32_t* proj, int32_t m, int32_t k, int8_t* selected) {
  std::vector<WeightKey> keys(m), best;
  for (int i = 0; i < m; ++i) keys[i] = {weights[i], proj[i], i};
  std::vector<char> sel;
  topk_select(keys.data(), m, k, best, sel);
  for (int i = 0; i < m; ++i) selected[i] = sel[i];
}

// bench_render (raster.cpp:513-573): 4 rows x (time_ms, fps, rn_total, rn_per_tile,
// blended_total, blended_per_pixel).
int ref_bench_render(void* h, const psm_camera* cam, int32_t reps, const psm_raster_config* cfg, double* rows6x4) {
  auto* r = static_cast<RefScene*>(h);
  try {
    const BenchReport rep = bench_render(r->scene, r->has_labels ? &r->labels : nullptr, to_cam(cam), reps, to_cfg(cfg));
    for (size_t i = 0; i < rep.rows.size(); ++i) {
      const BenchRow& b = rep.rows[i];
      double* o = rows6x4 + 6 * i;
      o[0] = b.time_ms; o[1] = b.fps; o[2] = static_cast<double>(b.rn_total); o[3] = b.rn_per_tile;
      o[4] = static_cast<double>(b.blended_total); o[5] = b.blended_per_pixel;
    }
  } catch (const std::invalid_argument&) {
    return PSM_EINVAL;
  }
  return PSM_OK;
}

// ---- panoptic rows (F1, F2)

namespace {
// SceneMap with f_sem, f_ins and the instance queries (feature, mean, cov column-major,
// alive, class id), as pack_queries / psm_queries lay them out.
SceneMap panoptic_scene(const double* surfels13, int64_t n, const double* f_sem, int32_t c_sem, const double* f_ins,
                        int32_t c_ins, int32_t n_queries, const double* q_feat, const double* q_mean,
                        const double* q_cov, const int32_t* q_alive, const int32_t* q_class) {
  SceneMap sc;
  sc.surfels.resize(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    Surfel& sf = sc.surfels[i];
    sf = to_surfel(surfels13 + 13 * i);
    sf.f_sem = VecX(c_sem);
    for (int c = 0; c < c_sem; ++c) sf.f_sem[c] = f_sem[i * c_sem + c];
    sf.f_ins = VecX(c_ins);
    for (int c = 0; c < c_ins; ++c) sf.f_ins[c] = f_ins[i * c_ins + c];
  }
  for (int q = 0; q < n_queries; ++q) {
    InstanceQuery iq;
    iq.feature = VecX(c_ins);
    for (int c = 0; c < c_ins; ++c) iq.feature[c] = q_feat[q * c_ins + c];
    iq.mean = Vec3(q_mean[3 * q], q_mean[3 * q + 1], q_mean[3 * q + 2]);
    for (int c = 0; c < 3; ++c)
      for (int r = 0; r < 3; ++r) iq.cov(r, c) = q_cov[9 * q + 3 * c + r];
    iq.alive = q_alive[q] != 0;
    iq.class_id = q_class ? q_class[q] : -1;
    sc.queries.push_back(iq);
  }
  return sc;
}
}  // namespace

// assign_labels (panoptic.cpp:36-91): dist_out n x n_queries (per-surfel rows), argmax_out n.
int ref_assign_labels(const double* surfels13, int64_t n, const double* f_ins, int32_t c_ins, int32_t n_queries,
                      const double* q_feat, const double* q_mean, const double* q_cov, const int32_t* q_alive,
                      double* dist_out, int32_t* argmax_out) {
  try {
    const SceneMap sc = panoptic_scene(surfels13, n, nullptr, 0, f_ins, c_ins, n_queries, q_feat, q_mean, q_cov,
                                       q_alive, nullptr);
    const LabelAssignment la = assign_labels(sc.queries, nullptr, sc);
    for (int64_t s = 0; s < n; ++s) {
      for (int q = 0; q < n_queries; ++q) dist_out[s * n_queries + q] = la.dist(q, s);
      argmax_out[s] = la.argmax[s];
    }
  } catch (const std::invalid_argument&) {
    return PSM_EINVAL;
  }
  return PSM_OK;
}

// render_panoptic (metrics.cpp:339-369): ids / classes / sem_classes planes (W*H int32).
int ref_render_panoptic(const double* surfels13, int64_t n, const double* f_sem, int32_t c_sem, const double* f_ins,
                        int32_t c_ins, int32_t n_queries, const double* q_feat, const double* q_mean,
                        const double* q_cov, const int32_t* q_alive, const int32_t* q_class, const psm_camera* cam,
                        const psm_raster_config* cfg, int32_t* ids, int32_t* classes, int32_t* sem_classes) {
  try {
    const SceneMap sc = panoptic_scene(surfels13, n, f_sem, c_sem, f_ins, c_ins, n_queries, q_feat, q_mean, q_cov,
                                       q_alive, q_class);
    const PanopticRender pr = render_panoptic(sc, to_cam(cam), to_cfg(cfg));
    put(ids, pr.ids);
    put(classes, pr.classes);
    put(sem_classes, pr.sem_classes);
  } catch (const std::invalid_argument&) {
    return PSM_EINVAL;
  }
  return PSM_OK;
}

// A panoptic SceneMap (f_sem, f_ins, queries) built once, for timing render_panoptic alone.
void* ref_panoptic_scene_create(const double* surfels13, int64_t n, const double* f_sem, int32_t c_sem,
                                const double* f_ins, int32_t c_ins, int32_t n_queries, const double* q_feat,
                                const double* q_mean, const double* q_cov, const int32_t* q_alive,
                                const int32_t* q_class) {
  return new SceneMap(panoptic_scene(surfels13, n, f_sem, c_sem, f_ins, c_ins, n_queries, q_feat, q_mean, q_cov,
                                     q_alive, q_class));
}
void ref_panoptic_scene_free(void* h) { delete static_cast<SceneMap*>(h); }

// render_panoptic (metrics.cpp:339-369) over a scene built by ref_panoptic_scene_create.
int ref_render_panoptic_h(void* h, const psm_camera* cam, const psm_raster_config* cfg, int32_t* ids,
                          int32_t* classes, int32_t* sem_classes) {
  try {
    const PanopticRender pr = render_panoptic(*static_cast<SceneMap*>(h), to_cam(cam), to_cfg(cfg));
    put(ids, pr.ids);
    put(classes, pr.classes);
    put(sem_classes, pr.sem_classes);
  } catch (const std::invalid_argument&) {
    return PSM_EINVAL;
  }
  return PSM_OK;
}

// ---- backward row (F4)

// project_surfel_backward (raster.cpp:179-203) of one surfel under its own projection:
// g_hinv row-major 3x3 in; d_center[3], d_rotation[4] (w, x, y, z), d_scales[2] out.
// Returns 1 (projected), 0 (culled, outputs untouched) or -1 (degenerate quaternion).
int ref_project_surfel_backward(const double* s13, const psm_camera* pcam, const psm_raster_config* pcfg,
                                const double* g_hinv, double* d_center, double* d_rotation, double* d_scales) {
  const Surfel sf = to_surfel(s13);
  const Camera cam = to_cam(pcam);
  try {
    auto p = project_surfel(sf, cam, to_cfg(pcfg));
    if (!p.has_value()) return 0;
    Mat3 g;
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) g(r, c) = g_hinv[3 * r + c];
    const SurfelGeomGrads gg = project_surfel_backward(sf, cam, *p, g);
    for (int k = 0; k < 3; ++k) d_center[k] = gg.d_center[k];
    for (int k = 0; k < 4; ++k) d_rotation[k] = gg.d_rotation[k];
    for (int k = 0; k < 2; ++k) d_scales[k] = gg.d_scales[k];
  } catch (const std::invalid_argument&) {
    return -1;
  }
  return 1;
}

// pipeline_backward (pipeline.cpp:253-600) of a scene without queries and without a SOGMM
// model, under the loss weights given (l_geo and l_ins have no terms here; pass l_iso = 0
// to leave only the render's gradients): the frame is (camera, rgb_gt W*H*3, sem_gt W*H or
// NULL). smooth != 0 uses PipelineConfig::smooth()'s raster settings (pipeline.cpp:56-64)
// instead of *pcfg. Outputs (each may be NULL): the scene gradients in psm_scene_grads
// layout, and the colour-plane gradient the reference fed its blending backward
// (loss_rgb_backward of the forward colour, pipeline.cpp:266).
int ref_pipeline_backward(void* h, const psm_camera* pcam, const psm_raster_config* pcfg, int32_t smooth,
                          const double* rgb_gt, const int32_t* sem_gt, double lambda_s, double l_rgb, double l_sem,
                          double l_iso, psm_scene_grads* out, double* g_color_plane) {
  auto* r = static_cast<RefScene*>(h);
  const Camera cam = to_cam(pcam);
  PipelineConfig cfg = smooth ? PipelineConfig::smooth() : PipelineConfig{};
  if (!smooth) cfg.raster = to_cfg(pcfg);
  cfg.raster.threads = pcfg->threads;
  cfg.weights.lambda_s = lambda_s;
  cfg.weights.l_rgb = l_rgb;
  cfg.weights.l_sem = l_sem;
  cfg.weights.l_iso = l_iso;
  FrameBundle frame;
  frame.camera = cam;
  frame.rgb = Image(cam.width, cam.height, 3);
  std::memcpy(frame.rgb.data.data(), rgb_gt, sizeof(double) * frame.rgb.data.size());
  if (sem_gt) {
    frame.sem_gt = IntPlane(cam.width, cam.height, 1);
    std::memcpy(frame.sem_gt.data.data(), sem_gt, sizeof(int32_t) * frame.sem_gt.data.size());
  }
  try {
    const BackwardResult bw = pipeline_backward(r->scene, nullptr, frame, cfg);
    const Gradients& g = bw.grads;
    const int64_t n = static_cast<int64_t>(r->scene.surfels.size());
    const int c_sem = r->scene.c_sem();
    for (int64_t s = 0; s < n; ++s) {
      if (out->opacity) out->opacity[s] = g.opacity[s];
      for (int k = 0; k < 3; ++k) {
        if (out->color) out->color[3 * s + k] = g.color[s][k];
        if (out->center) out->center[3 * s + k] = g.center[s][k];
      }
      for (int k = 0; k < 4 && out->rotation; ++k) out->rotation[4 * s + k] = g.rotation[s][k];
      for (int k = 0; k < 2 && out->scales; ++k) out->scales[2 * s + k] = g.scales[s][k];
      for (int c = 0; c < c_sem && out->f_sem; ++c) out->f_sem[s * c_sem + c] = g.f_sem(c, s);
    }
    if (g_color_plane) {
      const RenderTargets t = render(r->scene, nullptr, cam, cfg.raster);
      const Image gc = loss_rgb_backward(t.color, frame.rgb, lambda_s, l_rgb);
      std::memcpy(g_color_plane, gc.data.data(), sizeof(double) * gc.data.size());
    }
  } catch (const std::invalid_argument&) {
    return PSM_EINVAL;
  }
  return PSM_OK;
}

}  // extern "C"
