/* psm.h — C-ABI of the B200 surfel rasterizer (Ψ-Map render hot path).
 *
 * This is the drop-in boundary for `psimap::render` / `render_into` /
 * `bench_render` (reference: proj/include/psimap/raster.hpp:142-172,
 * proj/src/raster.cpp:266-573). No torch, no C++ types, no exceptions cross
 * it: plain pointers and sizes, int status codes. The C++ drop-in shim with the
 * reference's own names and types sits on top of it (include/psimap_b200.hpp).
 *
 * Buffer layouts are the reference's (proj/include/psimap/core_types.hpp:17-53,
 * proj/include/psimap/image.hpp:11-43):
 *   surfels13  N x 13 doubles, AoS, per surfel: center[3], rotation (w,x,y,z)[4],
 *              scales[2], opacity, color[3]   (Surfel, core_types.hpp:17-25)
 *   f_sem      N x C_sem doubles, row-major (Surfel::f_sem of every surfel;
 *              C_sem taken from surfel 0 like SceneMap::c_sem, core_types.hpp:108)
 *   labels     N x N_q doubles, surfel-major: the column-major Eigen MatX
 *              N_q x N passed as `const MatX* labels` (raster.hpp:142), so each
 *              surfel's distribution is contiguous (raster.cpp:337,352). May be NULL.
 *   planes     W x H x C, row-major, channel fastest: data[(y*W + x)*C + c]
 *              (Plane<T>, image.hpp:11-43). Written as fp32 / int32.
 *
 * Thread-safety: a context is used by one host thread at a time; distinct
 * contexts (one per device) are independent (reference render is reentrant,
 * raster.hpp:147).
 */
#ifndef PSM_H
#define PSM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define PSM_OK 0
#define PSM_EINVAL 1       /* bad argument, or a degenerate quaternion on a surfel that passed
                              the depth cull: mirrors std::invalid_argument thrown by
                              rotation_from_quat (proj/src/math_util.cpp:46-50) inside
                              project_surfel (proj/src/raster.cpp:99) */
#define PSM_ENOMEM 2
#define PSM_ECUDA 3
#define PSM_EUNSUPPORTED 4 /* valid for the reference, not implemented on the GPU path */

typedef struct psm_ctx psm_ctx;
typedef struct psm_scene psm_scene;

/* Camera (proj/include/psimap/core_types.hpp:36-53). r_cw is column-major like
 * Eigen::Matrix3d: r_cw[col*3 + row]. */
typedef struct psm_camera {
  double r_cw[9];
  double t_cw[3];
  double fx, fy, cx, cy;
  int32_t width, height;
  double near_clip, far_clip;
} psm_camera;

/* Binning (raster.hpp:17 adds Ellipse): CIRCLE = bin_circle (raster.cpp:144-147),
 * AABB = bin_aabb (raster.cpp:149-152), ELLIPSE = the exact support-ellipse vs
 * tile test (north-star "Precise Tile Intersection"; a subset of AABB's lists
 * that leaves every output plane unchanged; falls back to AABB when
 * support_cutoff == 0). */
enum { PSM_BIN_CIRCLE = 0, PSM_BIN_AABB = 1, PSM_BIN_ELLIPSE = 2 };
/* Blending (raster.hpp:18) */
enum { PSM_BLEND_FULL = 0, PSM_BLEND_TOPK = 1 };

/* RasterConfig (proj/include/psimap/raster.hpp:42-54). Defaults via
 * psm_default_config(). The GPU path requires tile_size == 16. */
typedef struct psm_raster_config {
  int32_t tile_size;
  double chi2;
  double alpha_min;
  double t_min;
  int32_t support_cutoff;
  int32_t binning;
  int32_t blending;
  int32_t top_k;            /* effective K = max(top_k, 1) (raster.cpp:318); GPU K <= 32 */
  double background[3];
  int32_t render_depth_normal;
  int32_t threads;          /* host worker count in the reference; ignored on the GPU */
} psm_raster_config;

/* RenderTargets (raster.hpp:56-66) as fp32/int32 planes. Any pointer may be
 * NULL to skip that plane's write-back (the plane is still computed on the
 * device). on_device = 1: pointers are device memory of the context's device
 * and the render is asynchronous on the context stream; 0: host memory, the
 * call copies back and synchronises. */
typedef struct psm_targets {
  float* color;        /* W*H*3 */
  float* depth;        /* W*H*2: expected depth, dominant-surfel depth */
  float* normal;       /* W*H*3 */
  float* sem_feat;     /* W*H*C_sem */
  float* ins_dist;     /* W*H*N_q */
  int32_t* ins_argmax; /* W*H, -1 where nothing accumulated */
  float* alpha_acc;    /* W*H */
  int32_t* blend_count;/* W*H */
  int32_t on_device;
} psm_targets;

/* Counters: TileGrid::rn_total / rn_per_tile (raster.hpp:36-37),
 * RenderTargets::blended_total (raster.hpp:65), plus the projected count. */
typedef struct psm_counters {
  uint64_t rn_total;
  double rn_per_tile;
  uint64_t blended_total;
  int64_t n_proj;
  int32_t tiles_x, tiles_y;
  int64_t nonempty_tiles;
} psm_counters;

/* Debug export for the parity suite (host pointers, caller-owned; any may be NULL).
 *   tile_keys   [cap_keys] sorted (tile << 32 | depth rank) keys, rank = position of the
 *               surfel in the (sort_depth, source) order of all projected surfels
 *   tile_vals   [cap_keys] source surfel index of each key (the tile lists of
 *               TileGrid::tiles, raster.hpp:35, as scene indices)
 *   tile_ranges [2 * tiles] [start, end) of each tile in tile_keys
 *   depth_order [cap_proj]  source index at each depth rank ((sort_depth, source)
 *               order of raster.cpp:78-83)
 *   topk_src    [W*H*K] the set of selected source indices per pixel (ordered by
 *               weight, -1 padded) (topk_select, raster.cpp:225-251 + compaction
 *               438-454); written when blending == TOPK. */
typedef struct psm_debug {
  uint64_t* tile_keys;
  int32_t* tile_vals;
  int64_t cap_keys;
  int32_t* tile_ranges;
  int32_t* depth_order;
  int64_t cap_proj;
  int32_t* topk_src;
} psm_debug;

/* Stage timings of the last synchronised render when profiling is on (CUDA events
 * on the context stream), milliseconds. Profiling does not make a device-target
 * render synchronous: the times are read when the frame is synchronised (psm_sync,
 * or a render that returns counters or host planes). */
typedef struct psm_stage_times {
  float preprocess;   /* K1: project_surfel, hot records, box, per-tile bucket sizes (raster.cpp:94-142,321-353,59-74) */
  float tile_scan;    /* K3: bucket offsets = per-tile ranges, RN-Total (raster.cpp:84-88) */
  float emit;         /* K4: (tile, surfel) pairs into their buckets (raster.cpp:69-73) */
  float tile_sort;    /* K5: per-tile sort by (sort_depth, source) (raster.cpp:77-83) */
  float blend;        /* K7: per-pixel compositing + Top-K + features (raster.cpp:355-506) */
  float total;
} psm_stage_times;

void psm_default_config(psm_raster_config* cfg);

/* Context: one per device; owns a stream (or borrows `stream` if non-NULL, a
 * cudaStream_t) and grow-only scratch arenas reused across frames (the
 * render_into buffer-reuse contract, raster.cpp:255-262). */
int psm_create(int device, void* stream, psm_ctx** out);
int psm_destroy(psm_ctx* ctx);
const char* psm_last_error(const psm_ctx* ctx);
int psm_set_profiling(psm_ctx* ctx, int enabled);
int psm_get_stage_times(const psm_ctx* ctx, psm_stage_times* out);
int psm_sync(psm_ctx* ctx);

/* Upload a scene once (the SceneMap + labels the reference borrows by const&
 * per call, raster.hpp:142-148). Geometry stays fp64 on the device for
 * bit-exact decisions; features and labels are stored fp32. */
int psm_scene_upload(psm_ctx* ctx, const double* surfels13, int64_t n, const double* f_sem,
                     int32_t c_sem, const double* labels, int32_t n_q, psm_scene** out);
/* psm_scene_free first settles ctx's pending asynchronous frames (psm_sync semantics), which
 * may still read the scene; frames pending on other contexts must be synchronised by the caller.
 * psm_assign_labels likewise settles ctx's pending frames before it rewrites the labels. */
int psm_scene_free(psm_ctx* ctx, psm_scene* scene);
int psm_scene_info(const psm_scene* scene, int64_t* n, int32_t* c_sem, int32_t* n_q);

/* render_into (raster.cpp:273-511). counters may be NULL. With on_device
 * targets and counters == NULL the call is asynchronous: psm_sync waits for every
 * asynchronous frame since the last synchronisation, checks each one's counters and
 * re-renders, in order, from the first that outgrew the context's buffers. */
int psm_render(psm_ctx* ctx, const psm_scene* scene, const psm_camera* cam,
               const psm_raster_config* cfg, const psm_targets* targets, psm_counters* counters);

/* Same render plus the debug export of sorted keys, tile ranges, depth order and Top-K ids. */
int psm_render_debug(psm_ctx* ctx, const psm_scene* scene, const psm_camera* cam,
                     const psm_raster_config* cfg, const psm_targets* targets,
                     psm_counters* counters, psm_debug* debug);

/* n_views independent renders (one per camera) into n_views target sets;
 * views share the scene upload. counters may be NULL or an array of n_views.
 * With device targets and counters == NULL the batch is asynchronous and pipelined:
 * views alternate between the context and an internal second context on a second
 * stream (one view's front end overlaps the other's blend); later work on the
 * context's stream is ordered after every view, and psm_sync validates them all
 * (psm_last_counters then holds the last view's counters). Views of different
 * parity (rendered by different contexts) must not share target planes. */
int psm_render_batch(psm_ctx* ctx, const psm_scene* scene, const psm_camera* cams, int32_t n_views,
                     const psm_raster_config* cfg, const psm_targets* targets,
                     psm_counters* counters);

/* Counters of the most recent render, valid after psm_sync. */
int psm_last_counters(const psm_ctx* ctx, psm_counters* out);

/* ---- Panoptic layer ----------------------------
 * A scene created with PSM_SCENE_EXACT_FEATURES also keeps fp64 copies of its
 * features and labels on the device, so psm_render_panoptic reproduces the
 * reference's fp64 feature/label sums (and hence its argmaxes) bit for bit. */
#define PSM_SCENE_EXACT_FEATURES 1

typedef struct psm_scene_desc {
  const double* surfels13; /* N x 13 (Surfel: centre 3, quaternion w,x,y,z 4, scales 2, opacity, colour 3) */
  int64_t n;
  const double* f_sem;     /* N x C_sem row-major, may be NULL when c_sem == 0 */
  int32_t c_sem;
  const double* labels;    /* per-surfel N_q contiguous (MatX N_q x N column-major), may be NULL */
  int32_t n_q;
  const double* f_ins;     /* N x C_ins row-major (Surfel::f_ins; psm_assign_labels), may be NULL */
  int32_t c_ins;
  int32_t flags;           /* PSM_SCENE_EXACT_FEATURES */
} psm_scene_desc;
int psm_scene_create(psm_ctx* ctx, const psm_scene_desc* desc, psm_scene** out);

/* Instance queries (InstanceQuery, core_types.hpp:76-84). `feature` holds the
 * features assign_labels uses: InstanceQuery::feature, or the columns of its
 * optional `features` matrix (panoptic.hpp:37). */
typedef struct psm_queries {
  int32_t n;
  int32_t c_ins;
  const double* feature;   /* n x c_ins */
  const double* mean;      /* n x 3 */
  const double* cov;       /* n x 9, column-major */
  const int32_t* alive;    /* n */
  const int32_t* class_id; /* n (used by psm_render_panoptic callers; may be NULL here) */
} psm_queries;

/* assign_labels (proj/src/panoptic.cpp:36-91) on the device. The scene's label
 * channels become the N_q = queries->n column distribution (dead queries 0).
 * dist_out (host, N x n, per-surfel contiguous) and argmax_out (host, N; -1 when
 * no query is alive) may be NULL. The scene must have f_ins with c_ins ==
 * queries->c_ins. Synchronous. */
int psm_assign_labels(psm_ctx* ctx, psm_scene* scene, const psm_queries* queries, double* dist_out,
                      int32_t* argmax_out);

/* PanopticRender (metrics.hpp:70-78): int32 W*H planes, -1 = void. */
typedef struct psm_panoptic_targets {
  int32_t* ids;         /* label argmax where alpha_acc >= 0.5 */
  int32_t* classes;     /* query_class[id] */
  int32_t* sem_classes; /* first argmax of the semantic feature plane */
  int32_t on_device;
} psm_panoptic_targets;

/* render_panoptic (proj/src/metrics.cpp:339-369) over a scene whose labels are
 * assigned: the blend accumulates features and labels in fp64 in blend order and
 * writes the three planes directly (no feature planes are materialised).
 * query_class: n_query_class class ids (InstanceQuery::class_id). Needs a scene
 * created with PSM_SCENE_EXACT_FEATURES. Same synchronisation rules as psm_render. */
int psm_render_panoptic(psm_ctx* ctx, const psm_scene* scene, const psm_camera* cam,
                        const psm_raster_config* cfg, const int32_t* query_class, int32_t n_query_class,
                        const psm_panoptic_targets* targets, psm_counters* counters);

/* ---- Backward of the render --------------------------
 * The blending backward of the training pipeline (proj/src/pipeline.cpp:347-460)
 * and project_surfel_backward (raster.cpp:179-203): given dL/d(colour, semantic
 * feature, label distribution) planes, the gradients of every surfel parameter.
 * Depth and normal planes carry no gradient, as in the reference. */
typedef struct psm_plane_grads {
  const double* color;    /* W*H*3, NULL = 0 */
  const double* sem_feat; /* W*H*C_sem, NULL = 0 */
  const double* ins_dist; /* W*H*N_q, NULL = 0 */
} psm_plane_grads;

typedef struct psm_scene_grads { /* host outputs, each may be NULL */
  double* opacity;  /* N */
  double* color;    /* N*3 */
  double* f_sem;    /* N*C_sem */
  double* labels;   /* N*N_q (per surfel, the MatX column) */
  double* center;   /* N*3 */
  double* rotation; /* N*4 (w, x, y, z) */
  double* scales;   /* N*2 */
} psm_scene_grads;

/* Re-runs the forward (recording each pixel's contributors) and back-propagates.
 * Synchronous. Gradients are sums over pixels in an unspecified order (fp64 atomics). */
int psm_render_backward(psm_ctx* ctx, const psm_scene* scene, const psm_camera* cam,
                        const psm_raster_config* cfg, const psm_plane_grads* grads, psm_scene_grads* out);

/* ---- Stage entry points (raster.hpp:87-126) --------------------------------
 * The reference's stage functions as device-backed batch calls with host inputs and
 * outputs (synchronous on the context stream). Results are bit-identical to the
 * reference's: the same fp64 arithmetic as the render pipeline (--fmad=false, the
 * glibc-exact exp). */

/* ProjectedSurfel (raster.hpp:21-30). 2x2 / 3x3 matrices column-major like Eigen. */
typedef struct psm_projected {
  int32_t source;           /* index into the scene (the reference's project_surfel leaves -1) */
  int32_t pad;
  double screen_center[2];
  double sigma[4];          /* J Sigma J^T, pixel^2 */
  double sort_depth;        /* camera-space z of the centre */
  double h[9];              /* tangent (u, v, 1) -> camera point */
  double h_inv[9];
  double footprint_inv[4];  /* inverse of sigma + 0.3 I */
  double normal_vis[3];
} psm_projected;

/* project_surfel (raster.cpp:94-142) of n surfels (N x 13 host AoS). status[i] = 1 when
 * surfel i projects (out[i] filled, out[i].source = -1 as the reference returns it), 0 when
 * culled. A degenerate quaternion on a surfel that passes the depth cull returns PSM_EINVAL
 * (std::invalid_argument in the reference); *bad_index (may be NULL) is its index. */
int psm_project_surfels(psm_ctx* ctx, const double* surfels13, int64_t n, const psm_camera* cam,
                        const psm_raster_config* cfg, psm_projected* out, int32_t* status, int64_t* bad_index);

/* bin_circle / bin_aabb (raster.cpp:51-90,144-152) of n projected surfels: per tile (row-major
 * tiles_x x tiles_y) the indices into `projected` whose box touches it, ordered by
 * (sort_depth, source). binning: PSM_BIN_CIRCLE (circle box, cfg->chi2) or PSM_BIN_AABB
 * (aabb box from `chi2`, bin_aabb's argument). tile_counts[tiles] and counters (rn_total,
 * rn_per_tile, tiles_x/y, nonempty_tiles) are always written; list (cap entries, the
 * concatenated per-tile lists) when non-NULL and cap >= rn_total. */
int psm_bin_projected(psm_ctx* ctx, const psm_projected* projected, int64_t n, const psm_camera* cam,
                      const psm_raster_config* cfg, int32_t binning, double chi2, int32_t* tile_counts,
                      int32_t* list, int64_t cap, psm_counters* counters);

/* sample_surfel_alpha + evaluate_alpha (raster.cpp:154-177) at m queries: surfel proj_index[q]
 * of `projected` (opacity[proj_index[q]]) at pixel position (px[q], py[q]). alpha is
 * evaluate_alpha's (0 outside the support or below alpha_min); u, v, w2, inside are
 * sample_surfel_alpha's (zero unless inside). */
typedef struct psm_alpha_sample {
  double alpha, u, v, w2;
  int32_t inside;
  int32_t pad;
} psm_alpha_sample;
int psm_sample_alpha(psm_ctx* ctx, const psm_projected* projected, const double* opacity, int64_t n_projected,
                     const int32_t* proj_index, const double* px, const double* py, int64_t m,
                     const psm_camera* cam, const psm_raster_config* cfg, psm_alpha_sample* out);

/* topk_select (raster.cpp:225-251) over n_lists independent lists (CSR: list l is entries
 * [offsets[l], offsets[l+1]) of weights / proj): selected[e] = 1 for the k best entries of
 * each list by (weight desc, proj asc), all of them when k >= the list's length. k >= 1
 * (render calls it with max(top_k, 1), raster.cpp:318; k = 0 is undefined in the reference). */
int psm_topk_select(psm_ctx* ctx, const double* weights, const int32_t* proj, const int64_t* offsets,
                    int32_t n_lists, int32_t k, int8_t* selected);

/* render with a RenderCache (raster.hpp:75-82, raster.cpp:310-315,399-403,507-510): the render
 * of psm_render into `targets` (host or device planes) plus the forward intermediates the
 * reference keeps for the backward pass, as host arrays:
 *   projected   [n_proj]   the projected surfels in source order (RenderCache::projected)
 *   tile_counts [tiles]    + tile_lists [rn_total]: TileGrid::tiles as indices into projected
 *   pixel_offsets [W*H+1]  + contribs [total]: RenderCache::pixels, each pixel's contributors
 *                          in blend order as (index into projected, alpha, u, v)
 * Pass NULL arrays (or too-small capacities) to size them: the counts are always returned. */
typedef struct psm_contribution {
  int32_t proj;
  int32_t pad;
  double alpha, u, v;
} psm_contribution;
typedef struct psm_render_cache_out {
  psm_projected* projected;
  int64_t projected_cap;
  int64_t n_projected;     /* out */
  int32_t* tile_counts;    /* tiles_x * tiles_y entries (NULL: skipped) */
  int32_t* tile_lists;
  int64_t tile_lists_cap;
  int64_t n_tile_entries;  /* out: rn_total */
  int64_t* pixel_offsets;  /* W*H+1 entries (NULL: skipped) */
  psm_contribution* contribs;
  int64_t contribs_cap;
  int64_t n_contribs;      /* out */
} psm_render_cache_out;
int psm_render_cache(psm_ctx* ctx, const psm_scene* scene, const psm_camera* cam, const psm_raster_config* cfg,
                     const psm_targets* targets, psm_counters* counters, psm_render_cache_out* cache);

/* Workload: make_street_scene (proj/src/synthetic.cpp:236-312) with the same
 * RNG draw order, plus `scale_mult` applied to s1 after it is drawn
 * (density-normalised variants; 1.0 = verbatim). Two-phase:
 * call with NULL outputs to get n; then with buffers of n*13, n*c_sem and (if
 * labels != NULL) n*n_instances doubles. The camera is the reference's
 * look_at((0,0,0) -> (0,0,20), up (0,-1,0), f = 0.8 W, near 0.1, far 200). */
typedef struct psm_street_spec {
  int32_t n_surfels;
  uint64_t seed;
  double min_aspect;
  int32_t image_w, image_h;
  int32_t c_sem;
  int32_t n_instances;
  double scale_mult;
} psm_street_spec;
int psm_make_street_scene(const psm_street_spec* spec, int64_t* n_out, double* surfels13,
                          double* f_sem, double* labels, psm_camera* cam);
/* The same scene's Surfel::f_ins (n x 8, 0.3 N(0,1) draws in the generator's order). */
int psm_make_street_scene_ins(const psm_street_spec* spec, int64_t* n_out, double* f_ins);

/* Camera::look_at / Camera::make (proj/src/core_types.cpp:18-60). */
int psm_camera_look_at(const double eye[3], const double target[3], const double up[3], double fx,
                       double fy, int32_t width, int32_t height, double near_clip,
                       double far_clip, psm_camera* out);
int psm_camera_make(const double r_cw[9], const double t_cw[3], double fx, double fy, double cx,
                    double cy, int32_t width, int32_t height, double near_clip, double far_clip,
                    psm_camera* out);

#ifdef __cplusplus
}
#endif

#endif /* PSM_H */
