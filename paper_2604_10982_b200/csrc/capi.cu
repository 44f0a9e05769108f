// capi.cu — the C-ABI (include/psm.h): contexts, scene upload and the
// per-frame render pipeline K1..K7 on one CUDA stream.
//
// Reference entry points replaced: psimap::render / render_into
// (proj/src/raster.cpp:266-511, raster.hpp:142-148). Per frame:
//   K1 preprocess       project_surfel + hot records + box + tile count  (raster.cpp:94-142,321-353)
//   K2 compact + sort   stable radix sort of (depth bits, source)        (raster.cpp:78-83)
//   K3 scan             tile counts in rank order -> key offsets, RN-Total
//   K4 emit             (tile, source) in rank order                       (raster.cpp:59-74)
//   K5 tile sort        stable radix sort on the tile bits
//   K6 ranges           per-tile [start, end), non-empty count             (raster.cpp:84-88)
//   K7 blend            compositing + Top-K + features                     (raster.cpp:355-506)
// Scratch is grow-only and owned by the context (render_into's buffer reuse,
// raster.cpp:255-262). No CPU fallback: without a CUDA device every entry
// point returns PSM_ECUDA.
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "psm_device.cuh"
#include "psm_kernels.h"
#include "psm_panoptic.h"

#include "psm_ctx.h"

namespace psm {
namespace {

int fail(psm_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->err = msg;
  return code;
}

}  // namespace

int fail_cuda(psm_ctx* ctx, cudaError_t e, const char* expr, const char* file, int line) {
  char buf[512];
  std::snprintf(buf, sizeof buf, "CUDA error %s (%s) at %s:%d: %s", cudaGetErrorName(e), cudaGetErrorString(e), file,
                line, expr);
  return fail(ctx, PSM_ECUDA, buf);
}

namespace {

template <class T>
int ensure(psm_ctx* ctx, Buf& b, size_t count, T** out) {
  const size_t bytes = count * sizeof(T) + 16;
  if (b.bytes < bytes) {
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.bytes = 0;
    const size_t want = bytes + bytes / 4;  // grow-only with headroom
    cudaError_t e = cudaMalloc(&b.p, want);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(ctx, PSM_ENOMEM, std::string("cudaMalloc failed: ") + cudaGetErrorString(e));
    }
    b.bytes = want;
  }
  *out = static_cast<T*>(b.p);
  return PSM_OK;
}


void free_buf(Buf& b) {
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.bytes = 0;
}

int tile_bits(int tiles) {
  int b = 1;
  while ((1 << b) < tiles) ++b;
  return b;
}

// Stage boundary i (0..5); boundaries of skipped stages are recorded at the
// same point so they time as zero.
void record(psm_ctx* ctx, int i) {
  if (!ctx->profiling) return;
  while (ctx->ev_next <= i) cudaEventRecord(ctx->ev[ctx->ev_next++], ctx->stream);
}

// Validates the subset of RasterConfig the GPU path supports.
int check_config(psm_ctx* ctx, const psm_raster_config* cfg, int feat_dims) {
  if (cfg->tile_size != 16) return fail(ctx, PSM_EUNSUPPORTED, "GPU path requires tile_size == 16");
  if (cfg->binning < 0 || cfg->binning > 2) return fail(ctx, PSM_EINVAL, "binning must be 0 (circle), 1 (aabb), 2 (ellipse)");
  if (cfg->blending < 0 || cfg->blending > 1) return fail(ctx, PSM_EINVAL, "blending must be 0 (full) or 1 (topk)");
  const int k_sel = cfg->top_k > 1 ? cfg->top_k : 1;
  if (cfg->blending == PSM_BLEND_TOPK && blend_kmax_for(k_sel) < 0)
    return fail(ctx, PSM_EUNSUPPORTED, "GPU path supports top_k <= 32");
  if (blend_nch_for(feat_dims) < 0) return fail(ctx, PSM_EUNSUPPORTED, "GPU path supports C_sem + N_q <= 512");
  return PSM_OK;
}

// The render proper: K1..K7 enqueued on the context stream with every count kept
// on the device. The only host round trip is the first frame of a context (or a
// frame whose RN-Total outgrew the key buffers), which reads RN-Total to size
// them; frames after that run without a host sync. Leaves results in `pl`
// (device) and counters in the pinned ctx->h_small (valid after the stream syncs).
// Host-target frames pass `on_band`: the blend then runs as row bands of tiles and
// on_band(band, y0, y1) is called after each band's launch (it queues that band's
// device-to-host copies on the copy stream, overlapping the next band's blend).
using BandHook = std::function<int(int band, int y0, int y1)>;
// cumulative band ends in 64ths of the tile rows; <= 8 bands (band events, work counters
// small[8..16))
// (C3 e2e, measured: 4,12,64 -> 180 frames/s; eight equal bands 174; 3,10,24,64 179;
// 2,8,64 171)
#ifndef PSM_HOST_BAND_CUTS
#define PSM_HOST_BAND_CUTS 4, 12, 64
#endif

int render_impl(psm_ctx* ctx, const psm_scene* sc, const psm_camera* cam, const psm_raster_config* cfg,
                const Planes& pl, psm_debug* dbg, const BandHook* on_band = nullptr) {
  cudaStream_t st = ctx->stream;
  const int64_t n = sc->n;
  const int W = cam->width, H = cam->height;
  const int ts = cfg->tile_size;
  const int tiles_x = (W + ts - 1) / ts, tiles_y = (H + ts - 1) / ts;
  const int tiles = tiles_x * tiles_y;
  if (tiles >= (1 << 19)) return fail(ctx, PSM_EUNSUPPORTED, "image has 2^19 or more 16x16 tiles");
  const int feat_dims = sc->c_sem + sc->n_q;
  const bool topk = cfg->blending == PSM_BLEND_TOPK;
  const int k_sel = cfg->top_k > 1 ? cfg->top_k : 1;

  DevCamera dc;
  std::memcpy(dc.r, cam->r_cw, sizeof dc.r);
  std::memcpy(dc.t, cam->t_cw, sizeof dc.t);
  dc.fx = cam->fx; dc.fy = cam->fy; dc.cx = cam->cx; dc.cy = cam->cy;
  dc.w = W; dc.h = H; dc.near_clip = cam->near_clip; dc.far_clip = cam->far_clip;
  DevRaster rs;
  rs.chi2 = cfg->chi2; rs.alpha_min = cfg->alpha_min; rs.t_min = cfg->t_min;
  rs.bg[0] = cfg->background[0]; rs.bg[1] = cfg->background[1]; rs.bg[2] = cfg->background[2];
  rs.support_cutoff = cfg->support_cutoff != 0;
  rs.binning = cfg->binning;
  if (rs.binning == PSM_BIN_ELLIPSE && !rs.support_cutoff) rs.binning = PSM_BIN_AABB;  // exactness needs the cutoff
  rs.render_depth_normal = cfg->render_depth_normal != 0;
  rs.tile_size = ts;
  rs.tiles_x = tiles_x; rs.tiles_y = tiles_y;

  // device counters (8-byte slots): [0] err, [1] nonempty tiles, [2] blended_total, [3] list overflow,
  // [4] n_proj (u32), [5] RN-Total (u32), [6] RN kept (u32), [7] key overflow
  unsigned long long* small = nullptr;
  PSM_TRY(ensure(ctx, ctx->dev_small, 16, &small));  // [8, 16): blend work counters
  uint32_t* n_proj_dev = reinterpret_cast<uint32_t*>(small + 4);
  uint32_t* rn_dev = reinterpret_cast<uint32_t*>(small + 5);
  uint32_t* rn_eff_dev = reinterpret_cast<uint32_t*>(small + 6);
  int32_t* key_ovf = reinterpret_cast<int32_t*>(small + 7);
  int32_t* ranges = nullptr;
  PSM_TRY(ensure(ctx, ctx->ranges, static_cast<size_t>(tiles) * 2, &ranges));
  uint32_t* tcounts = nullptr;
  unsigned long long* dminmax = nullptr;
  if (n > 0) {
    PSM_TRY(ensure(ctx, ctx->tile_counts, static_cast<size_t>(tiles) * kSplit, &tcounts));
    PSM_TRY(ensure(ctx, ctx->dminmax, 2, &dminmax));
  }

  ctx->ev_next = 0;
  record(ctx, 0);
  // counters, ranges, tile counters and the depth range reset in one launch
  launch_frame_init(small, ranges, 2 * tiles, tcounts, n > 0 ? tiles * kSplit : 0, dminmax, st);
  PSM_CUDA_TRY(cudaGetLastError());
  uint32_t* tvals_s = nullptr;
  uint8_t* tmasks_s = nullptr;
  const int32_t* tclasses_s = nullptr;
  int64_t key_cap = 0;
  if (n > 0) {
    SurfRec* recs; BinRec* bins; uint64_t* dbits; int32_t* valid;
    uint32_t *cursor, *ttotals, *tstart;
    int32_t* tclasses;
    PSM_TRY(ensure(ctx, ctx->recs, n, &recs));
    PSM_TRY(ensure(ctx, ctx->bins, n, &bins));
    PSM_TRY(ensure(ctx, ctx->depth_bits, n, &dbits));
    PSM_TRY(ensure(ctx, ctx->valid, n, &valid));
    PSM_TRY(ensure(ctx, ctx->cursor, static_cast<size_t>(tiles) * kSplit, &cursor));
    PSM_TRY(ensure(ctx, ctx->tile_totals, tiles, &ttotals));
    PSM_TRY(ensure(ctx, ctx->tile_start, tiles, &tstart));
    // K3b's sort-class lists and counts, and the blend's heaviest-first tile order
    PSM_TRY(ensure(ctx, ctx->tclasses, static_cast<size_t>(tiles) * (psm::kSortClasses + 2), &tclasses));
    // K1: projection, records, per-tile bucket sizes
    launch_preprocess(sc->surfels, n, dc, rs, recs, bins, dbits, tcounts, valid, n_proj_dev, dminmax,
                      reinterpret_cast<int32_t*>(small), st);
    PSM_CUDA_TRY(cudaGetLastError());
    record(ctx, 1);

    // key capacity: sized from the last frame's RN-Total; the first frame reads it (one host sync)
    if (ctx->key_cap == 0) {
      launch_tile_scan(tcounts, tiles, 0xffffffffu, ranges, cursor, ttotals, tstart, rn_dev, rn_eff_dev, small + 1,
                       key_ovf, tclasses, st);
      uint32_t rn_host = 0;
      PSM_CUDA_TRY(cudaMemcpyAsync(&rn_host, rn_dev, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
      PSM_CUDA_TRY(cudaStreamSynchronize(st));
      ctx->key_cap = static_cast<int64_t>(rn_host) + static_cast<int64_t>(rn_host) / 2 + 4096;
    }
    key_cap = ctx->key_cap;
    if (key_cap > 0x7fffffffLL) return fail(ctx, PSM_EUNSUPPORTED, "RN-Total exceeds 2^31 tile assignments");
    uint32_t* tvals;
    uint8_t* tmasks;
    uint64_t *tkeys, *tkeys2;
    PSM_TRY(ensure(ctx, ctx->tvals, key_cap, &tvals));
    PSM_TRY(ensure(ctx, ctx->tmasks, key_cap, &tmasks));
    PSM_TRY(ensure(ctx, ctx->kscratch, key_cap, &tkeys));
    PSM_TRY(ensure(ctx, ctx->kscratch2, key_cap, &tkeys2));
    int src_bits = 1;
    while ((int64_t{1} << src_bits) < n) ++src_bits;

    // K3: bucket offsets = per-tile ranges, RN-Total, non-empty tiles
    launch_tile_scan(tcounts, tiles, static_cast<uint32_t>(key_cap), ranges, cursor, ttotals, tstart, rn_dev,
                     rn_eff_dev, small + 1, key_ovf, tclasses, st);
    PSM_CUDA_TRY(cudaGetLastError());
    record(ctx, 2);
    // K4: every (surfel, tile) pair into its tile's bucket
    launch_emit(valid, n, recs, bins, rs, H, cursor, tstart, static_cast<uint32_t>(key_cap), tkeys, dbits, dminmax,
                src_bits, W, st);
    PSM_CUDA_TRY(cudaGetLastError());
    record(ctx, 3);
    // K5: per-tile sort by (depth bits, source)
    launch_sort_tiles(ranges, tiles, tkeys, tkeys2, tvals, tmasks, dbits, dminmax, src_bits, tclasses, st, ctx->side,
                      ctx->side2, ctx->fork, ctx->join, ctx->join2);
    PSM_CUDA_TRY(cudaGetLastError());
    tvals_s = tvals;
    tmasks_s = tmasks;
    tclasses_s = tclasses;
    record(ctx, 4);
  }
  // K7: blend
  BlendParams bp;
  std::memset(&bp, 0, sizeof bp);
  bp.ranges = ranges;
  bp.vals = tvals_s;
  bp.masks = tmasks_s;
  bp.recs = static_cast<const SurfRec*>(ctx->recs.p);
  bp.feat = sc->feat;
  bp.feat_dims = feat_dims; bp.c_sem = sc->c_sem; bp.n_q = sc->n_q;
  bp.width = W; bp.height = H; bp.tiles_x = tiles_x;
  bp.cam_cx = cam->cx; bp.cam_cy = cam->cy; bp.cam_fx = cam->fx; bp.cam_fy = cam->fy;
  bp.chi2 = cfg->chi2; bp.alpha_min = cfg->alpha_min; bp.t_min = cfg->t_min;
  bp.bg0 = cfg->background[0]; bp.bg1 = cfg->background[1]; bp.bg2 = cfg->background[2];
  bp.support_cutoff = cfg->support_cutoff != 0;
  bp.render_depth_normal = cfg->render_depth_normal != 0;
  bp.k_sel = k_sel;
  bp.color = pl.color; bp.depth = pl.depth; bp.normal = pl.normal; bp.sem_feat = pl.sem; bp.ins_dist = pl.ins;
  bp.alpha_acc = pl.alpha; bp.ins_argmax = pl.arg; bp.blend_count = pl.cnt;
  bp.blended_total = small + 2;
  bp.list_overflow = reinterpret_cast<int32_t*>(small + 3);
  const size_t npx = static_cast<size_t>(W) * H;
  if (dbg && dbg->topk_src && topk) {
    int32_t* tk;
    PSM_TRY(ensure(ctx, ctx->topk_dbg, npx * k_sel, &tk));
    bp.topk_dbg = tk;
  }
  // render with labels: the fp64 feature phase (exact ins_argmax) over the scene's fp64 rows
  const bool planes64 = !pl.pan_ids && !pl.cache && sc->n_q > 0 && sc->feat64 != nullptr;
  if (planes64) {
    bp.planes64 = 1;
    bp.feat64 = sc->feat64;
  }
  const bool full_list = (!topk && feat_dims > 0) || pl.cache;
  if (full_list) {
    if (ctx->list_cap == 0) ctx->list_cap = 128;
    uint2* lists;
    const size_t lslots = static_cast<size_t>(psm_list_slots(W, H, ctx->list_cap));
    PSM_TRY(ensure(ctx, ctx->lists, lslots, &lists));
    bp.lists = lists;
    bp.list_cap = ctx->list_cap;
    if (pl.pan_ids || planes64) {
      double* lw;
      PSM_TRY(ensure(ctx, ctx->lists_w, lslots, &lw));
      bp.lists_w = lw;
    }
    if (pl.cache) {
      double* lt;
      PSM_TRY(ensure(ctx, ctx->lists_t, lslots, &lt));
      bp.lists_t = lt;
      if (topk) {
        int32_t* tk;
        PSM_TRY(ensure(ctx, ctx->topk_pos, npx * k_sel, &tk));
        bp.topk_pos = tk;
      }
    }
  }
  if (pl.pan_ids) {
    bp.feat64 = sc->feat64;
    bp.pan_ids = pl.pan_ids;
    bp.pan_classes = pl.pan_classes;
    bp.pan_sem = pl.pan_sem;
    bp.query_class = pl.qclass;
    bp.n_query_class = pl.n_qclass;
  }
  if (!on_band) {
    bp.work = reinterpret_cast<int32_t*>(small + 8);
    if (tclasses_s) bp.order = tclasses_s + (psm::kSortClasses + 1) * static_cast<int64_t>(tiles);
    launch_blend(bp, tiles, topk, st);
    PSM_CUDA_TRY(cudaGetLastError());
  } else {
    // Band b ends at kBandCuts[b]/64 of the tile rows. Host-target frames are bound by the
    // copies (PCIe), so the first band is small (its copies start soon after the front end)
    // and the rest are few and large (every copy costs ~4 us on the copy engine).
    static constexpr int kBandCuts[] = {PSM_HOST_BAND_CUTS};
    constexpr int n_cuts = static_cast<int>(sizeof(kBandCuts) / sizeof(kBandCuts[0]));
    static_assert(n_cuts <= 8 && kBandCuts[n_cuts - 1] == 64, "band cuts: <= 8 bands, the last at 64/64");
    int ty1 = 0;
    for (int b = 0; b < n_cuts && ty1 < tiles_y; ++b) {
      const int ty0 = ty1;
      ty1 = (tiles_y * kBandCuts[b] + 63) / 64;
      if (ty1 <= ty0) ty1 = ty0 + 1;
      if (ty1 > tiles_y || b == n_cuts - 1) ty1 = tiles_y;
      bp.tile_base = ty0 * tiles_x;
      bp.work = reinterpret_cast<int32_t*>(small + 8 + b);
      launch_blend(bp, (ty1 - ty0) * tiles_x, topk, st);
      PSM_CUDA_TRY(cudaGetLastError());
      PSM_TRY((*on_band)(b, ty0 * ts, ty1 * ts < H ? ty1 * ts : H));
    }
  }
  record(ctx, 5);

  // counters -> pinned host memory (read after the stream syncs)
  PSM_CUDA_TRY(cudaMemcpyAsync(ctx->h_small, small, 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
  ctx->last.tiles_x = tiles_x;
  ctx->last.tiles_y = tiles_y;

  if (dbg) {
    PSM_CUDA_TRY(cudaStreamSynchronize(st));
    const unsigned long long* h = reinterpret_cast<const unsigned long long*>(ctx->h_small);
    const int64_t n_proj = static_cast<int64_t>(static_cast<uint32_t>(h[4]));
    const int64_t rn = static_cast<int64_t>(static_cast<uint32_t>(h[6]));
    if (dbg->tile_ranges) PSM_CUDA_TRY(cudaMemcpy(dbg->tile_ranges, ranges, sizeof(int32_t) * 2 * tiles, cudaMemcpyDeviceToHost));
    const int64_t kcopy = rn < dbg->cap_keys ? rn : dbg->cap_keys;
    if (kcopy > 0 && dbg->tile_vals) PSM_CUDA_TRY(cudaMemcpy(dbg->tile_vals, tvals_s, sizeof(int32_t) * kcopy, cudaMemcpyDeviceToHost));
    if ((kcopy > 0 && dbg->tile_keys) || dbg->depth_order) {
      // debug only: the global depth rank of every projected surfel ((sort_depth, source)
      // order), by compaction + the stable radix sort, for the (tile << 32 | rank) keys
      int32_t* rank_of;
      uint64_t *dk, *keys_c, *keys_s;
      uint32_t *pos, *src_c, *src_s, *scan_tmp, *hist, *totals;
      PSM_TRY(ensure(ctx, ctx->rank_of, n, &rank_of));
      PSM_TRY(ensure(ctx, ctx->dbg_keys, rn > 0 ? rn : 1, &dk));
      PSM_TRY(ensure(ctx, ctx->keys_c, n, &keys_c));
      PSM_TRY(ensure(ctx, ctx->keys_s, n, &keys_s));
      PSM_TRY(ensure(ctx, ctx->pos, n, &pos));
      PSM_TRY(ensure(ctx, ctx->src_c, n, &src_c));
      PSM_TRY(ensure(ctx, ctx->src_s, n, &src_s));
      PSM_TRY(ensure(ctx, ctx->scan_tmp, scan_cta_words(n) + 8, &scan_tmp));
      PSM_TRY(ensure(ctx, ctx->hist, radix_hist_words(n), &hist));
      PSM_TRY(ensure(ctx, ctx->totals, 256, &totals));
      const int32_t* valid = static_cast<const int32_t*>(ctx->valid.p);
      const uint64_t* dbits = static_cast<const uint64_t*>(ctx->depth_bits.p);
      exclusive_scan_i32(valid, n, pos, totals + 255, scan_tmp, st);
      launch_compact(valid, reinterpret_cast<const int32_t*>(pos), dbits, n, keys_c, src_c, st);
      bool in_alt = false;
      radix_sort_u64(keys_c, src_c, keys_s, src_s, n_proj_dev, n, 0, 64, hist, totals, st, &in_alt);
      const uint32_t* order = in_alt ? src_s : src_c;
      launch_rank_of(order, n_proj_dev, n, rank_of, st);
      launch_debug_keys(ranges, tiles, tvals_s, rank_of, dk, st);
      PSM_CUDA_TRY(cudaGetLastError());
      if (kcopy > 0 && dbg->tile_keys)
        PSM_CUDA_TRY(cudaMemcpyAsync(dbg->tile_keys, dk, sizeof(uint64_t) * kcopy, cudaMemcpyDeviceToHost, st));
      const int64_t pcopy = n_proj < dbg->cap_proj ? n_proj : dbg->cap_proj;
      if (pcopy > 0 && dbg->depth_order)
        PSM_CUDA_TRY(cudaMemcpyAsync(dbg->depth_order, order, sizeof(int32_t) * pcopy, cudaMemcpyDeviceToHost, st));
    }
    if (bp.topk_dbg)
      PSM_CUDA_TRY(cudaMemcpyAsync(dbg->topk_src, bp.topk_dbg, sizeof(int32_t) * npx * k_sel, cudaMemcpyDeviceToHost, st));
    PSM_CUDA_TRY(cudaStreamSynchronize(st));
  }
  return PSM_OK;
}

// After the stream has synchronised: did the frame fit its buffers? Grows them if not
// (the caller then re-renders). Also raises PSM_EINVAL for a degenerate quaternion.
int check_frame(psm_ctx* ctx, bool* rerun) {
  const unsigned long long* h = reinterpret_cast<const unsigned long long*>(ctx->h_small);
  *rerun = false;
  if (static_cast<int32_t>(h[0])) return fail(ctx, PSM_EINVAL, "degenerate quaternion");
  const uint32_t rn = static_cast<uint32_t>(h[5]);
  if (static_cast<int32_t>(h[7])) {  // RN-Total outgrew the key buffers
    ctx->key_cap = static_cast<int64_t>(rn) + static_cast<int64_t>(rn) / 2 + 4096;
    *rerun = true;
  }
  const int32_t m = static_cast<int32_t>(h[3]);
  if (m > ctx->list_cap && ctx->list_cap > 0) {  // a pixel had more contributors than the Full-mode list holds
    ctx->list_cap = m;
    *rerun = true;
  }
  return PSM_OK;
}

void finish_counters(psm_ctx* ctx) {
  const unsigned long long* h = reinterpret_cast<const unsigned long long*>(ctx->h_small);
  ctx->last.nonempty_tiles = static_cast<int64_t>(h[1]);
  ctx->last.blended_total = h[2];
  ctx->last.n_proj = static_cast<int64_t>(static_cast<uint32_t>(h[4]));
  ctx->last.rn_total = static_cast<uint64_t>(static_cast<uint32_t>(h[5]));
  ctx->last.rn_per_tile = h[1] > 0 ? static_cast<double>(ctx->last.rn_total) / static_cast<double>(h[1]) : 0.0;
}

void read_times(psm_ctx* ctx) {
  if (!ctx->profiling || ctx->ev_next < 6) return;
  float t[5] = {};
  for (int i = 0; i < 5; ++i) cudaEventElapsedTime(&t[i], ctx->ev[i], ctx->ev[i + 1]);
  ctx->times.preprocess = t[0];
  ctx->times.tile_scan = t[1];
  ctx->times.emit = t[2];
  ctx->times.tile_sort = t[3];
  ctx->times.blend = t[4];
  cudaEventElapsedTime(&ctx->times.total, ctx->ev[0], ctx->ev[5]);
}

int sync_impl(psm_ctx* ctx);

// Validates (and if needed re-renders) the views the twin context rendered in the last
// batch; after it the twin's frames are complete in stream order before ctx's next work.
int drain_twin(psm_ctx* ctx) {
  if (!ctx->twin_pending) return PSM_OK;
  ctx->twin_pending = false;
  const int st = sync_impl(ctx->twin);
  if (st != PSM_OK) return fail(ctx, st, std::string("batch view: ") + ctx->twin->err);
  return PSM_OK;
}

// pt != NULL: render_panoptic. The standard planes then live in context scratch, the
// feature planes are not materialised, and pt's three id planes are the outputs.
int render_common(psm_ctx* ctx, const psm_scene* sc, const psm_camera* cam, const psm_raster_config* cfg,
                  const psm_targets* tg_in, psm_counters* counters, psm_debug* dbg,
                  const psm_panoptic_targets* pt = nullptr, const int32_t* qclass = nullptr, int32_t n_qclass = 0) {
  const psm_targets scratch_only = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, 1};
  const psm_targets* tg = pt ? &scratch_only : tg_in;
  if (!ctx || !sc || !cam || !cfg || !tg) return fail(ctx, PSM_EINVAL, "null argument");
  if (cam->width <= 0 || cam->height <= 0) return fail(ctx, PSM_EINVAL, "camera: image size must be positive");
  // Camera::make's invariant (core_types.cpp:23-25); the depth keys order positive depths only
  if (!(cam->near_clip > 0) || !(cam->near_clip < cam->far_clip))
    return fail(ctx, PSM_EINVAL, "camera: require 0 < near < far");
  PSM_TRY(check_config(ctx, cfg, sc->c_sem + sc->n_q));
  PSM_CUDA_TRY(cudaSetDevice(ctx->device));
  const size_t npx = static_cast<size_t>(cam->width) * cam->height;
  Planes pl;
  // device planes: caller's when on_device and non-NULL, else context scratch
  auto pick = [&](void* user, psm::Buf& b, size_t count, size_t elem, void** out) -> int {
    if (tg->on_device && user) {
      *out = user;
      return PSM_OK;
    }
    char* p;
    PSM_TRY(ensure(ctx, b, count * elem, &p));
    *out = p;
    return PSM_OK;
  };
  const int cs = sc->c_sem, nq = sc->n_q;
  PSM_TRY(pick(tg->color, ctx->plane_color, npx * 3, 4, reinterpret_cast<void**>(&pl.color)));
  PSM_TRY(pick(tg->depth, ctx->plane_depth, npx * 2, 4, reinterpret_cast<void**>(&pl.depth)));
  PSM_TRY(pick(tg->normal, ctx->plane_normal, npx * 3, 4, reinterpret_cast<void**>(&pl.normal)));
  PSM_TRY(pick(tg->alpha_acc, ctx->plane_alpha, npx, 4, reinterpret_cast<void**>(&pl.alpha)));
  PSM_TRY(pick(tg->ins_argmax, ctx->plane_arg, npx, 4, reinterpret_cast<void**>(&pl.arg)));
  PSM_TRY(pick(tg->blend_count, ctx->plane_cnt, npx, 4, reinterpret_cast<void**>(&pl.cnt)));
  pl.sem = nullptr;
  pl.ins = nullptr;
  // feature planes are always produced (context scratch when the caller passes NULL),
  // except by render_panoptic, which reduces them to ids inside the blend
  if (cs > 0 && !pt) PSM_TRY(pick(tg->sem_feat, ctx->plane_sem, npx * cs, 4, reinterpret_cast<void**>(&pl.sem)));
  if (nq > 0 && !pt) PSM_TRY(pick(tg->ins_dist, ctx->plane_ins, npx * nq, 4, reinterpret_cast<void**>(&pl.ins)));
  if (pt) {
    if (!sc->feat64 && cs + nq > 0)
      return fail(ctx, PSM_EUNSUPPORTED, "render_panoptic needs a scene created with PSM_SCENE_EXACT_FEATURES");
    if (n_qclass < 0 || (n_qclass > 0 && !qclass)) return fail(ctx, PSM_EINVAL, "query classes");
    auto pick_pan = [&](int32_t* user, psm::Buf& b, int32_t** out) -> int {
      if (pt->on_device && user) {
        *out = user;
        return PSM_OK;
      }
      return ensure(ctx, b, npx, out);
    };
    PSM_TRY(pick_pan(pt->ids, ctx->pan_ids, &pl.pan_ids));
    PSM_TRY(pick_pan(pt->classes, ctx->pan_classes, &pl.pan_classes));
    PSM_TRY(pick_pan(pt->sem_classes, ctx->pan_sem, &pl.pan_sem));
    int32_t* qc = nullptr;
    PSM_TRY(ensure(ctx, ctx->qclass, static_cast<size_t>(n_qclass > 0 ? n_qclass : 1), &qc));
    if (n_qclass > 0)
      PSM_CUDA_TRY(cudaMemcpyAsync(qc, qclass, sizeof(int32_t) * n_qclass, cudaMemcpyHostToDevice, ctx->stream));
    pl.qclass = qc;
    pl.n_qclass = n_qclass;
  }
  const bool host_out = pt ? !pt->on_device : !tg->on_device;
  // host targets: each finished row band of every plane is copied on the copy stream while
  // the next band blends; the main stream then waits for the copies (the planes are
  // context scratch that the next frame overwrites)
  const BandHook band_d2h = [&](int b, int y0, int y1) -> int {
    cudaStream_t cs_ = ctx->copy;
    PSM_CUDA_TRY(cudaEventRecord(ctx->band_ev[b], ctx->stream));
    PSM_CUDA_TRY(cudaStreamWaitEvent(cs_, ctx->band_ev[b], 0));
    const size_t p0 = static_cast<size_t>(y0) * cam->width, np = static_cast<size_t>(y1 - y0) * cam->width;
    auto d2h = [&](void* dst, const void* src, size_t ch) -> int {
      if (dst && np)
        PSM_CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(dst) + p0 * ch * 4, static_cast<const char*>(src) + p0 * ch * 4,
                                     np * ch * 4, cudaMemcpyDeviceToHost, cs_));
      return PSM_OK;
    };
    PSM_TRY(d2h(tg->color, pl.color, 3));
    PSM_TRY(d2h(tg->depth, pl.depth, 2));
    PSM_TRY(d2h(tg->normal, pl.normal, 3));
    PSM_TRY(d2h(tg->alpha_acc, pl.alpha, 1));
    PSM_TRY(d2h(tg->ins_argmax, pl.arg, 1));
    PSM_TRY(d2h(tg->blend_count, pl.cnt, 1));
    if (pl.sem && tg->sem_feat) PSM_TRY(d2h(tg->sem_feat, pl.sem, cs));
    if (pl.ins && tg->ins_dist) PSM_TRY(d2h(tg->ins_dist, pl.ins, nq));
    if (pt) {
      PSM_TRY(d2h(pt->ids, pl.pan_ids, 1));
      PSM_TRY(d2h(pt->classes, pl.pan_classes, 1));
      PSM_TRY(d2h(pt->sem_classes, pl.pan_sem, 1));
    }
    if (y1 == cam->height) {
      PSM_CUDA_TRY(cudaEventRecord(ctx->copy_done, cs_));
      PSM_CUDA_TRY(cudaStreamWaitEvent(ctx->stream, ctx->copy_done, 0));
    }
    return PSM_OK;
  };
  const BandHook* hook = host_out ? &band_d2h : nullptr;
  // earlier asynchronous frames are validated before a synchronous one, or when the list is full
  const bool async = !(counters || host_out || dbg);
  if (!async) PSM_TRY(drain_twin(ctx));
  if (!ctx->pend.empty() && (!async || ctx->pend.size() >= static_cast<size_t>(psm_ctx::kMaxPend)))
    PSM_TRY(sync_impl(ctx));
  ctx->h_small = ctx->h_ring + 8 * (async ? ctx->pend.size() : static_cast<size_t>(psm_ctx::kMaxPend));
  PSM_TRY(render_impl(ctx, sc, cam, cfg, pl, dbg, hook));
  if (!async) {
    for (int attempt = 0;; ++attempt) {
      PSM_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
      bool rerun = false;
      PSM_TRY(check_frame(ctx, &rerun));
      if (!rerun) break;
      if (attempt >= 3) return fail(ctx, PSM_ENOMEM, "render buffers did not converge");
      PSM_TRY(render_impl(ctx, sc, cam, cfg, pl, dbg, hook));
    }
    finish_counters(ctx);
    read_times(ctx);
    if (counters) *counters = ctx->last;
  } else {
    ctx->pend.push_back({sc, *cam, *cfg, pl});
  }
  return PSM_OK;
}

// psm_sync: wait, validate the last asynchronous frame, re-render it if it outgrew its buffers.
int sync_impl(psm_ctx* ctx) {
  PSM_CUDA_TRY(cudaSetDevice(ctx->device));
  PSM_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  if (!ctx->pend.empty()) {
    std::vector<psm_ctx::Pending> pend;
    pend.swap(ctx->pend);  // the list is consumed whatever the outcome
    size_t first = pend.size();
    for (size_t j = 0; j < pend.size(); ++j) {  // every frame's flags (errors, capacities)
      ctx->h_small = ctx->h_ring + 8 * j;
      bool rerun = false;
      PSM_TRY(check_frame(ctx, &rerun));
      if (rerun && first == pend.size()) first = j;
    }
    ctx->h_small = ctx->h_ring + 8 * psm_ctx::kMaxPend;
    for (size_t j = first; j < pend.size(); ++j) {  // re-render in the original order
      const psm_ctx::Pending& f = pend[j];
      for (int attempt = 0;; ++attempt) {
        PSM_TRY(render_impl(ctx, f.scene, &f.cam, &f.cfg, f.pl, nullptr));
        PSM_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
        bool rerun = false;
        PSM_TRY(check_frame(ctx, &rerun));
        if (!rerun) break;
        if (attempt >= 3) return fail(ctx, PSM_ENOMEM, "render buffers did not converge");
      }
    }
    if (first == pend.size()) ctx->h_small = ctx->h_ring + 8 * (pend.size() - 1);  // the last frame's counters
  }
  finish_counters(ctx);
  read_times(ctx);
  return PSM_OK;
}

}  // namespace
}  // namespace psm

using psm::fail;

extern "C" {

int psm_create(int device, void* stream, psm_ctx** out) {
  if (!out) return PSM_EINVAL;
  *out = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count <= 0) {
    cudaGetLastError();
    return PSM_ECUDA;  // no CPU fallback
  }
  if (device < 0 || device >= count) return PSM_EINVAL;
  psm_ctx* ctx = new psm_ctx();
  ctx->device = device;
  if (cudaSetDevice(device) != cudaSuccess) { delete ctx; return PSM_ECUDA; }
  if (stream) {
    ctx->stream = static_cast<cudaStream_t>(stream);
  } else {
    if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) { delete ctx; return PSM_ECUDA; }
    ctx->own_stream = true;
  }
  for (auto& e : ctx->ev) cudaEventCreate(&e);
  if (cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&ctx->side2, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->join, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->join2, cudaEventDisableTiming) != cudaSuccess) {
    delete ctx;
    return PSM_ECUDA;
  }
  if (cudaStreamCreateWithFlags(&ctx->copy, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->copy_done, cudaEventDisableTiming) != cudaSuccess) {
    delete ctx;
    return PSM_ECUDA;
  }
  for (auto& e : ctx->band_ev)
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) { delete ctx; return PSM_ECUDA; }
  const size_t ring_bytes = 8 * sizeof(int64_t) * (psm_ctx::kMaxPend + 1);
  if (cudaMallocHost(&ctx->h_ring, ring_bytes) != cudaSuccess) { delete ctx; return PSM_ENOMEM; }
  std::memset(ctx->h_ring, 0, ring_bytes);
  ctx->h_small = ctx->h_ring + 8 * psm_ctx::kMaxPend;
  *out = ctx;
  return PSM_OK;
}

int psm_destroy(psm_ctx* ctx) {
  if (!ctx) return PSM_OK;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  psm::Buf* bufs[] = {&ctx->recs, &ctx->bins, &ctx->depth_bits, &ctx->dminmax, &ctx->tile_counts, &ctx->cursor, &ctx->tile_totals, &ctx->tile_start, &ctx->kscratch, &ctx->kscratch2, &ctx->valid, &ctx->pos,
                      &ctx->keys_c, &ctx->src_c, &ctx->keys_s, &ctx->src_s,
                      &ctx->tkeys, &ctx->tvals, &ctx->tkeys2, &ctx->tvals2, &ctx->ranges, &ctx->scan_tmp, &ctx->hist, &ctx->khist, &ctx->totals,
                      &ctx->dev_small, &ctx->lists, &ctx->rank_of, &ctx->dbg_keys, &ctx->topk_dbg, &ctx->tmasks, &ctx->tclasses,
                      &ctx->lists_w, &ctx->pan_ids, &ctx->pan_classes, &ctx->pan_sem, &ctx->qclass, &ctx->lab_tmp,
                      &ctx->lab_scratch, &ctx->lab_dist, &ctx->lab_arg, &ctx->lists_t, &ctx->topk_pos, &ctx->bw_gin,
                      &ctx->bw_out,
                      &ctx->plane_color, &ctx->plane_depth, &ctx->plane_normal, &ctx->plane_sem, &ctx->plane_ins,
                      &ctx->plane_arg, &ctx->plane_alpha, &ctx->plane_cnt};
  for (psm::Buf* b : bufs) psm::free_buf(*b);
  for (auto& e : ctx->ev) if (e) cudaEventDestroy(e);
  if (ctx->fork) cudaEventDestroy(ctx->fork);
  if (ctx->join) cudaEventDestroy(ctx->join);
  if (ctx->join2) cudaEventDestroy(ctx->join2);
  if (ctx->side) cudaStreamDestroy(ctx->side);
  if (ctx->side2) cudaStreamDestroy(ctx->side2);
  for (auto& e : ctx->band_ev) if (e) cudaEventDestroy(e);
  if (ctx->copy_done) cudaEventDestroy(ctx->copy_done);
  if (ctx->copy) cudaStreamDestroy(ctx->copy);
  if (ctx->h_ring) cudaFreeHost(ctx->h_ring);
  if (ctx->twin) psm_destroy(ctx->twin);
  if (ctx->batch_fork) cudaEventDestroy(ctx->batch_fork);
  if (ctx->batch_join) cudaEventDestroy(ctx->batch_join);
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
  return PSM_OK;
}

const char* psm_last_error(const psm_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int psm_set_profiling(psm_ctx* ctx, int enabled) {
  if (!ctx) return PSM_EINVAL;
  ctx->profiling = enabled != 0;
  return PSM_OK;
}

int psm_get_stage_times(const psm_ctx* ctx, psm_stage_times* out) {
  if (!ctx || !out) return PSM_EINVAL;
  *out = ctx->times;
  return PSM_OK;
}

int psm_sync(psm_ctx* ctx) {
  if (!ctx) return PSM_EINVAL;
  const bool twin_last = ctx->twin_pending && ctx->twin_last;
  PSM_TRY(psm::drain_twin(ctx));  // views of the last batch rendered by the twin context
  PSM_TRY(psm::sync_impl(ctx));
  if (twin_last) ctx->last = ctx->twin->last;  // psm_last_counters: the batch's last view
  return PSM_OK;
}

int psm_last_counters(const psm_ctx* ctx, psm_counters* out) {
  if (!ctx || !out) return PSM_EINVAL;
  *out = ctx->last;
  return PSM_OK;
}

int psm_scene_create(psm_ctx* ctx, const psm_scene_desc* d, psm_scene** out) {
  if (!ctx || !out || !d) return PSM_EINVAL;
  *out = nullptr;
  int64_t n = d->n;
  int32_t c_sem = d->c_sem, n_q = d->n_q, c_ins = d->c_ins;
  if (n < 0 || n > 0x7fffffffLL || c_sem < 0 || n_q < 0 || c_ins < 0) return fail(ctx, PSM_EINVAL, "scene: bad sizes");
  if (n > 0 && !d->surfels13) return fail(ctx, PSM_EINVAL, "scene: null surfels");
  if (c_sem > 0 && n > 0 && !d->f_sem) return fail(ctx, PSM_EINVAL, "scene: null f_sem with c_sem > 0");
  if (!d->labels) n_q = 0;
  if (!d->f_ins) c_ins = 0;
  if (n == 0) c_sem = 0;  // SceneMap::c_sem() of an empty scene (core_types.hpp:108)
  PSM_CUDA_TRY(cudaSetDevice(ctx->device));
  psm_scene* sc = new psm_scene();
  sc->device = ctx->device;
  sc->n = n;
  sc->c_sem = c_sem;
  sc->n_q = n_q;
  sc->c_ins = c_ins;
  sc->flags = d->flags;
  const int D = c_sem + n_q;
  // fp64 rows are kept for PSM_SCENE_EXACT_FEATURES and whenever the scene has labels (the
  // render's fp64 label phase gives the reference's ins_argmax exactly)
  const bool exact = (d->flags & PSM_SCENE_EXACT_FEATURES) != 0 || n_q > 0;
  if (n > 0) {
    cudaError_t e = cudaMalloc(&sc->surfels, sizeof(double) * 13 * n);
    if (e == cudaSuccess) e = cudaMemcpy(sc->surfels, d->surfels13, sizeof(double) * 13 * n, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && D > 0) {
      std::vector<double> f64(exact ? static_cast<size_t>(n) * D : 0);
      std::vector<float> f(static_cast<size_t>(n) * D);
      for (int64_t i = 0; i < n; ++i) {
        for (int c = 0; c < c_sem; ++c) {
          const double v = d->f_sem[i * c_sem + c];
          f[i * D + c] = static_cast<float>(v);
          if (exact) f64[i * D + c] = v;
        }
        for (int q = 0; q < n_q; ++q) {
          const double v = d->labels[i * n_q + q];
          f[i * D + c_sem + q] = static_cast<float>(v);
          if (exact) f64[i * D + c_sem + q] = v;
        }
      }
      e = cudaMalloc(&sc->feat, sizeof(float) * f.size());
      if (e == cudaSuccess) e = cudaMemcpy(sc->feat, f.data(), sizeof(float) * f.size(), cudaMemcpyHostToDevice);
      if (e == cudaSuccess && exact) {
        e = cudaMalloc(&sc->feat64, sizeof(double) * f64.size());
        if (e == cudaSuccess)
          e = cudaMemcpy(sc->feat64, f64.data(), sizeof(double) * f64.size(), cudaMemcpyHostToDevice);
      }
    }
    if (e == cudaSuccess && c_ins > 0) {
      e = cudaMalloc(&sc->f_ins, sizeof(double) * c_ins * n);
      if (e == cudaSuccess) e = cudaMemcpy(sc->f_ins, d->f_ins, sizeof(double) * c_ins * n, cudaMemcpyHostToDevice);
    }
    if (e != cudaSuccess) {
      psm_scene_free(ctx, sc);
      return psm::fail_cuda(ctx, e, "scene upload", __FILE__, __LINE__);
    }
  }
  *out = sc;
  return PSM_OK;
}

int psm_scene_upload(psm_ctx* ctx, const double* surfels13, int64_t n, const double* f_sem, int32_t c_sem,
                     const double* labels, int32_t n_q, psm_scene** out) {
  psm_scene_desc d{surfels13, n, f_sem, c_sem, labels, n_q, nullptr, 0, 0};
  return psm_scene_create(ctx, &d, out);
}

int psm_assign_labels(psm_ctx* ctx, psm_scene* sc, const psm_queries* qs, double* dist_out, int32_t* argmax_out) {
  if (!ctx || !sc || !qs) return PSM_EINVAL;
  const int32_t nq = qs->n;
  if (nq < 0 || (nq > 0 && (!qs->feature || !qs->mean || !qs->cov || !qs->alive)))
    return fail(ctx, PSM_EINVAL, "assign_labels: bad queries");
  if (sc->n > 0 && qs->c_ins != sc->c_ins)
    return fail(ctx, PSM_EINVAL, "feature_similarity: dimension mismatch");  // panoptic.cpp:12-14
  if (sc->c_sem + nq > 512) return fail(ctx, PSM_EUNSUPPORTED, "GPU path supports C_sem + N_q <= 512");
  PSM_CUDA_TRY(cudaSetDevice(ctx->device));
  // asynchronous frames still pending on this context (or its batch twin) may be re-rendered
  // at psm_sync against this scene: settle them before its labels change
  PSM_TRY(psm::drain_twin(ctx));
  if (!ctx->pend.empty()) PSM_TRY(psm::sync_impl(ctx));
  const int64_t n = sc->n;
  const int c_ins = qs->c_ins;
  // alive queries and their inverse covariances (panoptic.cpp:44-62), host side, once
  std::vector<int32_t> alive_index, alive_slot(static_cast<size_t>(nq > 0 ? nq : 1), -1);
  for (int q = 0; q < nq; ++q)
    if (qs->alive[q]) {
      alive_slot[q] = static_cast<int32_t>(alive_index.size());
      alive_index.push_back(q);
    }
  const int na = static_cast<int>(alive_index.size());
  std::vector<double> qtab(static_cast<size_t>(na) * (c_ins + 12) + 1);
  double* fq = qtab.data();
  double* mean = fq + static_cast<size_t>(na) * c_ins;
  double* inv = mean + 3 * na;
  for (int a = 0; a < na; ++a) {
    const int q = alive_index[a];
    for (int c = 0; c < c_ins; ++c) fq[a * c_ins + c] = qs->feature[static_cast<int64_t>(q) * c_ins + c];
    for (int i = 0; i < 3; ++i) mean[a * 3 + i] = qs->mean[q * 3 + i];
    psm_query_inverse(qs->cov + q * 9, inv + a * 9);
  }
  const int D = sc->c_sem + nq;
  const bool exact = sc->feat64 != nullptr || (sc->flags & PSM_SCENE_EXACT_FEATURES) || nq > 0;
  cudaStream_t st = ctx->stream;
  // the rows are rewritten in place when the width is unchanged (each thread reads its
  // own row's f_sem columns before writing it); otherwise into new buffers
  const bool in_place = nq == sc->n_q && (D == 0 || (sc->feat && (!exact || sc->feat64)));
  float* feat = in_place ? sc->feat : nullptr;
  double* feat64 = in_place ? sc->feat64 : nullptr;
  if (!in_place && n > 0 && D > 0) {
    cudaError_t e = cudaMalloc(&feat, sizeof(float) * n * D);
    if (e == cudaSuccess && exact) e = cudaMalloc(&feat64, sizeof(double) * n * D);
    if (e != cudaSuccess) {
      cudaFree(feat);
      return psm::fail_cuda(ctx, e, "assign_labels feature rows", __FILE__, __LINE__);
    }
  }
  double *dqtab = nullptr, *scratch = nullptr, *ddist = nullptr;
  int32_t *didx = nullptr, *darg = nullptr;
  PSM_TRY(psm::ensure(ctx, ctx->lab_tmp, qtab.size() + static_cast<size_t>(na) + (nq > 0 ? nq : 1), &dqtab));
  didx = reinterpret_cast<int32_t*>(dqtab + qtab.size());
  PSM_CUDA_TRY(cudaMemcpyAsync(dqtab, qtab.data(), sizeof(double) * qtab.size(), cudaMemcpyHostToDevice, st));
  if (na > 0)
    PSM_CUDA_TRY(cudaMemcpyAsync(didx, alive_index.data(), sizeof(int32_t) * na, cudaMemcpyHostToDevice, st));
  PSM_CUDA_TRY(cudaMemcpyAsync(didx + na, alive_slot.data(), sizeof(int32_t) * (nq > 0 ? nq : 1),
                               cudaMemcpyHostToDevice, st));
  if (n > 0 && na > 0) PSM_TRY(psm::ensure(ctx, ctx->lab_scratch, static_cast<size_t>(n) * na, &scratch));
  if (n > 0 && dist_out && nq > 0) PSM_TRY(psm::ensure(ctx, ctx->lab_dist, static_cast<size_t>(n) * nq, &ddist));
  if (n > 0 && argmax_out) PSM_TRY(psm::ensure(ctx, ctx->lab_arg, static_cast<size_t>(n), &darg));
  psm::LabelParams lp;
  lp.n = n;
  lp.c_sem = sc->c_sem;
  lp.n_q = nq;
  lp.d_in = sc->c_sem + sc->n_q;
  lp.c_ins = c_ins;
  lp.n_alive = na;
  lp.surfels = sc->surfels;
  lp.f_ins = sc->f_ins;
  lp.feat_in = sc->feat;
  lp.feat64_in = sc->feat64;
  lp.feat_out = feat;
  lp.feat64_out = feat64;
  lp.q_feat = dqtab;
  lp.q_mean = dqtab + static_cast<size_t>(na) * c_ins;
  lp.q_inv = lp.q_mean + 3 * na;
  lp.alive_index = didx;
  lp.alive_slot = didx + na;
  lp.scratch = scratch;
  lp.dist = ddist;
  lp.argmax = darg;
  if (n > 0 && na > 0 && c_ins > 0 && !sc->f_ins) {
    if (!in_place) { cudaFree(feat); cudaFree(feat64); }
    return fail(ctx, PSM_EINVAL, "assign_labels: the scene has no f_ins");
  }
  if (n > 0 && (D > 0 || darg)) psm::launch_assign_labels(lp, st);
  PSM_CUDA_TRY(cudaGetLastError());
  if (!in_place) {  // retire the old rows once the kernel has read them
    PSM_CUDA_TRY(cudaStreamSynchronize(st));
    if (n > 0 && D > 0) {
      cudaFree(sc->feat);
      cudaFree(sc->feat64);
      sc->feat = feat;
      sc->feat64 = feat64;
    }
  }
  sc->n_q = nq;
  if (ddist) PSM_CUDA_TRY(cudaMemcpyAsync(dist_out, ddist, sizeof(double) * n * nq, cudaMemcpyDeviceToHost, st));
  if (darg) PSM_CUDA_TRY(cudaMemcpyAsync(argmax_out, darg, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st));
  if (dist_out || argmax_out) PSM_CUDA_TRY(cudaStreamSynchronize(st));
  if (argmax_out && n > 0 && na == 0)
    for (int64_t i = 0; i < n; ++i) argmax_out[i] = -1;
  if (dist_out && nq > 0 && n > 0 && !ddist) std::memset(dist_out, 0, sizeof(double) * n * nq);
  return PSM_OK;
}

}  // extern "C"

namespace psm {

// The forward in cache mode (RenderCache, raster.cpp:310-315,399-403): planes in context
// scratch; every pixel's contributors (tile-list position, transmittance before it) in the
// context's lists; re-rendered until its buffers fit. Synchronous.
int cache_forward(psm_ctx* ctx, const psm_scene* sc, const psm_camera* cam, const psm_raster_config* cfg, Planes& pl) {
  cudaStream_t st = ctx->stream;
  const size_t npx = static_cast<size_t>(cam->width) * cam->height;
  pl = Planes{};
  PSM_TRY(ensure(ctx, ctx->plane_color, npx * 3, &pl.color));
  PSM_TRY(ensure(ctx, ctx->plane_depth, npx * 2, &pl.depth));
  PSM_TRY(ensure(ctx, ctx->plane_normal, npx * 3, &pl.normal));
  PSM_TRY(ensure(ctx, ctx->plane_alpha, npx, &pl.alpha));
  PSM_TRY(ensure(ctx, ctx->plane_arg, npx, &pl.arg));
  PSM_TRY(ensure(ctx, ctx->plane_cnt, npx, &pl.cnt));
  pl.sem = nullptr;
  pl.ins = nullptr;
  pl.cache = true;
  if (ctx->list_cap == 0) ctx->list_cap = 128;
  PSM_TRY(drain_twin(ctx));  // validate earlier asynchronous frames first
  if (!ctx->pend.empty()) PSM_TRY(sync_impl(ctx));
  ctx->h_small = ctx->h_ring + 8 * psm_ctx::kMaxPend;
  for (int attempt = 0;; ++attempt) {
    PSM_TRY(render_impl(ctx, sc, cam, cfg, pl, nullptr));
    PSM_CUDA_TRY(cudaStreamSynchronize(st));
    bool rerun = false;
    PSM_TRY(check_frame(ctx, &rerun));
    if (!rerun) break;
    if (attempt >= 3) return fail(ctx, PSM_ENOMEM, "render buffers did not converge");
  }
  finish_counters(ctx);
  return PSM_OK;
}

}  // namespace psm

extern "C" {

int psm_render_backward(psm_ctx* ctx, const psm_scene* sc, const psm_camera* cam, const psm_raster_config* cfg,
                        const psm_plane_grads* g, psm_scene_grads* out) {
  if (!ctx || !sc || !cam || !cfg || !g || !out) return PSM_EINVAL;
  if (cam->width <= 0 || cam->height <= 0) return psm::fail(ctx, PSM_EINVAL, "camera: image size must be positive");
  PSM_TRY(psm::check_config(ctx, cfg, sc->c_sem + sc->n_q));
  PSM_CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  const int64_t n = sc->n;
  const int cs = sc->c_sem, nq = sc->n_q, W = cam->width, H = cam->height;
  const size_t npx = static_cast<size_t>(W) * H;
  psm::Planes pl{};
  PSM_TRY(psm::cache_forward(ctx, sc, cam, cfg, pl));
  psm::finish_counters(ctx);
  // upstream plane gradients to the device
  const size_t n_gc = g->color ? npx * 3 : 0, n_gs = (g->sem_feat && cs > 0) ? npx * cs : 0,
               n_gi = (g->ins_dist && nq > 0) ? npx * nq : 0;
  double* gin = nullptr;
  PSM_TRY(psm::ensure(ctx, ctx->bw_gin, n_gc + n_gs + n_gi + 1, &gin));
  if (n_gc) PSM_CUDA_TRY(cudaMemcpyAsync(gin, g->color, sizeof(double) * n_gc, cudaMemcpyHostToDevice, st));
  if (n_gs)
    PSM_CUDA_TRY(cudaMemcpyAsync(gin + n_gc, g->sem_feat, sizeof(double) * n_gs, cudaMemcpyHostToDevice, st));
  if (n_gi)
    PSM_CUDA_TRY(cudaMemcpyAsync(gin + n_gc + n_gs, g->ins_dist, sizeof(double) * n_gi, cudaMemcpyHostToDevice, st));
  // gradient accumulators: opacity, colour, f_sem, labels, H^-1 (summed), centre, quaternion, scales
  const size_t nn = static_cast<size_t>(n);
  const size_t o_op = 0, o_col = nn, o_fs = o_col + 3 * nn, o_lab = o_fs + cs * nn, o_h = o_lab + nq * nn,
               o_c = o_h + 9 * nn, o_r = o_c + 3 * nn, o_s = o_r + 4 * nn, total = o_s + 2 * nn;
  double* acc = nullptr;
  PSM_TRY(psm::ensure(ctx, ctx->bw_out, total + 1, &acc));
  PSM_CUDA_TRY(cudaMemsetAsync(acc, 0, sizeof(double) * (o_c + 1), st));
  if (n > 0) {
    psm::BackwardParams bp{};
    bp.width = W;
    bp.height = H;
    bp.k_sel = cfg->top_k > 1 ? cfg->top_k : 1;
    bp.topk = cfg->blending == PSM_BLEND_TOPK;
    bp.list_cap = ctx->list_cap;
    bp.c_sem = cs;
    bp.n_q = nq;
    bp.cam_cx = cam->cx; bp.cam_cy = cam->cy; bp.cam_fx = cam->fx; bp.cam_fy = cam->fy;
    bp.bg0 = cfg->background[0]; bp.bg1 = cfg->background[1]; bp.bg2 = cfg->background[2];
    bp.lists = static_cast<const uint2*>(ctx->lists.p);
    bp.lists_t = static_cast<const double*>(ctx->lists_t.p);
    bp.topk_pos = bp.topk ? static_cast<const int32_t*>(ctx->topk_pos.p) : nullptr;
    bp.blend_count = pl.cnt;
    bp.vals = static_cast<const uint32_t*>(ctx->tvals.p);
    bp.recs = static_cast<const psm::SurfRec*>(ctx->recs.p);
    bp.surfels = sc->surfels;
    bp.feat64 = sc->feat64;
    bp.feat32 = sc->feat;
    bp.g_color = n_gc ? gin : nullptr;
    bp.g_sem = n_gs ? gin + n_gc : nullptr;
    bp.g_ins = n_gi ? gin + n_gc + n_gs : nullptr;
    bp.d_opacity = acc + o_op;
    bp.d_color = acc + o_col;
    bp.d_fsem = acc + o_fs;
    bp.d_lab = acc + o_lab;
    bp.d_hinv = acc + o_h;
    psm::launch_pixel_backward(bp, st);
    PSM_CUDA_TRY(cudaGetLastError());
    psm::DevCamera dc;
    std::memcpy(dc.r, cam->r_cw, sizeof dc.r);
    psm::launch_geom_backward(sc->surfels, bp.recs, static_cast<const int32_t*>(ctx->valid.p), n, dc, acc + o_h,
                              acc + o_c, acc + o_r, acc + o_s, st);
    PSM_CUDA_TRY(cudaGetLastError());
  }
  auto d2h = [&](double* dst, size_t off, size_t count) -> int {
    if (dst && count) PSM_CUDA_TRY(cudaMemcpyAsync(dst, acc + off, sizeof(double) * count, cudaMemcpyDeviceToHost, st));
    return PSM_OK;
  };
  PSM_TRY(d2h(out->opacity, o_op, nn));
  PSM_TRY(d2h(out->color, o_col, 3 * nn));
  PSM_TRY(d2h(out->f_sem, o_fs, cs * nn));
  PSM_TRY(d2h(out->labels, o_lab, nq * nn));
  PSM_TRY(d2h(out->center, o_c, 3 * nn));
  PSM_TRY(d2h(out->rotation, o_r, 4 * nn));
  PSM_TRY(d2h(out->scales, o_s, 2 * nn));
  PSM_CUDA_TRY(cudaStreamSynchronize(st));
  return PSM_OK;
}

int psm_render_cache(psm_ctx* ctx, const psm_scene* sc, const psm_camera* cam, const psm_raster_config* cfg,
                     const psm_targets* targets, psm_counters* counters, psm_render_cache_out* cache) {
  if (!ctx || !sc || !cam || !cfg || !targets) return PSM_EINVAL;
  // 1. the render itself into the caller's targets (synchronous: counters requested)
  psm_counters c{};
  PSM_TRY(psm::render_common(ctx, sc, cam, cfg, targets, &c, nullptr));
  if (counters) *counters = c;
  if (!cache) return PSM_OK;
  cudaStream_t st = ctx->stream;
  const int64_t n = sc->n;
  const int W = cam->width, H = cam->height;
  const int64_t npx = static_cast<int64_t>(W) * H;
  // 2. the forward in cache mode: contributor lists in context scratch
  psm::Planes pl{};
  PSM_TRY(psm::cache_forward(ctx, sc, cam, cfg, pl));
  const int tiles = ctx->last.tiles_x * ctx->last.tiles_y;
  const int64_t rn = static_cast<int64_t>(ctx->last.rn_total);
  // 3. projected index of every source: exclusive scan of the projection flags
  uint32_t *proj_of = nullptr, *scan_tmp = nullptr, *n_proj_dev = nullptr;
  int64_t* offs = nullptr;
  uint32_t* scan_tmp2 = nullptr;
  uint32_t* tot = nullptr;
  PSM_TRY(psm::ensure(ctx, ctx->pos, n > 0 ? n : 1, &proj_of));
  PSM_TRY(psm::ensure(ctx, ctx->scan_tmp, psm::scan_cta_words(n > npx ? n : npx) + 8, &scan_tmp));
  PSM_TRY(psm::ensure(ctx, ctx->totals, 512, &tot));
  n_proj_dev = tot + 256;
  uint32_t n_proj = 0;
  if (n > 0) {
    psm::exclusive_scan_i32(static_cast<const int32_t*>(ctx->valid.p), n, proj_of, n_proj_dev, scan_tmp, st);
    PSM_CUDA_TRY(cudaGetLastError());
    PSM_CUDA_TRY(cudaMemcpyAsync(&n_proj, n_proj_dev, sizeof n_proj, cudaMemcpyDeviceToHost, st));
    PSM_CUDA_TRY(cudaStreamSynchronize(st));
  }
  cache->n_projected = n_proj;
  cache->n_tile_entries = rn;
  // per-pixel offsets: exclusive scan of the contributor counts (<= list_cap after cache_forward)
  uint32_t* off32 = nullptr;
  PSM_TRY(psm::ensure(ctx, ctx->keys_c, npx + 1, reinterpret_cast<uint64_t**>(&offs)));
  PSM_TRY(psm::ensure(ctx, ctx->src_c, npx + 1, &off32));
  scan_tmp2 = tot + 300;
  uint32_t total = 0;
  if (npx > 0) {
    psm::exclusive_scan_i32(pl.cnt, npx, off32, scan_tmp2, scan_tmp, st);
    PSM_CUDA_TRY(cudaGetLastError());
    PSM_CUDA_TRY(cudaMemcpyAsync(&total, scan_tmp2, sizeof total, cudaMemcpyDeviceToHost, st));
    PSM_CUDA_TRY(cudaStreamSynchronize(st));
  }
  cache->n_contribs = total;
  std::vector<int64_t> hoffs(static_cast<size_t>(npx) + 1);
  {
    std::vector<uint32_t> h32(static_cast<size_t>(npx));
    if (npx > 0) PSM_CUDA_TRY(cudaMemcpy(h32.data(), off32, sizeof(uint32_t) * npx, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < npx; ++i) hoffs[i] = h32[i];
    hoffs[npx] = total;
  }
  if (cache->pixel_offsets) std::memcpy(cache->pixel_offsets, hoffs.data(), sizeof(int64_t) * (npx + 1));
  if (cache->contribs && cache->contribs_cap >= static_cast<int64_t>(total) && total > 0) {
    psm_contribution* dcon = nullptr;
    PSM_CUDA_TRY(cudaMemcpyAsync(offs, hoffs.data(), sizeof(int64_t) * (npx + 1), cudaMemcpyHostToDevice, st));
    PSM_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&dcon), sizeof(psm_contribution) * total, st));
    psm::launch_cache_pixels(static_cast<const uint2*>(ctx->lists.p), ctx->list_cap, pl.cnt, offs,
                             static_cast<const uint32_t*>(ctx->tvals.p), static_cast<const psm::SurfRec*>(ctx->recs.p),
                             proj_of, W, H, cam->cx, cam->cy, cam->fx, cam->fy, dcon, st);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(cache->contribs, dcon, sizeof(psm_contribution) * total, cudaMemcpyDeviceToHost, st);
    cudaFreeAsync(dcon, st);
    if (e != cudaSuccess) return psm::fail_cuda(ctx, e, "cache contributions", __FILE__, __LINE__);
    PSM_CUDA_TRY(cudaStreamSynchronize(st));
  }
  // 4. RenderCache::projected (source order) and the tile lists as projected indices
  if (cache->projected && cache->projected_cap >= static_cast<int64_t>(n_proj) && n_proj > 0) {
    psm_projected* dproj = nullptr;
    PSM_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&dproj), sizeof(psm_projected) * n_proj, st));
    psm::DevCamera dc;
    std::memcpy(dc.r, cam->r_cw, sizeof dc.r);
    std::memcpy(dc.t, cam->t_cw, sizeof dc.t);
    dc.fx = cam->fx; dc.fy = cam->fy; dc.cx = cam->cx; dc.cy = cam->cy;
    dc.w = W; dc.h = H; dc.near_clip = cam->near_clip; dc.far_clip = cam->far_clip;
    psm::launch_cache_projected(sc->surfels, n, dc, cfg->chi2, static_cast<const int32_t*>(ctx->valid.p), proj_of,
                                dproj, st);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(cache->projected, dproj, sizeof(psm_projected) * n_proj, cudaMemcpyDeviceToHost, st);
    cudaFreeAsync(dproj, st);
    if (e != cudaSuccess) return psm::fail_cuda(ctx, e, "cache projected", __FILE__, __LINE__);
    PSM_CUDA_TRY(cudaStreamSynchronize(st));
  }
  if (cache->tile_counts || (cache->tile_lists && cache->tile_lists_cap >= rn)) {
    std::vector<int32_t> rg(static_cast<size_t>(tiles) * 2);
    if (tiles > 0)
      PSM_CUDA_TRY(cudaMemcpy(rg.data(), ctx->ranges.p, sizeof(int32_t) * 2 * tiles, cudaMemcpyDeviceToHost));
    if (cache->tile_counts)
      for (int t = 0; t < tiles; ++t) cache->tile_counts[t] = rg[2 * t + 1] - rg[2 * t];
    if (cache->tile_lists && cache->tile_lists_cap >= rn && rn > 0) {
      // the tile buckets are dense in tile order over [0, rn_total) (K3's exclusive scan)
      int32_t* dl = nullptr;
      PSM_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&dl), sizeof(int32_t) * rn, st));
      psm::launch_gather_proj(static_cast<const uint32_t*>(ctx->tvals.p), proj_of, rn, dl, st);
      std::vector<int32_t> all(static_cast<size_t>(rn));
      cudaError_t e = cudaGetLastError();
      if (e == cudaSuccess) e = cudaMemcpyAsync(all.data(), dl, sizeof(int32_t) * rn, cudaMemcpyDeviceToHost, st);
      cudaFreeAsync(dl, st);
      if (e == cudaSuccess) e = cudaStreamSynchronize(st);
      if (e != cudaSuccess) return psm::fail_cuda(ctx, e, "cache tile lists", __FILE__, __LINE__);
      int64_t at = 0;
      for (int t = 0; t < tiles; ++t)
        for (int32_t q = rg[2 * t]; q < rg[2 * t + 1]; ++q) cache->tile_lists[at++] = all[q];
    }
  }
  return PSM_OK;
}

int psm_render_panoptic(psm_ctx* ctx, const psm_scene* scene, const psm_camera* cam, const psm_raster_config* cfg,
                        const int32_t* query_class, int32_t n_query_class, const psm_panoptic_targets* targets,
                        psm_counters* counters) {
  if (!targets) return PSM_EINVAL;
  return psm::render_common(ctx, scene, cam, cfg, nullptr, counters, nullptr, targets, query_class, n_query_class);
}

int psm_scene_free(psm_ctx* ctx, psm_scene* sc) {
  if (!sc) return PSM_OK;
  if (ctx) {  // settle this context's pending asynchronous frames, which may still reference the scene
    PSM_TRY(psm::drain_twin(ctx));
    if (!ctx->pend.empty()) PSM_TRY(psm::sync_impl(ctx));
  }
  cudaSetDevice(sc->device);
  if (sc->surfels) cudaFree(sc->surfels);
  if (sc->feat) cudaFree(sc->feat);
  if (sc->feat64) cudaFree(sc->feat64);
  if (sc->f_ins) cudaFree(sc->f_ins);
  delete sc;
  return PSM_OK;
}

int psm_scene_info(const psm_scene* sc, int64_t* n, int32_t* c_sem, int32_t* n_q) {
  if (!sc) return PSM_EINVAL;
  if (n) *n = sc->n;
  if (c_sem) *c_sem = sc->c_sem;
  if (n_q) *n_q = sc->n_q;
  return PSM_OK;
}

int psm_render(psm_ctx* ctx, const psm_scene* scene, const psm_camera* cam, const psm_raster_config* cfg,
               const psm_targets* targets, psm_counters* counters) {
  return psm::render_common(ctx, scene, cam, cfg, targets, counters, nullptr);
}

int psm_render_debug(psm_ctx* ctx, const psm_scene* scene, const psm_camera* cam, const psm_raster_config* cfg,
                     const psm_targets* targets, psm_counters* counters, psm_debug* debug) {
  return psm::render_common(ctx, scene, cam, cfg, targets, counters, debug);
}

int psm_render_batch(psm_ctx* ctx, const psm_scene* scene, const psm_camera* cams, int32_t n_views,
                     const psm_raster_config* cfg, const psm_targets* targets, psm_counters* counters) {
  if (!ctx || !cams || !targets || n_views < 0) return PSM_EINVAL;
  bool pipelined = !counters && n_views >= 2;
  for (int32_t v = 0; v < n_views && pipelined; ++v) pipelined = targets[v].on_device != 0;
  if (!pipelined) {  // counters or host planes: every view synchronises anyway
    for (int32_t v = 0; v < n_views; ++v) {
      const int st = psm_render(ctx, scene, cams + v, cfg, targets + v, counters ? counters + v : nullptr);
      if (st != PSM_OK) return st;
    }
    return PSM_OK;
  }
  // device targets, no counters: views alternate between this context and its twin on two
  // streams (asynchronous, like psm_render; psm_sync validates both contexts' frames)
  // earlier unvalidated frames first: a re-render after this batch could overwrite its planes
  if (ctx->twin_pending || !ctx->pend.empty()) PSM_TRY(psm_sync(ctx));
  PSM_CUDA_TRY(cudaSetDevice(ctx->device));
  if (!ctx->twin) {
    PSM_TRY(psm_create(ctx->device, nullptr, &ctx->twin));
    PSM_CUDA_TRY(cudaEventCreateWithFlags(&ctx->batch_fork, cudaEventDisableTiming));
    PSM_CUDA_TRY(cudaEventCreateWithFlags(&ctx->batch_join, cudaEventDisableTiming));
  }
  psm_ctx* tw = ctx->twin;
  tw->profiling = ctx->profiling;
  PSM_CUDA_TRY(cudaEventRecord(ctx->batch_fork, ctx->stream));  // the twin starts after earlier work
  PSM_CUDA_TRY(cudaStreamWaitEvent(tw->stream, ctx->batch_fork, 0));
  for (int32_t v = 0; v < n_views; ++v) {
    psm_ctx* c = (v & 1) ? tw : ctx;
    const int st = psm_render(c, scene, cams + v, cfg, targets + v, nullptr);
    if (st != PSM_OK) return c == ctx ? st : fail(ctx, st, std::string("batch view: ") + tw->err);
  }
  ctx->twin_pending = true;
  ctx->twin_last = (n_views & 1) == 0;
  PSM_CUDA_TRY(cudaEventRecord(ctx->batch_join, tw->stream));  // later work on ctx->stream sees every view
  PSM_CUDA_TRY(cudaStreamWaitEvent(ctx->stream, ctx->batch_join, 0));
  return PSM_OK;
}

}  // extern "C"
