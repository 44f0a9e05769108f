// psm_ctx.h — the opaque C-ABI handles (psm_ctx, psm_scene) and the context's scratch,
// shared by capi.cu (render pipeline) and stages.cu (stage entry points).
#ifndef PSM_CTX_H
#define PSM_CTX_H

#include <string>
#include <vector>

#include "psm_device.cuh"

struct psm_scene {
  int device = 0;
  int64_t n = 0;
  int32_t c_sem = 0, n_q = 0;
  double* surfels = nullptr;  // N x 13 fp64
  float* feat = nullptr;      // N x (c_sem + n_q) fp32
  double* feat64 = nullptr;   // N x (c_sem + n_q) fp64 (PSM_SCENE_EXACT_FEATURES)
  double* f_ins = nullptr;    // N x c_ins fp64 (assign_labels)
  int32_t c_ins = 0;
  int32_t flags = 0;
};

namespace psm {

struct Buf {
  void* p = nullptr;
  size_t bytes = 0;
};

struct Planes {
  float *color, *depth, *normal, *sem, *ins, *alpha;
  int32_t *arg, *cnt;
  // render_panoptic (pan_ids != NULL): the three id planes and the device query classes
  int32_t *pan_ids = nullptr, *pan_classes = nullptr, *pan_sem = nullptr;
  const int32_t* qclass = nullptr;
  int32_t n_qclass = 0;
  bool cache = false;  // backward cache: per-pixel contributor lists with transmittance
};

}  // namespace psm

struct psm_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaStream_t side = nullptr, side2 = nullptr;  // concurrent side work within a frame (large tile buckets)
  cudaEvent_t fork = nullptr, join = nullptr, join2 = nullptr;
  cudaStream_t copy = nullptr;   // device-to-host copies of finished row bands (host targets)
  cudaEvent_t band_ev[8] = {};
  cudaEvent_t copy_done = nullptr;
  std::string err;
  bool profiling = false;
  cudaEvent_t ev[8] = {};
  int ev_next = 0;
  psm_stage_times times{};
  psm_counters last{};
  // scratch
  psm::Buf recs, bins, depth_bits, dminmax, tile_counts, cursor, tile_totals, tile_start, kscratch, kscratch2, valid, pos, keys_c, src_c, keys_s, src_s;
  psm::Buf tkeys, tvals, tkeys2, tvals2, ranges, scan_tmp, hist, khist, totals, dev_small, lists, rank_of, dbg_keys, topk_dbg;
  psm::Buf lists_w, pan_ids, pan_classes, pan_sem, qclass, lab_tmp, lab_scratch, lab_dist, lab_arg;
  psm::Buf lists_t, topk_pos, bw_gin, bw_out, tmasks, tclasses;
  int64_t key_cap = 0;   // tile-key capacity (grow-only, from RN-Total)
  int32_t list_cap = 0;  // Full-mode per-pixel list capacity (grow-only)
  psm::Buf plane_color, plane_depth, plane_normal, plane_sem, plane_ins, plane_arg, plane_alpha, plane_cnt;
  // Pinned counter read-back: one 8-slot record per pending asynchronous frame plus one
  // for synchronous frames (h_ring[kMaxPend]); h_small points at the current frame's.
  static constexpr int kMaxPend = 64;
  int64_t* h_ring = nullptr;
  int64_t* h_small = nullptr;
  // Asynchronous frames (device targets, no counters) not yet validated: psm_sync checks
  // each one's counters in order and, from the first that outgrew its buffers, re-renders
  // it and every later one (so planes shared between pending frames end as the last wrote
  // them). A synchronous frame, or a full list, drains the list first.
  struct Pending {
    const psm_scene* scene;
    psm_camera cam;
    psm_raster_config cfg;
    psm::Planes pl;
  };
  std::vector<Pending> pend;
  // psm_render_batch: a second context (own stream and scratch) that renders every other
  // view, so one view's front end overlaps the other's blend and the small latency-bound
  // launches interleave; created on first use, joined back into `stream` after the batch.
  psm_ctx* twin = nullptr;
  cudaEvent_t batch_fork = nullptr, batch_join = nullptr;
  bool twin_pending = false;  // the twin rendered views not yet validated (psm_sync drains it)
  bool twin_last = false;     // ... including the batch's last view (its counters are the last)
};


#define PSM_TRY(expr)            \
  do {                           \
    int _st = (expr);            \
    if (_st != PSM_OK) return _st; \
  } while (0)

namespace psm {
int fail_cuda(psm_ctx* ctx, cudaError_t e, const char* expr, const char* file, int line);
}  // namespace psm

#endif  // PSM_CTX_H
